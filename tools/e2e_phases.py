import sys, time
sys.path.insert(0,'/root/repo')
import numpy as np
import paracut_b200 as pc
from paracut_b200 import _native
from paracut_b200.instances import make_instance
g = make_instance('cfg4', seed=0)
for rep in range(2):
    t0=time.perf_counter()
    S=_native.GridSolver(g, precision='f32'); t1=time.perf_counter()
    S.init_cold(); S.synchronize(); t2=time.perf_counter()
    S.shadow(); e,gp,d=S.check(np.array([0.0])); t3=time.perf_counter()
    lab=S.check_labels(0, packed=True); S.keep_best(0); t4=time.perf_counter()
    S.apply(); n=S.run(99); t5=time.perf_counter()
    S.shadow(); S.check(np.array([0.0])); S.check_labels(0,packed=True); S.keep_best(0); t6=time.perf_counter()
    lab,x=S.get_best(); t7=time.perf_counter()
    print("create %.1f init %.1f check0 %.1f labels %.1f run %.1f check %.1f best %.1f ms" % tuple(1e3*v for v in (t1-t0,t2-t1,t3-t2,t4-t3,t5-t4,t6-t5,t7-t6)))
    del S
t0=time.perf_counter()
res=pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=100, check_every=101, precision='f32'))
print("solve total %.1f ms wall_time %.1f" % ((time.perf_counter()-t0)*1e3, res.wall_time*1e3))
