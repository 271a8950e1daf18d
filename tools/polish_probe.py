import sys, time
sys.path.insert(0,'/root/repo')
import numpy as np, paracut_b200 as pc
from paracut_b200.instances import make_instance, CONFIGS
g = make_instance(CONFIGS['cfg2_int'], seed=0)
thr=(0.0,1e-6,-1e-6,1e-3,-1e-3)
for k32 in (300, 500, 1000):
    t0=time.perf_counter()
    r32 = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=k32, check_every=k32+1, precision='f32', thresholds=thr))
    z = r32.dual_state.z
    t1=time.perf_counter()
    r64 = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=200, check_every=2, precision='f64', thresholds=thr, gap_tol=0.0, warm_start=pc.DualState(z=z), force_warm=True))
    t2=time.perf_counter()
    print(k32, "f32 gap %.3g E %.1f | polish f64: iters %d certified %s gap %.3g E %.1f | %.2f s + %.2f s" % (r32.gap, r32.energy, r64.iterations, r64.certified, r64.gap, r64.energy, t1-t0, t2-t1))
