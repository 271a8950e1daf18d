"""Handle creation (weights upload) and get_best rates at cfg5 size."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from paracut_b200 import _native
from paracut_b200.instances import make_instance
g = make_instance(sys.argv[1] if len(sys.argv) > 1 else "cfg5", seed=0)
nbytes = g.w.nbytes + sum(a.nbytes for a in g.dir_weights)
for rep in range(3):
    t0 = time.perf_counter()
    S = _native.GridSolver(g, precision="f32")
    S.synchronize()
    t1 = time.perf_counter()
    S.init_cold(); S.shadow(); S.check(np.array([0.0])); S.keep_best(0); S.synchronize()
    t2 = time.perf_counter()
    lab, x = S.get_best()
    t3 = time.perf_counter()
    S.close()
    print("create %.1f ms (%.1f GB/s)  get_best %.1f ms (%.1f GB/s)" % ((t1 - t0) * 1e3, nbytes / (t1 - t0) / 1e9,
          (t3 - t2) * 1e3, (lab.nbytes + x.nbytes) / (t3 - t2) / 1e9))
