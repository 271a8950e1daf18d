import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from paracut_b200 import _native
from paracut_b200.instances import make_instance
g = make_instance('cfg4', seed=0)
for rep in range(3):
    t0 = time.perf_counter()
    S = _native.GridSolver(g, precision='f32')
    t1 = time.perf_counter()
    S.close()
    t2 = time.perf_counter()
    print("create %.1f ms  destroy %.1f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3), flush=True)
