"""Wall-time breakdown of one bench-style end-to-end solve (cfg4 f32, 200
iterations) through paracut_b200.solve, with PCB_TRACE-style phase timing
taken from the host around each public step."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paracut_b200 as pc
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance

wl = sys.argv[1] if len(sys.argv) > 1 else 'cfg4'
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
g = make_instance(CONFIGS[wl], seed=0)
for rep in range(3):
    t = [time.perf_counter()]
    S = _native.GridSolver(g, precision='f32'); S.synchronize(); t.append(time.perf_counter())
    S.init_cold(); S.synchronize(); t.append(time.perf_counter())
    S.shadow(); S.check(np.array([0.0])); S.check_labels(0, packed=True); S.keep_best(0); t.append(time.perf_counter())
    S.apply(); S.run(K - 1, norms=True); S.synchronize(); t.append(time.perf_counter())
    S.shadow(); S.check(np.array([0.0])); S.check_labels(0, packed=True); S.keep_best(0); t.append(time.perf_counter())
    lab, x = S.get_best(); t.append(time.perf_counter())
    S.close(); del S; t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print("create %.1f init %.1f check0 %.1f run %.1f checkK %.1f get_best %.1f close %.1f  total %.1f ms"
          % (tuple(d) + (sum(d),)))
for rep in range(3):
    t0 = time.perf_counter()
    res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=K, check_every=K + 1, precision='f32'))
    _ = res.labeling.sum()
    t1 = time.perf_counter()
    del res
    print("solve total %.1f ms" % ((t1 - t0) * 1e3))

import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=K, check_every=K + 1, precision='f32'))
_ = res.labeling.sum()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
