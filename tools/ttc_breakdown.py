"""Time-to-cut wall time split: the same solve with checks every 10
iterations, and the same iteration count with a single final check."""
import sys, time
sys.path.insert(0, ".")
import paracut_b200 as pc
from paracut_b200.instances import CONFIGS, make_instance

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
g = make_instance(CONFIGS[name], seed=0)
thr = (0.0, 1e-6, -1e-6, 1e-3)
cfg = pc.SolverConfig(max_iters=20000, check_every=10, precision="f32", thresholds=thr)
r = pc.solve(g, pc.decompose_grid(g), cfg)  # warm
for rep in range(4):
    t0 = time.perf_counter()
    r = pc.solve(g, pc.decompose_grid(g), cfg)
    _ = r.labeling.sum()
    t1 = time.perf_counter()
    K = r.iterations
    r = None
    r = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=K, check_every=K + 1,
                                                          precision="f32", thresholds=thr))
    _ = r.labeling.sum()
    t2 = time.perf_counter()
    r = None
    print("%s: %d iterations, checks every 10: %.1f ms; one final check: %.1f ms"
          % (name, K, (t1 - t0) * 1e3, (t2 - t1) * 1e3))
