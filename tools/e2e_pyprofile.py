"""cProfile (by own time) of the bench's end-to-end solve from pinned inputs."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paracut_b200 as pc
from paracut_b200.instances import CONFIGS, make_instance
from bench import pinned_instance

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = pinned_instance(make_instance(CONFIGS[wl], seed=0))
cfg = pc.SolverConfig(max_iters=K, check_every=K + 1, precision="f32")
for rep in range(3):
    res = None
    t0 = time.perf_counter()
    res = pc.solve(g, pc.decompose_grid(g), cfg)
    t1 = time.perf_counter()
    _ = np.count_nonzero(res.labeling)
    t2 = time.perf_counter()
    print("solve %.2f ms, count_nonzero %.2f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3))
res = None
pr = cProfile.Profile()
pr.enable()
res = pc.solve(g, pc.decompose_grid(g), cfg)
_ = np.count_nonzero(res.labeling)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
