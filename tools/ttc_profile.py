"""cProfile of one time-to-cut solve (where does the host time go?)."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import paracut_b200 as pc
from paracut_b200.instances import CONFIGS, make_instance

g = make_instance(CONFIGS[sys.argv[1]], seed=0)
cfg = pc.SolverConfig(max_iters=20000, check_every=10, precision=sys.argv[2],
                      thresholds=(0.0, 1e-6, -1e-6, 1e-3))
r = pc.solve(g, pc.decompose_grid(g), cfg)  # warm
t0 = time.perf_counter()
r = None
pr = cProfile.Profile()
pr.enable()
r = pc.solve(g, pc.decompose_grid(g), cfg)
_ = r.labeling.sum()
pr.disable()
print("wall", time.perf_counter() - t0, r.iterations)
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
