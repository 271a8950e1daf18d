"""f32 -> f64 polish: how many exact iterations certify from an f32 state of age K?"""
import sys, time, json
sys.path.insert(0, ".")
import paracut_b200 as pc
from paracut_b200.instances import CONFIGS, make_instance

name = sys.argv[1]
g = make_instance(CONFIGS[name], seed=0)
dec = pc.decompose_grid(g)
for K in [int(v) for v in sys.argv[2:]]:
    cfg = pc.SolverConfig(max_iters=K, check_every=10, precision="f32",
                          thresholds=(0.0, 1e-6, -1e-6, 1e-3), polish_iters=3000)
    res = None
    t0 = time.perf_counter()
    res = pc.solve(g, dec, cfg)
    wall = time.perf_counter() - t0
    print(json.dumps({"K": K, "iters": res.iterations, "polish": res.iterations - K,
                      "certified": bool(res.certified), "wall_s": wall}), flush=True)
