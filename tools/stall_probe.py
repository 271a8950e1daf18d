"""f32 + stall-triggered f64 polish: wall time to a certified cut vs the stall window."""
import sys, time, json
sys.path.insert(0, ".")
import paracut_b200 as pc
from paracut_b200.instances import CONFIGS, make_instance

name = sys.argv[1]
g = make_instance(CONFIGS[name], seed=0)
dec = pc.decompose_grid(g)
for W in [int(v) for v in sys.argv[2:]]:
    cfg = pc.SolverConfig(max_iters=4000, check_every=10, precision="f32",
                          thresholds=(0.0, 1e-6, -1e-6, 1e-3), polish_iters=3000,
                          polish_stall=W)
    res = None
    t0 = time.perf_counter()
    res = pc.solve(g, dec, cfg)
    wall = time.perf_counter() - t0
    ps = res.monitor.get("polish_start", [None])[0]
    print(json.dumps({"W": W, "iters": res.iterations, "polish_start": ps,
                      "certified": bool(res.certified), "wall_s": round(wall, 3),
                      "energy": res.energy}), flush=True)
