"""Time-to-certified-cut table (DESIGN 6b): one warm-up solve per row, then the
median of two timed solves (one live handle at a time)."""
import json, statistics, sys, time
sys.path.insert(0, ".")
import paracut_b200 as pc
from paracut_b200.instances import CONFIGS, make_instance

ROWS = [("cfg4", "f32", 0), ("cfg5", "f32", 0), ("cfg2_int", "f64", 0),
        ("cfg2_int", "f32", 10), ("cfg5_int", "f32", 40)]
for name, prec, stall in ROWS:
    if len(sys.argv) > 1 and name not in sys.argv[1:]:
        continue
    g = make_instance(CONFIGS[name], seed=0)
    cfg = pc.SolverConfig(max_iters=4000, check_every=10, precision=prec,
                          thresholds=(0.0, 1e-6, -1e-6, 1e-3),
                          polish_iters=3000 if stall else 0, polish_stall=stall)
    walls, res = [], None
    for rep in range(3):
        res = None
        t0 = time.perf_counter()
        res = pc.solve(g, pc.decompose_grid(g), cfg)
        _ = res.labeling.sum()
        if rep:
            walls.append(time.perf_counter() - t0)
    ps = res.monitor.get("polish_start", [None])[0]
    print(json.dumps({"wl": name, "prec": prec, "polish_stall": stall, "iters": res.iterations,
                      "polish_start": ps, "certified": bool(res.certified),
                      "wall_s": round(statistics.median(walls), 3), "energy": res.energy}),
          flush=True)
    res = None
