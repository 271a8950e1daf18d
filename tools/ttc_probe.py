"""Wall time to a certified optimal cut (gap <= 1e-6) on BASELINE workloads."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
import paracut_b200 as pc
from paracut_b200.instances import CONFIGS, make_instance

for wl in sys.argv[1:]:
    name, prec = wl.split(":")
    g = make_instance(CONFIGS[name], seed=0)
    for ls in (False, True):
        cfg = pc.SolverConfig(max_iters=3000, check_every=10, precision=prec,
                              thresholds=(0.0, 1e-6, -1e-6, 1e-3), level_sets=ls,
                              polish_iters=500 if prec == "f32" else 0)
        res = None
        t0 = time.perf_counter()
        res = pc.solve(g, pc.decompose_grid(g), cfg)
        wall = time.perf_counter() - t0
        print(json.dumps({"wl": name, "prec": prec, "level_sets": ls, "wall_s": wall,
                          "iters": res.iterations, "certified": bool(res.certified),
                          "gap": res.gap, "energy": res.energy}), flush=True)
