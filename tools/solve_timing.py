"""Wall time of paracut_b200.solve on a BASELINE workload with gap checks
(time to certified cut when it certifies), per phase."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paracut_b200 as pc  # noqa: E402
from paracut_b200.instances import CONFIGS, make_instance  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
prec = sys.argv[2] if len(sys.argv) > 2 else "f32"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
ce = int(sys.argv[4]) if len(sys.argv) > 4 else 10
g = make_instance(CONFIGS[wl], seed=0)
thr = (0.0, 1e-6, -1e-6, 1e-3, -1e-3) if CONFIGS[wl].integer else (0.0,)
pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=2, check_every=1, precision=prec))
for ce_ in (iters + 1, ce):
    t0 = time.perf_counter()
    res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=iters, check_every=ce_,
                                                            precision=prec, gap_tol=1e-6,
                                                            thresholds=thr))
    wall = time.perf_counter() - t0
    print("%s %s max_iters %d check_every %d: iterations %d certified %s gap %.3g energy %.6f "
          "wall %.3f s (solve wall_time %.3f s)" % (wl, prec, iters, ce_, res.iterations,
                                                    res.certified, res.gap, res.energy, wall,
                                                    res.wall_time))
