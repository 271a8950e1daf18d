"""Steady-state timing of one workload for A/B runs: 200 warm-up iterations from
the cold start, then wall time of 200 graph-replayed iterations (three
repeats) and the per-family kernel times of 40 eager iterations."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
prec = sys.argv[2] if len(sys.argv) > 2 else "f32"
g = make_instance(CONFIGS[wl], seed=0)
S = _native.GridSolver(g, precision=prec)
S.set_graph_after(0)
S.init_cold()
S.run(200, norms=False)
S.synchronize()
ts = []
for rep in range(3):
    t0 = time.perf_counter()
    S.run(200, norms=False)
    S.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3 / 200)
S.set_profiling(True)
S.run(40, norms=False)
ms, cnt = S.profile_read()
S.set_profiling(False)
print("%s %s: %.4f ms/iter (min of %s); families %s" % (
    wl, prec, min(ts), " ".join("%.4f" % t for t in ts),
    " ".join("%.4f" % (m / max(c, 1)) for m, c in zip(ms, cnt))), flush=True)
