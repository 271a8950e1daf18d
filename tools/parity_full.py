"""Full-size parity outside the test suite (too long for it): the oracle (the
reference loop in its operation order, all host cores) against the device
modes on one BASELINE workload at its iteration count; relative error of
x = w - sum_j y_j.  usage: python tools/parity_full.py cfg5 [iters]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paracut_b200 as pc  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paracut_b200.instances import CONFIGS, make_instance  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
k = int(sys.argv[2]) if len(sys.argv) > 2 else CONFIGS[wl].iters
g = make_instance(CONFIGS[wl], seed=0)
t0 = time.perf_counter()
run = orc.AARRunner(g, threads=orc.max_threads())
run.run(k, final_shadow=True)
x_ref = g.w - run.p.sum(axis=0)
print("%s k=%d oracle %.1f s on %d threads" % (wl, k, time.perf_counter() - t0, orc.max_threads()),
      flush=True)
del run
scale = float(np.max(np.abs(x_ref)))
for prec in ("f32", "f64s"):
    res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=k, check_every=k + 1,
                                                             precision=prec))
    x = g.w - res.dual_state.y.sum(axis=0)
    print("%s k=%d %s: max|x - x_ref| / max|x_ref| = %.3e (tolerance %g)"
          % (wl, k, prec, float(np.max(np.abs(x - x_ref))) / scale, 1e-4 if prec == "f32" else 1e-6),
          flush=True)
    del res, x
