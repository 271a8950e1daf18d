"""init_cold + N fp32 AAR iterations on one workload (a short command for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paracut_b200 import _native  # noqa: E402
from paracut_b200.instances import CONFIGS, make_instance  # noqa: E402

wl, iters = sys.argv[1], int(sys.argv[2])
g = make_instance(CONFIGS[wl], seed=0)
S = _native.GridSolver(g, precision="f32")
S.init_cold()
S.run(iters, norms=False)
S.synchronize()
if hasattr(S, "verify_stats"):
    print("verify stats", S.verify_stats())
