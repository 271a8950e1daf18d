"""A short gap-checked solve (cfg4 f32, checks every 10, 4 thresholds) for an
ncu launch list of the check cycle's kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paracut_b200 as pc  # noqa: E402
from paracut_b200.instances import CONFIGS, make_instance  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
g = make_instance(CONFIGS[wl], seed=0)
cfg = pc.SolverConfig(max_iters=30, check_every=10, precision="f32",
                      thresholds=(0.0, 1e-6, -1e-6, 1e-3))
res = pc.solve(g, pc.decompose_grid(g), cfg)
print("iterations", res.iterations, "gap", res.gap)
