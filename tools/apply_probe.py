"""One shadow + check + apply on a BASELINE workload (for ncu of the check kernels)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance

g = make_instance(CONFIGS[sys.argv[1]], seed=0)
S = _native.GridSolver(g, precision=sys.argv[2] if len(sys.argv) > 2 else "f32")
S.init_cold()
S.run(20)
for _ in range(2):
    S.shadow()
    S.check(np.array([0.0, 1e-6, -1e-6, 1e-3]))
    S.apply()
S.synchronize()
print("ok")
