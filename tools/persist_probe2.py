import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paracut_b200 as pc
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance
g = make_instance(CONFIGS["cfg3"], seed=5, dims=(96, 80))
for ps in ("1", "0"):
    os.environ["PCB_PERSIST"] = ps
    S = _native.GridSolver(g, precision="f32")
    S.init_cold()
    y, _ = S.shadow(want_y=True)
    print(ps, "shadow0 finite", np.all(np.isfinite(y)), np.abs(y).max())
    S.check(np.array([0.0]))
    S.apply()
    S.run(5)
    y, _ = S.shadow(want_y=True)
    print(ps, "shadow5 finite", np.all(np.isfinite(y)), "z finite", np.all(np.isfinite(S.get_z())))
