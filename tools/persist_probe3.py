import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paracut_b200 as pc
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance
g = make_instance(CONFIGS["cfg3"], seed=5, dims=(96, 80))
for ps in ("1", "0", "1"):
    os.environ["PCB_PERSIST"] = ps
    S = _native.GridSolver(g, precision="f32")
    S.init_cold()
    bad = None
    for it in range(150):
        S.run(1, norms=False)
        if it % 10 == 9 or it > 140:
            z = S.get_z()
            if not np.all(np.isfinite(z)):
                bad = it
                break
    print(ps, "first non-finite at", bad)
    res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=150, check_every=151, precision="f32"))
    x = g.w - res.dual_state.y.sum(axis=0)
    print(ps, "solve x finite", np.all(np.isfinite(x)))
