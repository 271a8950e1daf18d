import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paracut_b200 as pc
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance
for wl, dims in (("cfg3", (96, 80)), ("cfg3", (64, 64)), ("cfg2", (96, 80)), ("cfg4", (24, 20, 28)), ("cfg4", (16, 16, 16))):
    g = make_instance(CONFIGS[wl], seed=5, dims=dims)
    out = []
    for ps in ("1", "0"):
        os.environ["PCB_PERSIST"] = ps
        S = _native.GridSolver(g, precision="f32")
        S.init_cold()
        for it in range(20):
            S.run(1, norms=False)
            z = S.get_z()
            if not np.all(np.isfinite(z)):
                break
        out.append((it, np.all(np.isfinite(z)), z))
    print(wl, dims, "persist finite", out[0][1], "at it", out[0][0], "| static finite", out[1][1],
          "maxdiff", float(np.nanmax(np.abs(out[0][2] - out[1][2]))))
