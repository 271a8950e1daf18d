"""What separates the plateau labeling from the optimal one?  cfg4 seed 0: the
threshold-0 labeling at iteration 400 against the certified labeling."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paracut_b200 as pc
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
k0 = int(sys.argv[2]) if len(sys.argv) > 2 else 400
g = make_instance(CONFIGS[wl], seed=0)
cfg = pc.SolverConfig(max_iters=20000, check_every=10, precision="f32",
                      thresholds=(0.0, 1e-6, -1e-6, 1e-3), polish_iters=5000, polish_stall=5, polish_gap=1e-2)
res = pc.solve(g, pc.decompose_grid(g), cfg)
opt = res.labeling.astype(bool)
print("certified", res.certified, "iterations", res.iterations, "energy %.6f" % res.energy)
S = _native.GridSolver(g, precision="f32")
S.init_cold()
S.run(k0, norms=False)
S.shadow()
e, gap, dual = S.check(np.array([0.0, 1e-6, -1e-6, 1e-3]))
print("k=%d energies" % k0, e, "gaps", gap)
t = int(np.argmin(gap))
lab = S.check_labels(t).astype(bool)
x = S.check_x(t)
d = np.flatnonzero(lab != opt)
print("differing nodes:", d.size)
dims = g.dims
for i in d[:20]:
    idx = np.unravel_index(i, dims)
    print(" node", idx, "x = %.6g" % x[i], "label", int(lab[i]), "-> optimal", int(opt[i]))
print("|x| quantiles of all nodes:", np.quantile(np.abs(x), [0.0001, 0.001, 0.01]))
print("nodes with |x| < 1e-2:", int((np.abs(x) < 1e-2).sum()), " < 1e-1:", int((np.abs(x) < 1e-1).sum()))
