"""Reproduce a fuzz case: f32 with check_every=ce vs the oracle (optionally an older .so)."""
import os, sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paracut_b200 import _native
if len(sys.argv) > 2 and sys.argv[2].endswith(".so"):
    _native.LIB_PATH = os.path.abspath(sys.argv[2])
import paracut_b200 as pc
from test_gpu_fuzz import _random_instance
from oracle import oracle as orc

seed = int(sys.argv[1])
rng = np.random.default_rng(1000 + seed)
g = _random_instance(rng)
_split = str(int(rng.choice([64, 512, 4096])))
os.environ["PCB_SPLIT_TARGET"] = os.environ.get("FORCE_SPLIT") or _split
print("split", os.environ["PCB_SPLIT_TARGET"])
k = int(rng.integers(1, 40))
z_ref, y_ref, _ = orc.aar(g, k, threads=4)
x_ref = g.w - y_ref.sum(axis=0)
dec = pc.decompose_grid(g)
for ce in (k + 1, 1, 2, 3, 5):
    r = pc.solve(g, dec, pc.SolverConfig(max_iters=k, check_every=ce, precision="f32"))
    x = g.w - r.dual_state.y.sum(axis=0)
    print(g.connectivity, g.dims, "k", k, "ce", ce, "iters", r.iterations, r.certified, "err %.3g" % np.max(np.abs(x - x_ref)))
