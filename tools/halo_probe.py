"""Debug: 2D-8 halo slabs after set_z vs the global z (which nodes differ)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paracut_b200 import _native
from paracut_b200.distributed import LocalComm, ShardedAAR
from paracut_b200.instances import CONFIGS, make_instance

g = make_instance(CONFIGS["cfg3"], seed=9, dims=(48, 64))
S = _native.GridSolver(g, precision="f32")
S.init_cold()
S.run(15)
z15 = S.get_z()
sh = ShardedAAR(g, LocalComm(4), range(4), lambda sub: _native.GridSolver(sub, precision="f32"),
                device="cuda")
sh.set_z(z15)
z = sh.assemble(sh.local_z())
d = np.abs(z - z15).reshape(4, 48, 64)
for j in range(4):
    bad = np.argwhere(d[j] > 1e-5)
    print(j, d[j].max(), len(bad), bad[:10].tolist(), sorted(set(bad[:, 0].tolist()))[:20])
# round trip on the single handle
S2 = _native.GridSolver(g, precision="f32")
S2.set_z(z15)
print("single roundtrip", np.abs(S2.get_z() - z15).max())
sl = sh.geo.slab_grid(g, 0)
H = _native.GridSolver(sl, precision="f32")
zs = z15.reshape(4, 48, 64)[:, 0:13].reshape(4, -1)
H.set_z(np.ascontiguousarray(zs))
print("slab0 roundtrip", np.abs(H.get_z() - zs).reshape(4, 13, 64).max(axis=(1, 2)))
