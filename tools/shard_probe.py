"""Per-family kernel times of the sharded path's handles (P virtual ranks on
one GPU), overlapped schedule with and without the fused last slab family."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paracut_b200 import _native  # noqa: E402
from paracut_b200.distributed import LocalComm, ShardedAAR  # noqa: E402
from paracut_b200.instances import CONFIGS, make_instance  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = make_instance(CONFIGS[wl], seed=0)
for fu in (False, True):
    sh = ShardedAAR(g, LocalComm(P), range(P), lambda s: _native.GridSolver(s, precision="f32"),
                    device="cuda", overlap=True, fused_last=fu)
    sh.init_cold()
    sh.run(3, norms=False)
    torch.cuda.synchronize()
    for h in sh.slab + sh.pencil:
        h.set_profiling(True)
    sh.run(10, norms=False)
    torch.cuda.synchronize()
    for name, hs in (("slab", sh.slab), ("pencil", sh.pencil)):
        for h in hs:
            ms, cnt = h.profile_read()
            print("fused=%s %s per-family ms/launch %s launches %s" %
                  (fu, name, [round(float(m) / max(int(c), 1), 4) for m, c in zip(ms, cnt)],
                   [int(c) for c in cnt]), flush=True)
            h.set_profiling(False)
    del sh
