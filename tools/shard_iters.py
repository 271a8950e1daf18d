"""A short sharded run for ncu: P virtual ranks, overlapped schedule, fused last family."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paracut_b200 import _native  # noqa: E402
from paracut_b200.distributed import LocalComm, ShardedAAR  # noqa: E402
from paracut_b200.instances import CONFIGS, make_instance  # noqa: E402

wl, P, fu = sys.argv[1], int(sys.argv[2]), sys.argv[3] == "1"
g = make_instance(CONFIGS[wl], seed=0)
sh = ShardedAAR(g, LocalComm(P), range(P), lambda s: _native.GridSolver(s, precision="f32"),
                device="cuda", overlap=True, fused_last=fu)
sh.init_cold()
sh.run(8, norms=False)
torch.cuda.synchronize()
print("ok")
