"""Time the slab-sharded driver with P virtual ranks on one GPU (LocalComm).
Not a scaling number (all ranks share one device); it measures the driver's
per-iteration overhead and checks the plumbing at full size."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paracut_b200 import _native  # noqa: E402
from paracut_b200.distributed import LocalComm, ShardedAAR  # noqa: E402
from paracut_b200.instances import CONFIGS, make_instance  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
g = make_instance(CONFIGS[wl], seed=0)
r, n = len(g.dir_weights), g.n
for P, ov in [(P, ov) for P in (1, 2, 4, 8) for ov in (False, True)]:
    sh = ShardedAAR(g, LocalComm(P), range(P), lambda s: _native.GridSolver(s, precision="f32"),
                    device="cuda", overlap=ov)
    sh.init_cold()
    sh.run(3, norms=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sh.run(20, norms=False)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    sh.capture()
    sh.run_graph(3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sh.run_graph(20)
    torch.cuda.synchronize()
    dg = (time.perf_counter() - t0) / 20
    print("%s P=%d virtual ranks on 1 GPU, %s: eager %.3f ms/iter, graph %.3f ms/iter (%.2e updates/s)"
          % (wl, P, "overlapped" if sh.overlap else "serial", dt * 1e3, dg * 1e3, r * n / dg))
    del sh
