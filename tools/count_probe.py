"""Sweep counters (build with -DPCB_COUNT): warp trips / lane gates / bends per node."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
g = make_instance(CONFIGS[wl], seed=0)
S = _native.GridSolver(g, precision="f32")
S.init_cold()
for k0, k1 in ((0, 5), (5, 60), (60, 200)):
    _native.debug_counters(reset=True)
    S.run(k1 - k0, norms=False)
    S.synchronize()
    c = _native.debug_counters(reset=True).astype(float)
    nodes = S.r * S.n * (k1 - k0)
    wpos = nodes / 32
    print("%s iters %d-%d: trips/warp-pos %.3f  gates/node %.3f  bends/node %.3f  issued %.3f retired %.3f (tiles per warp-tile)"
          % (wl, k0, k1, c[0] / wpos, c[1] / nodes, c[2] / nodes, c[3] / (wpos / 8), c[4] / (wpos / 8)))
