"""ms per AAR iteration over a cold-start solve, in windows, with the verified
sweeps on (default) and off (PCB_VERIFY=0): where the verified path pays."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paracut_b200 import _native  # noqa: E402
from paracut_b200.instances import CONFIGS, make_instance  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else CONFIGS[wl].iters
win = int(sys.argv[3]) if len(sys.argv) > 3 else 50
g = make_instance(CONFIGS[wl], seed=0)
for mode in ("1", "0"):
    os.environ["PCB_VERIFY"] = mode
    S = _native.GridSolver(g, precision="f32")
    st = torch.cuda.Stream()
    S.set_stream(st.cuda_stream)
    for rep in range(2):
        _native.debug_counters(reset=True)
        S.init_cold()
        out = []
        reps = []
        tot = 0.0
        prev_rep = None
        for w0 in range(0, iters, win):
            n = min(win, iters - w0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            S.run(n, norms=False)
            e1.record(st)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            tot += ms
            out.append(ms / n)
            if mode == "1" and rep == 1:
                vst = S.verify_stats(scans=True)
                cur = (vst[2].sum(), vst[1].sum())
                if prev_rep is not None:
                    dsw = cur[1] - prev_rep[1]
                    reps.append("%.1f%%" % (100.0 * (cur[0] - prev_rep[0]) / max(dsw, 1)
                                           / (g.n / max(g.dims))) if dsw else "-")
                prev_rep = cur
        if rep == 1:
            line = "verify=%s %s total %.1f ms (%.3f ms/iter): " % (mode, wl, tot, tot / iters)
            line += " ".join("%.3f" % v for v in out)
            if mode == "1":
                m_, sw, rp, sc, ch = S.verify_stats(scans=True)
                line += " | verified sweeps %s repaired %s scans %s changed %s" % (
                    list(map(int, sw)), list(map(int, rp)), list(map(int, sc)), list(map(int, ch)))
            if reps:
                line += " | repaired per verified sweep by window %s" % (reps,)
            if mode == "1":
                dc = _native.debug_counters(reset=True)
                line += " | repair fast/noqL/oobsearch/oobstring/slow %s" % (list(map(int, dc[:5])),)
            S.set_profiling(True)
            S.run(20, norms=False)
            torch.cuda.synchronize()
            fms, fc = S.profile_read()
            S.set_profiling(False)
            line += " | last-20 per-family ms %s" % (["%.3f" % (a / max(b, 1)) for a, b in zip(fms, fc)],)
            print(line, flush=True)
    S.close()
