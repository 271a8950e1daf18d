"""Time to a certified cut (gap <= 1e-6, checks every 10) on one workload under
solver-configuration variants: precision, polish hand-over, level sets.

    python tools/ttc_variants.py WL [variant ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paracut_b200 as pc  # noqa: E402
from paracut_b200.instances import CONFIGS, make_instance  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
g = make_instance(CONFIGS[wl], seed=0)
thr = (0.0, 1e-6, -1e-6, 1e-3)
variants = {
    "f32": dict(precision="f32"),
    "f32+polish40": dict(precision="f32", polish_iters=5000, polish_stall=40),
    "f32+polish20": dict(precision="f32", polish_iters=5000, polish_stall=20),
    "f32+polish10": dict(precision="f32", polish_iters=5000, polish_stall=10),
    "f32+polish10g": dict(precision="f32", polish_iters=5000, polish_stall=10, polish_gap=1e-2),
    "f32+polish5g": dict(precision="f32", polish_iters=5000, polish_stall=5, polish_gap=1e-2),
    "f64s": dict(precision="f64s"),
    "f32+polish20+levels": dict(precision="f32", polish_iters=5000, polish_stall=20, level_sets=True),
    "f64s+levels": dict(precision="f64s", level_sets=True),
}
names = sys.argv[2:] or list(variants)
for name in names:
    kw = variants[name]
    cfg = pc.SolverConfig(max_iters=kw.pop("max_iters", 5000), check_every=10, thresholds=thr, **kw)
    pc.solve(g, pc.decompose_grid(g), cfg)  # warm
    t0 = time.perf_counter()
    res = pc.solve(g, pc.decompose_grid(g), cfg)
    dt = time.perf_counter() - t0
    ps = res.monitor.get("polish_start")
    gaps = [round(r.gap, 3) for r in res.trace][::10]
    print("%-22s %.3f s  iterations %d  certified %s  gap %.2e  polish_start %s"
          % (name, dt, res.iterations, res.certified, res.gap, ps[0] if ps else None), flush=True)
    print("   gaps every 100 it:", gaps[:40], flush=True)
