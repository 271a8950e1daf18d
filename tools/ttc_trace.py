import sys, time
sys.path.insert(0, '.')
import numpy as np
import paracut_b200 as pc
from paracut_b200.instances import CONFIGS, make_instance
g = make_instance(CONFIGS["cfg4"], seed=0)
cfg = pc.SolverConfig(max_iters=20000, check_every=10, precision="f32",
                      thresholds=(0.0, 1e-6, -1e-6, 1e-3), polish_iters=5000, polish_stall=5, polish_gap=1e-2)
for rep in range(2):
    t0 = time.perf_counter()
    res = pc.solve(g, pc.decompose_grid(g), cfg)
    print("wall %.3f iterations %d polish_start %s" % (time.perf_counter() - t0, res.iterations, res.monitor.get("polish_start")))
for row in res.trace[-30:]:
    print(row.iteration, "%.4g" % row.gap, "%.3f" % row.wall_s)
print([ (r.iteration, float("%.3g" % r.gap)) for r in res.trace[::10]])
