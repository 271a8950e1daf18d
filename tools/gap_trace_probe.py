"""Gap trajectory of an f32 solve (where does fp32 stall on integer data?)."""
import sys, json
sys.path.insert(0, ".")
import paracut_b200 as pc
from paracut_b200.instances import CONFIGS, make_instance

name, iters = sys.argv[1], int(sys.argv[2])
g = make_instance(CONFIGS[name], seed=0)
for prec in ("f32", "f64"):
    cfg = pc.SolverConfig(max_iters=iters, check_every=10, precision=prec,
                          thresholds=(0.0, 1e-6, -1e-6, 1e-3))
    res = pc.solve(g, pc.decompose_grid(g), cfg)
    print(prec, res.iterations, res.certified, json.dumps([(t.iteration, float("%.4g" % t.gap)) for t in res.trace]), flush=True)
