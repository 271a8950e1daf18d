"""Short fixed workload for ncu: build a BASELINE instance, warm up, run a few AAR iterations.

    python tools/profile_step.py [--workload cfg4] [--iters 3] [--precision f32]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paracut_b200 import _native  # noqa: E402
from paracut_b200.instances import CONFIGS, make_instance  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg4")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--precision", default="f32")
ap.add_argument("--dims", default=None)
args = ap.parse_args()
dims = tuple(int(v) for v in args.dims.split("x")) if args.dims else None
g = make_instance(CONFIGS[args.workload], seed=0, dims=dims)
S = _native.GridSolver(g, precision=args.precision)
S.init_cold()
S.run(args.warmup, norms=False)
S.synchronize()
t0 = time.perf_counter()
S.run(args.iters, norms=False)
S.synchronize()
dt = time.perf_counter() - t0
print("workload %s dims %s: %.3f ms/iter (wall)" % (args.workload, g.dims, dt * 1e3 / args.iters))
