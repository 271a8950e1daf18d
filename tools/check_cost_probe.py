"""Cost of one certificate check (shadow, gap pass, packed labels, keep_best)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance

name = sys.argv[1]
g = make_instance(CONFIGS[name], seed=0)
thr = np.array([0.0, 1e-6, -1e-6, 1e-3])
for prec in ("f32", "f64"):
    S = _native.GridSolver(g, precision=prec)
    S.init_cold()
    S.run(20)
    S.synchronize()
    def tm(f, reps=5):
        f(); S.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            f()
        S.synchronize()
        return (time.perf_counter() - t0) / reps * 1e3
    out = {
        "run10": tm(lambda: S.run(10)) / 10,
        "run10_nonorm": tm(lambda: S.run(10, norms=False)) / 10,
        "shadow": tm(lambda: S.shadow()),
        "check4": tm(lambda: S.check(thr)),
        "labels_packed": tm(lambda: S.check_labels(0, packed=True)),
        "keep_best": tm(lambda: S.keep_best(0)),
        "shadow+apply": tm(lambda: (S.shadow(), S.apply())),
        "level_set": tm(lambda: S.level_set()),
    }
    print(name, prec, {k: round(v, 3) for k, v in out.items()}, flush=True)
    S.close()
