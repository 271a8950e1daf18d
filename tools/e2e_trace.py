"""Phase timing of the bench's end-to-end solve (pinned host inputs, K iterations,
certificates at k = 0 and k = K): PCB_TRACE phases of pcb_create on stderr, then
host-timed steps of the same sequence with a sync after each, then the time of
every one of the first K iterations from the cold start."""
import os, sys, time
os.environ.setdefault("PCB_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paracut_b200 as pc
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance
from bench import pinned_instance

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = pinned_instance(make_instance(CONFIGS[wl], seed=0))
thr = np.array([0.0])
for rep in range(3):
    t = [time.perf_counter()]
    S = _native.GridSolver(g, precision="f32"); S.synchronize(); t.append(time.perf_counter())
    S.init_cold(); S.synchronize(); t.append(time.perf_counter())
    S.shadow(); S.synchronize(); t.append(time.perf_counter())
    S.check(thr); S.check_labels(0, packed=True); S.keep_best(0); S.synchronize(); t.append(time.perf_counter())
    S.apply(); S.synchronize(); t.append(time.perf_counter())
    S.run(K - 1, norms=True); S.synchronize(); t.append(time.perf_counter())
    S.shadow(); S.synchronize(); t.append(time.perf_counter())
    S.check(thr); S.check_labels(0, packed=True); S.keep_best(0); S.synchronize(); t.append(time.perf_counter())
    lab, x = S.get_best(labels=True, x=False); t.append(time.perf_counter())
    S.close(); del S; t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print("create %.2f init %.2f shadow0 %.2f check0 %.2f apply %.2f run %.2f shadowK %.2f checkK %.2f "
          "labels %.2f close %.2f  total %.2f ms" % (tuple(d) + (sum(d),)), flush=True)
os.environ["PCB_TRACE"] = "0"
cfg = pc.SolverConfig(max_iters=K, check_every=K + 1, precision="f32")
for rep in range(4):
    t0 = time.perf_counter()
    res = pc.solve(g, pc.decompose_grid(g), cfg)
    _ = np.count_nonzero(res.labeling)
    t1 = time.perf_counter()
    res = None
    print("solve total %.2f ms" % ((t1 - t0) * 1e3), flush=True)
S = _native.GridSolver(g, precision="f32")
for rep in range(2):
    S.init_cold(); S.synchronize()
    ts = []
    for k in range(K):
        t0 = time.perf_counter(); S.run(1, norms=False); S.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    print("per-iteration ms from cold:", " ".join("%.2f" % v for v in ts), flush=True)
    S.init_cold(); S.synchronize()
    t0 = time.perf_counter(); S.run(K, norms=False); S.synchronize()
    print("run(%d) from cold: %.2f ms" % (K, (time.perf_counter() - t0) * 1e3), flush=True)
