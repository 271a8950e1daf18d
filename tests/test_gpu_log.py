"""Solve log (pcb_log_*): step norms and check labelings kept on the device
until the solve ends give the same monitor and trace (jaccard column
included) as per-check host copies."""
import numpy as np
import pytest

import paracut_b200 as pc
from paracut_b200 import solvers
from paracut_b200.instances import CONFIGS, make_instance

pytestmark = pytest.mark.gpu


def _solve(g, cfg, log, monkeypatch):
    if not log:
        monkeypatch.setattr(solvers._Driver, "start_log", lambda self: None)
    else:
        monkeypatch.undo()
    return pc.solve(g, pc.decompose_grid(g), cfg)


@pytest.mark.parametrize("precision,polish", [("f64", 0), ("f32", 0), ("f32", 200)])
def test_log_matches_host_copies(monkeypatch, precision, polish):
    g = make_instance(CONFIGS["cfg2_int"], seed=3, dims=(96, 80))
    cfg = pc.SolverConfig(max_iters=400, check_every=10, precision=precision,
                          thresholds=(0.0, 1e-6, -1e-6), polish_iters=polish,
                          polish_stall=3 if polish else 0)
    a = _solve(g, cfg, False, monkeypatch)
    b = _solve(g, cfg, True, monkeypatch)
    assert a.iterations == b.iterations
    assert np.array_equal(a.labeling, b.labeling)
    assert np.array_equal(a.tv_solution, b.tv_solution)
    assert a.monitor.keys() == b.monitor.keys()
    for key in a.monitor:
        assert np.array_equal(np.asarray(a.monitor[key]), np.asarray(b.monitor[key])), key
    assert len(a.trace) == len(b.trace)
    for ra, rb in zip(a.trace, b.trace):
        assert (ra.iteration, ra.gap, ra.dual_objective, ra.energy) == \
               (rb.iteration, rb.gap, rb.dual_objective, rb.energy)
        assert ra.jaccard == rb.jaccard


def test_log_api_roundtrip():
    from paracut_b200 import _native
    g = make_instance(CONFIGS["cfg2_int"], seed=4, dims=(33, 47))
    S = _native.GridSolver(g, precision="f32")
    S.init_cold()
    S.log_start()
    S.run(5, norms=False)
    S.shadow()
    e, gp, _ = S.check(np.array([0.0, 1e-3]))
    s0 = S.log_labels(0)
    s1 = S.log_labels(1)
    S.apply(norm=False)
    norms = S.log_norms()
    assert norms.shape == (6,) and np.all(np.isfinite(norms))
    p0 = S.check_labels(0, packed=True)
    p1 = S.check_labels(1, packed=True)
    assert np.array_equal(S.log_label_get(s0), p0)
    assert np.array_equal(S.log_label_get(s1), p1)
    jac = S.log_jaccard(p0, 2)
    assert jac[0] == 0.0
    from paracut_b200.certify import jaccard_packed
    assert jac[1] == jaccard_packed(p1, p0)
