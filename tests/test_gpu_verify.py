"""Verified sweeps of the fp32 step: last iteration's
segmentation as a candidate, a complete KKT check, local repair with a taut
string between true points.  The results must stay within the north_star fp32
tolerance of the reference (the C oracle) whatever the hints are -- including
when the verified sweep is forced on from the first iterations (garbage hints,
nearly every chain repaired) -- and the path must actually run."""
import numpy as np
import pytest

from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance

pytestmark = pytest.mark.gpu


def _rel(x, ref):
    return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300))


def _run(g, k):
    S = _native.GridSolver(g, precision="f32")
    S.init_cold()
    S.run(k)
    y, _ = S.shadow(want_y=True)
    return S, g.w - y.sum(axis=0)


# (row lengths that are not multiples of 4: such rows have no TMA row map and
# keep the cp.async sweep, the case the verified sweep serves)
@pytest.mark.parametrize("dims,k", [((16, 40, 50), 200), ((24, 32, 54), 160)])
def test_verified_sweeps_match_oracle(dims, k, capsys):
    from oracle import oracle as orc
    g = make_instance(CONFIGS["cfg4"], seed=2, dims=dims)
    _, y_ref, _ = orc.aar(g, k, threads=orc.max_threads())
    x_ref = g.w - y_ref.sum(axis=0)
    S, x = _run(g, k)
    modes, sweeps, rep = S.verify_stats()
    with capsys.disabled():
        print("\n[verify] dims %s k=%d: verified sweeps %s, repaired chains %s, rel %.2e"
              % (dims, k, list(sweeps), list(rep), _rel(x, x_ref)))
    assert _rel(x, x_ref) <= 1e-4
    assert sweeps.sum() > 0  # the verified sweep ran


def test_forced_verification_with_stale_hints_is_exact(monkeypatch):
    """theta > 100 %: the verified family stays verified from its first probe
    (iteration ~65) on, when the hints are still far from the solution --
    many chains go through the repair, and the result still matches the
    oracle."""
    from oracle import oracle as orc
    monkeypatch.setenv("PCB_VERIFY_THETA", "1000")
    monkeypatch.setenv("PCB_ROW_TMA", "0")  # rows on cp.async: the verified family
    g = make_instance(CONFIGS["cfg4"], seed=3, dims=(12, 20, 36))
    k = 120
    _, y_ref, _ = orc.aar(g, k, threads=orc.max_threads())
    x_ref = g.w - y_ref.sum(axis=0)
    S, x = _run(g, k)
    modes, sweeps, rep = S.verify_stats()
    assert sweeps.sum() >= k - 70
    assert rep.sum() > 0
    assert _rel(x, x_ref) <= 1e-4


def test_verified_and_scan_steps_agree(monkeypatch):
    g = make_instance(CONFIGS["cfg4"], seed=4, dims=(20, 32, 62))
    k = 150
    S, x_v = _run(g, k)
    assert S.verify_stats()[1].sum() > 0
    monkeypatch.setenv("PCB_VERIFY", "0")
    _, x_s = _run(g, k)
    assert _rel(x_v, x_s) <= 2e-5
