"""Parity at BASELINE.json's full sizes and iteration counts against the C
oracle (oracle/paracut_oracle.c, the reference loop solvers.py:272-307 in the
reference's own operation order, OpenMP over chains on every host core).

Metric: x = w - sum_j y_j, relative error
max|x - x_ref| / max|x_ref|; tolerances (north_star): 1e-6 for fp64 (the
exact mode is in fact bitwise), 1e-4 for the fp32-state mode.  The errors are
printed so the GPU test log records them.

* cfg2 2D-4 1024^2, 500 iterations: f64 and f32;
* cfg4 3D-6 256^3, 500 iterations: f32 (the benchmarked path) and f64;
* cfg2 and cfg4 in the fast fp64 mode (f64s: split chains, fp64 state and
  scans -- the polish of a time-to-cut solve), 1e-6;
* cfg3 2D-8 4096^2, 1000 iterations: f32;
* cfg2_int 1024^2: the device certificate (pcb_check: labels, cut energy,
  gap, smooth dual at thresholds 0 and +-1e-6) of the oracle's own iterate
  at k = 500 against the oracle's certificate (certify.py:31-47).
"""
import numpy as np
import pytest

import paracut_b200 as pc
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance

pytestmark = pytest.mark.gpu


def _rel(x, ref):
    return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300))


def _report(capsys, msg):
    with capsys.disabled():
        print("\n[parity] " + msg, flush=True)


def _oracle(name, k):
    from oracle import oracle as orc
    g = make_instance(CONFIGS[name], seed=0)
    run = orc.AARRunner(g, threads=orc.max_threads())
    run.run(k, final_shadow=True)
    return g, run.z, run.p


def _device(g, k, precision):
    res = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(max_iters=k, check_every=k + 1, precision=precision))
    assert res.iterations == k
    return res.dual_state


@pytest.fixture(scope="module")
def cfg2_ref():
    return _oracle("cfg2", 500)


@pytest.fixture(scope="module")
def cfg4_ref():
    return _oracle("cfg4", 500)


def test_cfg2_full_f64_and_f32(cfg2_ref, capsys):
    g, z_ref, y_ref = cfg2_ref
    x_ref = g.w - y_ref.sum(axis=0)
    st = _device(g, 500, "f64")
    e64 = _rel(g.w - st.y.sum(axis=0), x_ref)
    bitwise = bool(np.array_equal(st.z, z_ref) and np.array_equal(st.y, y_ref))
    del st
    st = _device(g, 500, "f32")
    e32 = _rel(g.w - st.y.sum(axis=0), x_ref)
    _report(capsys, "cfg2 1024^2 k=500: f64 rel %.3e (bitwise %s), f32 rel %.3e" % (e64, bitwise, e32))
    assert e64 <= 1e-6
    assert e32 <= 1e-4


def test_cfg4_full_f32_and_f64(cfg4_ref, capsys):
    g, z_ref, y_ref = cfg4_ref
    x_ref = g.w - y_ref.sum(axis=0)
    st = _device(g, 500, "f32")
    e32 = _rel(g.w - st.y.sum(axis=0), x_ref)
    del st
    st = _device(g, 500, "f64")
    e64 = _rel(g.w - st.y.sum(axis=0), x_ref)
    bitwise = bool(np.array_equal(st.z, z_ref) and np.array_equal(st.y, y_ref))
    _report(capsys, "cfg4 256^3 k=500: f32 rel %.3e, f64 rel %.3e (bitwise %s)" % (e32, e64, bitwise))
    assert e32 <= 1e-4
    assert e64 <= 1e-6


@pytest.mark.parametrize("name", ["cfg2", "cfg4"])
def test_full_f64s(name, cfg2_ref, cfg4_ref, capsys):
    g, _, y_ref = cfg2_ref if name == "cfg2" else cfg4_ref
    x_ref = g.w - y_ref.sum(axis=0)
    st = _device(g, 500, "f64s")
    e = _rel(g.w - st.y.sum(axis=0), x_ref)
    _report(capsys, "%s k=500: f64s rel %.3e" % (name, e))
    assert e <= 1e-6


def test_cfg3_full_f32(capsys):
    g, _, y_ref = _oracle("cfg3", 1000)
    x_ref = g.w - y_ref.sum(axis=0)
    del y_ref
    st = _device(g, 1000, "f32")
    e32 = _rel(g.w - st.y.sum(axis=0), x_ref)
    _report(capsys, "cfg3 4096^2 2D-8 k=1000: f32 rel %.3e" % e32)
    assert e32 <= 1e-4


def test_cfg2_int_full_certificate_vs_oracle(capsys):
    from oracle import oracle as orc
    g, z_ref, y_ref = _oracle("cfg2_int", 500)
    s = y_ref.sum(axis=0)
    thr = np.array([0.0, 1e-6, -1e-6])
    S = _native.GridSolver(g, precision="f64")
    S.set_z(z_ref)
    S.shadow()
    e_dev, gap_dev, smooth_dev = S.check(thr)
    worst = 0.0
    for t, th in enumerate(thr):
        lab, gap, energy, smooth = orc.check(g, s, th)
        assert np.array_equal(S.check_labels(t), lab)
        assert e_dev[t] == energy  # integer capacities: exact sums
        assert abs(gap_dev[t] - gap) <= 1e-9 * max(1.0, abs(energy))
        worst = max(worst, abs(gap_dev[t] - gap))
    assert abs(smooth_dev - smooth) <= 1e-9 * abs(smooth)
    _report(capsys, "cfg2_int 1024^2 k=500 certificate: energies %s, gaps %s, max |dgap| %.2e"
            % (list(e_dev), list(gap_dev), worst))
