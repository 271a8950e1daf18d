"""Driver semantics of solve()/solve_aar on the device vs the reference."""
import numpy as np
import pytest

import paracut_b200 as pc
from conftest import golden_grid

pytestmark = pytest.mark.gpu


def _grid(g):
    return pc.GridEnergy(g.dims, g.connectivity, g.w, g.dir_weights)


@pytest.mark.parametrize("name", ["solve_2d4.npz", "solve_2d8.npz", "solve_3d6.npz"])
def test_gap_stopped_solve_matches_reference(name):
    g, d = golden_grid(name)
    g = _grid(g)
    res = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(gap_tol=1e-6, max_iters=20000, check_every=5))
    assert res.iterations == int(d["iterations"])
    assert res.certified == bool(d["certified"])
    assert np.array_equal(res.labeling, d["labeling"])
    assert np.array_equal(res.tv_solution, d["tv_solution"])
    assert res.energy == pytest.approx(float(d["energy"]), abs=1e-9)
    assert [r.iteration for r in res.trace] == list(d["trace_iter"])
    assert np.allclose([r.gap for r in res.trace], d["trace_gap"], rtol=1e-9, atol=1e-9)
    assert np.allclose([r.jaccard for r in res.trace], d["trace_jac"], atol=0)
    assert np.array_equal(res.dual_state.z, d["z"])
    assert np.array_equal(res.dual_state.y, d["y"])


def test_frozen_kat_energy():
    g, d = golden_grid("kat.npz")
    g = _grid(g)
    res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(gap_tol=1e-6, check_every=1))
    assert res.certified
    assert res.energy == pytest.approx(-1.7192866314283624, abs=1e-9)
    assert np.array_equal(res.labeling, d["labeling"])


def test_eps_thresholds_reach_maxflow_optimum():
    g, d = golden_grid("eps_int.npz")
    g = _grid(g)
    res = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(max_iters=400, check_every=401,
                                   thresholds=(0.0, 1e-6, -1e-6)))
    assert res.certified
    assert res.energy == float(d["maxflow"])
    assert g.energy(res.labeling) == float(d["maxflow"])


def test_edge_free_and_isolated():
    g = pc.GridEnergy((2, 2), "2D-4", np.array([1.0, -1.0, 0.0, 2.0]),
                      [np.zeros((2, 1)), np.zeros((1, 2))])
    res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(check_every=5))
    assert res.certified and res.iterations == 0
    assert res.labeling.tolist() == [1, 0, 0, 1]
    row = np.array([[0.0, 1.0, 0.5]])
    g = pc.GridEnergy((1, 4), "2D-4", np.array([3.0, -1.0, 0.25, -0.5]),
                      [row, np.zeros((0, 4))])
    res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(check_every=5))
    assert res.certified and res.labeling[0] == 1


def test_monitor_monotone_and_trace_semantics():
    rng = np.random.default_rng(0)
    g = pc.GridEnergy((16, 16), "2D-8", rng.uniform(-2, 2, 256),
                      [rng.uniform(0, 2, s) for s in ((16, 15), (15, 16), (15, 15), (15, 15))])
    for prec in ("f64", "f32"):
        res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(check_every=5, precision=prec))
        dn = np.diff(res.monitor["aar_step_norm"])
        assert dn.size and np.all(dn <= 1e-6 if prec == "f32" else dn <= 1e-9)
        assert res.trace[-1].jaccard == 0.0
        assert all(0.0 <= r.jaccard <= 1.0 for r in res.trace)
        assert g.energy(res.labeling) == pytest.approx(res.energy, abs=1e-9)
        assert np.array_equal(pc.threshold(res.tv_solution - res.threshold), res.labeling)


def test_warm_start_fingerprint_and_shape():
    rng = np.random.default_rng(7)

    def rg():
        return pc.GridEnergy((12, 12), "2D-4", rng.uniform(-2, 2, 144),
                             [rng.uniform(0, 2, (12, 11)), rng.uniform(0, 2, (11, 12))])
    g = rg()
    res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(check_every=5))
    st = res.dual_state
    assert st.fingerprint is not None and st.z is not None
    other = rg()
    with pytest.raises(ValueError, match="fingerprint"):
        pc.solve(other, pc.decompose_grid(other), pc.SolverConfig(warm_start=st))
    forced = pc.solve(other, pc.decompose_grid(other),
                      pc.SolverConfig(warm_start=st, force_warm=True))
    assert forced.certified
    bad = st.copy()
    bad.z = np.zeros((1, 5))
    with pytest.raises(ValueError, match="shape"):
        pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(warm_start=bad, force_warm=True))
    again = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(warm_start=st, check_every=5))
    assert again.iterations <= res.iterations


def test_dual_tol_stops():
    rng = np.random.default_rng(6)
    g = pc.GridEnergy((16, 16), "2D-4", rng.uniform(-2, 2, 256),
                      [rng.uniform(0, 2, (16, 15)), rng.uniform(0, 2, (15, 16))])
    res = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(dual_tol=1e-7, check_every=10 ** 9))
    assert res.iterations < 20000
    assert res.certified


def test_config_validation_and_other_algorithms():
    with pytest.raises(ValueError, match="algorithm"):
        pc.SolverConfig(algorithm="newton")
    with pytest.raises(ValueError, match="max_iters"):
        pc.SolverConfig(max_iters=0)
    with pytest.raises(ValueError, match="tolerances"):
        pc.SolverConfig(gap_tol=-1e-3)
    with pytest.raises(ValueError, match=">= 1"):
        pc.SolverConfig(threads=0)
    g = pc.GridEnergy((3, 3), "2D-4", np.zeros(9), [np.ones((3, 2)), np.ones((2, 3))])
    # w = 0: every scheme certifies the empty labeling at k = 0
    for alg in ("bcd", "ap", "aar", "fista"):
        res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(algorithm=alg))
        assert res.certified and res.iterations == 0 and res.energy == 0.0
