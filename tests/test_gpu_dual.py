"""BCD / AP / FISTA on the device (pcb_dual_init / pcb_dual_run) vs the
reference's solve_bcd / solve_ap / solve_fista (solvers.py:212-269, 310-341):
iterates bitwise, monitors and certificates to rounding."""
import numpy as np
import pytest

import paracut_b200 as pc
from paracut_b200 import _native
from conftest import dual_cases, golden_grid

pytestmark = pytest.mark.gpu

MON = {"bcd": "dual_objective", "ap": "ap_distance", "fista": "dual_objective"}


def _grid(g):
    return pc.GridEnergy(g.dims, g.connectivity, g.w, g.dir_weights)


@pytest.mark.parametrize("name", dual_cases())
def test_fixed_iterations_bitwise(name):
    alg = name.split("_")[1]
    g, d = golden_grid(name)
    g = _grid(g)
    dec = pc.decompose_grid(g)
    for k in d["ks"]:
        k = int(k)
        res = pc.solve(g, dec, pc.SolverConfig(algorithm=alg, max_iters=k, check_every=k + 1))
        assert res.iterations == k
        assert np.array_equal(res.dual_state.y, d["y_%d" % k]), (name, k)
        if "lam_%d" % k in d:
            assert np.array_equal(res.dual_state.lam, d["lam_%d" % k]), (name, k)
        assert np.allclose(res.monitor[MON[alg]], d["mon_%d" % k], rtol=1e-10, atol=1e-10)
        assert res.trace[-1].gap == pytest.approx(float(d["gap_%d" % k]), rel=1e-9, abs=1e-9)


@pytest.mark.parametrize("name", dual_cases())
def test_gap_stopped_solve_matches_reference(name):
    alg = name.split("_")[1]
    g, d = golden_grid(name)
    g = _grid(g)
    res = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(algorithm=alg, gap_tol=1e-6, max_iters=600, check_every=7))
    assert res.iterations == int(d["s_iterations"])
    assert res.certified == bool(d["s_certified"])
    assert np.array_equal(res.labeling, d["s_labeling"])
    assert np.array_equal(res.tv_solution, d["s_tv"])
    assert np.array_equal(res.dual_state.y, d["s_y"])
    assert res.energy == pytest.approx(float(d["s_energy"]), abs=1e-9)
    assert [r.iteration for r in res.trace] == list(d["s_trace_iter"])
    assert np.allclose([r.gap for r in res.trace], d["s_trace_gap"], rtol=1e-9, atol=1e-9)
    assert np.allclose([r.dual_objective for r in res.trace], d["s_trace_dual"],
                       rtol=1e-12, atol=1e-9)
    assert res.algorithm == alg
    assert res.dual_state.fingerprint == pc.instance_fingerprint(g)


@pytest.mark.parametrize("name", dual_cases())
def test_dual_tol_stop_matches_reference(name):
    alg = name.split("_")[1]
    g, d = golden_grid(name)
    g = _grid(g)
    res = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(algorithm=alg, dual_tol=1e-3, max_iters=400, check_every=50))
    assert res.iterations == int(d["t_iterations"])
    assert [r.iteration for r in res.trace] == list(d["t_trace_iter"])
    assert np.array_equal(res.dual_state.y, d["t_y"])


@pytest.mark.parametrize("alg", ["bcd", "ap", "fista"])
def test_warm_start_continues_bitwise(alg):
    g, d = golden_grid("dual_%s_r2d4.npz" % alg)
    g = _grid(g)
    dec = pc.decompose_grid(g)
    a = pc.solve(g, dec, pc.SolverConfig(algorithm=alg, max_iters=1, check_every=100))
    if alg == "fista":
        # FISTA restarts its momentum from a warm y: compare against a fresh
        # device run started from the same y
        S = _native.GridSolver(g, precision="f64")
        S.dual_init(_native.ALG_FISTA, a.dual_state.y)
        S.dual_run(5)
        b = pc.solve(g, dec, pc.SolverConfig(algorithm=alg, max_iters=5, check_every=100,
                                             warm_start=a.dual_state))
        assert np.array_equal(b.dual_state.y, S.shadow_get())
        return
    b = pc.solve(g, dec, pc.SolverConfig(algorithm=alg, max_iters=5, check_every=100,
                                         warm_start=a.dual_state))
    assert np.array_equal(b.dual_state.y, d["y_6"])


def test_dual_schemes_need_fp64_and_block_aar_calls():
    g, _ = golden_grid("dual_bcd_r2d4.npz")
    g = _grid(g)
    with pytest.raises(ValueError):
        pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(algorithm="bcd", precision="f32"))
    S = _native.GridSolver(g, precision="f64")
    S.dual_init(_native.ALG_AP)
    with pytest.raises(RuntimeError):
        S.run(1)
    with pytest.raises(ValueError):
        S.dual_init(7)
