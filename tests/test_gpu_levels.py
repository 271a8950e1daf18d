"""Best level set on the device (pcb_level_set) vs the reference's
best_level_set_gap (certify.py:50-65) and the oracle restatement."""
import numpy as np
import pytest

import paracut_b200 as pc
from paracut_b200 import _native
from paracut_b200.instances import energy_from_image, make_instance, synth_image
from conftest import golden_grid, level_cases

pytestmark = pytest.mark.gpu


def _grid(g):
    return pc.GridEnergy(g.dims, g.connectivity, g.w, g.dir_weights)


@pytest.mark.parametrize("name", level_cases())
def test_level_set_matches_reference(name):
    g, d = golden_grid(name)
    g = _grid(g)
    S = _native.GridSolver(g, precision="f64")
    u, e = S.level_set(d["x"])
    lab = (d["x"] > u).astype(np.uint8)
    assert np.array_equal(lab, d["labeling"]), name
    assert e == pytest.approx(float(d["energy"]), rel=1e-12, abs=1e-12)
    # public API: same labeling, reference certificate formulas
    lab2, cert = pc.best_level_set_gap(g, d["x"], d["s"])
    assert np.array_equal(lab2, d["labeling"])
    assert cert.gap == pytest.approx(float(d["gap"]), rel=1e-12, abs=1e-12)
    if str(d["conn"]) in ("2D-4", "3D-6") and name.startswith("levels_i"):
        assert e == float(d["energy"])  # integer weights: exact


def test_level_set_never_worse_than_threshold(oracle_lib):
    # reference test_certify.py:69-79, on partially solved random grids
    rng = np.random.default_rng(4)
    for trial in range(12):
        conn = ("2D-4", "2D-8", "3D-6")[trial % 3]
        dims = (int(rng.integers(3, 9)), int(rng.integers(3, 9)))
        if conn == "3D-6":
            dims = dims + (int(rng.integers(2, 5)),)
        shape_src = energy_from_image(rng.normal(size=dims), conn)
        g = pc.GridEnergy(dims, conn, rng.normal(size=int(np.prod(dims))),
                          [rng.uniform(0, 1, size=a.shape) * (rng.uniform(size=a.shape) < 0.8)
                           for a in shape_src.dir_weights])
        res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=int(rng.integers(1, 6)),
                                                                check_every=100))
        s = res.dual_state.y.sum(axis=0)
        x = g.w - s
        lab, cert = pc.best_level_set_gap(g, x, s)
        base = pc.discrete_gap(g, pc.threshold(x), s).gap
        assert cert.gap <= base + 1e-12
        assert set(np.unique(lab)) <= {0, 1}
        olab, ogap, _ = oracle_lib.best_level_set(g, x, s)
        assert cert.gap == pytest.approx(ogap, rel=1e-9, abs=1e-9)


def test_level_set_degenerate_values():
    g = make_instance("cfg1", seed=0, dims=(8, 9))
    S = _native.GridSolver(g, precision="f64")
    # a constant x: two level sets (all ones, empty)
    u, e = S.level_set(np.full(g.n, 0.25))
    lab = (np.full(g.n, 0.25) > u)
    e_all, e_none = -float(g.w.sum()), 0.0
    assert e == pytest.approx(min(e_all, e_none))
    assert lab.all() == (e_all < e_none)
    # signed zeros are one value (np.unique), NaN-free ties resolve to the first level
    x = np.zeros(g.n)
    x[::2] = -0.0
    u2, e2 = S.level_set(x)
    assert e2 == pytest.approx(e)


def test_solver_level_sets_certify_integer_plateaus():
    # integer instance: thresholding x at 0 can miss the optimum on exact-zero
    # plateaus; the level-set candidate at every check never does worse
    img = synth_image((96, 80), 6, 5, 20, seed=3)
    g = energy_from_image(img, "2D-4", integer=True)
    base = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=300, check_every=20))
    lv = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=300, check_every=20,
                                                            level_sets=True))
    for a, b in zip(base.trace, lv.trace):
        assert b.gap <= a.gap + 1e-12
    assert lv.gap <= base.gap
    assert lv.energy == float(round(lv.energy))


def test_level_set_full_size_scan_energy_is_exact_on_integers():
    # cfg2_int at full size: the one-sort scan energy of the chosen level set
    # equals the deterministic pcb_check energy of that labeling exactly
    g = make_instance("cfg2_int", seed=0)
    S = _native.GridSolver(g, precision="f32")
    S.init_cold()
    S.run(60, norms=False)
    S.shadow()
    S.check(np.array([0.0]))
    u, e = S.level_set()
    energies, gaps, _ = S.check(np.array([0.0, u]))
    assert e == energies[1]
    assert gaps[1] <= gaps[0]
