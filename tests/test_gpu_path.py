"""Lambda path on a resident instance (solve_path / pcb_scale_pairwise) vs the
reference's scaled_pairwise + force_warm warm starts (tests/golden/path_*)."""
import numpy as np
import pytest

import paracut_b200 as pc
from conftest import golden_grid

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["path_r3d6.npz", "path_i2d4.npz"])
def test_path_matches_reference_bitwise(name):
    g, d = golden_grid(name)
    g = pc.GridEnergy(g.dims, g.connectivity, g.w, g.dir_weights)
    lams = list(d["lambdas"])
    cfg = pc.SolverConfig(gap_tol=1e-6, max_iters=400, check_every=10)
    res = pc.solve_path(g, lams, cfg)
    for i, r in enumerate(res):
        assert r.iterations == int(d["iters_%d" % i]), i
        assert r.certified == bool(d["certified_%d" % i])
        assert r.energy == pytest.approx(float(d["energy_%d" % i]), abs=1e-9)
        assert r.gap == pytest.approx(float(d["gap_%d" % i]), rel=1e-9, abs=1e-9)
        assert np.array_equal(r.labeling, d["labeling_%d" % i])
        assert np.array_equal(r.dual_state.y, d["y_%d" % i]), i
        assert np.array_equal(r.dual_state.z, d["z_%d" % i]), i
        assert r.dual_state.fingerprint == str(d["fp_%d" % i])


def test_path_equals_explicit_warm_starts_and_f32_runs():
    g, d = golden_grid("path_r3d6.npz")
    g = pc.GridEnergy(g.dims, g.connectivity, g.w, g.dir_weights)
    cfg = pc.SolverConfig(gap_tol=1e-6, max_iters=300, check_every=10)
    lams = [0.5, 1.5]
    a = pc.solve_path(g, lams, cfg, keep_states=False)
    assert a[0].dual_state is None and a[1].dual_state is not None
    prev = None
    for i, lam in enumerate(lams):
        gl = g.scaled_pairwise(lam)
        prev = pc.solve(gl, pc.decompose_grid(gl),
                        pc.SolverConfig(gap_tol=1e-6, max_iters=300, check_every=10,
                                        warm_start=prev.dual_state if prev else None,
                                        force_warm=True))
        assert prev.iterations == a[i].iterations and np.array_equal(prev.labeling, a[i].labeling)
    assert np.array_equal(prev.dual_state.z, a[-1].dual_state.z)
    f = pc.solve_path(g, lams, pc.SolverConfig(gap_tol=1e-6, max_iters=300, check_every=10,
                                               precision="f32", polish_iters=100))
    assert all(r.certified for r in f)
    with pytest.raises(ValueError):
        pc.solve_path(g, [-1.0], cfg)
