"""fp64 device path vs the reference: bitwise at matched iterations.

The golden fixtures come from running the reference itself; the oracle is
pinned to them bitwise (test_oracle_golden.py), so equality here is equality
with the reference's numba/numpy arithmetic."""
import numpy as np
import pytest

import paracut_b200 as pc
from paracut_b200 import _native
from conftest import aar_cases, golden_grid, load_golden

pytestmark = pytest.mark.gpu


def test_tv1d_bitwise_vs_reference():
    d = load_golden("tv1d.npz")
    s, a, ptr, x = d["s"], d["a"], d["ptr"], d["x"]
    got = _native.tv1d_batch(s, a, ptr)
    assert np.array_equal(got, x)
    # public single-chain entry on a few chains, including the m=1 and long ones
    for c in (0, 1, ptr.size - 2, ptr.size - 5, ptr.size - 6):
        b, e = ptr[c], ptr[c + 1]
        assert np.array_equal(pc.tv1d_prox(s[b:e], a[b - c:e - c - 1]), x[b:e])


def test_tv1d_closed_forms_and_validation():
    s = np.array([1.0, -1.0])
    assert pc.tv1d_prox(s, np.array([1.0])).tolist() == [0.0, 0.0]
    assert pc.tv1d_prox(s, np.array([0.25])).tolist() == [0.75, -0.75]
    assert pc.tv1d_prox(s, np.array([0.0])).tolist() == [1.0, -1.0]
    rng = np.random.default_rng(1)
    sig = rng.normal(size=40)
    assert np.array_equal(pc.tv1d_prox(sig, np.zeros(39)), sig)
    const = np.full(25, -0.3)
    assert np.array_equal(pc.tv1d_prox(const, rng.uniform(0, 2, 24)), const)
    assert pc.tv1d_prox(np.array([4.2]), np.zeros(0)).tolist() == [4.2]
    with pytest.raises(ValueError):
        pc.tv1d_prox(np.zeros(0), np.zeros(0))
    with pytest.raises(ValueError):
        pc.tv1d_prox(np.zeros(3), np.zeros(3))
    with pytest.raises(ValueError):
        pc.tv1d_prox(np.zeros(3), np.array([1.0, -0.5]))


def test_deep_hull_spill_path():
    # convex prefix sums with huge weights drive hull depth far past the
    # shared-memory capacity; the global spill region must keep it exact
    from oracle import oracle as orc
    m = 3000
    i = np.arange(m, dtype=np.float64)
    s = (i - m / 2) ** 2 / m
    a = np.full(m - 1, 1e4)
    assert np.array_equal(pc.tv1d_prox(s, a), orc.tv1d_prox(s, a))
    s2 = np.sin(i / 7.0) * 50 + np.cos(i / 3.0)
    a2 = np.abs(np.sin(i[:-1])) * 30
    assert np.array_equal(pc.tv1d_prox(s2, a2), orc.tv1d_prox(s2, a2))


@pytest.mark.parametrize("name", aar_cases() + ["cfg1.npz"])
def test_aar_fixed_iterations_bitwise(name):
    g, d = golden_grid(name)
    for k in d["ks"]:
        k = int(k)
        res = pc.solve(g, pc.decompose_grid(g),
                       pc.SolverConfig(max_iters=k, check_every=k + 1, precision="f64"))
        assert res.iterations == int(d["iters_%d" % k])
        st = res.dual_state
        assert np.array_equal(st.z, d["z_%d" % k]), (name, k)
        assert np.array_equal(st.y, d["y_%d" % k]), (name, k)
        ref = d["norms_%d" % k]
        got = np.asarray(res.monitor.get("aar_step_norm", []))
        assert got.size == ref.size
        if ref.size:
            assert np.allclose(got, ref, rtol=1e-12, atol=1e-12)
        row = res.trace[-1]
        assert row.gap == pytest.approx(float(d["gap_%d" % k]), rel=1e-10, abs=1e-9)
        assert row.energy == pytest.approx(float(d["energy_%d" % k]), rel=1e-10, abs=1e-9)
        assert row.dual_objective == pytest.approx(float(d["dual_%d" % k]), rel=1e-10, abs=1e-9)


@pytest.mark.parametrize("name", aar_cases())
def test_prox_chains_csr_bitwise(name):
    # the operator-level drop-in for _kernels.prox_chains on the reference CSR classes
    from oracle import oracle as orc
    g, d = golden_grid(name)
    rng = np.random.default_rng(3)
    for cls in orc.decompose(g):
        if cls.num_chains == 0:
            continue
        v = rng.normal(0, 3, size=g.n)
        for proj in (True, False):
            want = np.zeros(g.n)
            orc.prox_chains(cls, v, want, proj)
            got = np.zeros(g.n)
            _native.prox_chains(cls.node_idx, cls.chain_ptr, cls.edge_w, 0, cls.num_chains,
                                v, got, proj)
            assert np.array_equal(got, want)


@pytest.mark.parametrize("name", ["aar_r2d4.npz", "aar_r2d8.npz", "aar_r3d6.npz",
                                  "aar_i2d8.npz", "aar_deg1.npz"])
def test_project_K_grid_bitwise(name):
    from oracle import oracle as orc
    g, d = golden_grid(name)
    gg = pc.GridEnergy(g.dims, g.connectivity, g.w, g.dir_weights)
    dec = pc.decompose_grid(gg)
    rng = np.random.default_rng(4)
    v = rng.normal(0, 2, size=(dec.r, g.n))
    assert np.array_equal(pc.project_K(dec, v), orc.project_K(orc.decompose(g), v))


def test_project_L_examples():
    c1 = pc.ChainClass(2, np.array([0, 1]), np.array([0, 2]), np.array([1.0]))
    c2 = pc.ChainClass(2, np.array([0, 1]), np.array([0, 2]), np.array([1.0]))
    dec = pc.ChainDecomposition(2, [c1, c2])
    lam = pc.project_L(np.array([2.0, 2.0]), dec, np.array([[1.0, 1.0], [0.0, 0.0]]))
    assert np.allclose(lam, [[1.5, 1.5], [0.5, 0.5]])
    cls = pc.ChainClass(3, np.array([1, 2]), np.array([0, 2]), np.array([1.0]))
    dec = pc.ChainDecomposition(3, [cls])
    with pytest.raises(ValueError, match="covered by no class"):
        pc.project_L(np.array([3.0, 0.5, -0.5]), dec, np.zeros((1, 3)))
    lam = pc.project_L(np.array([0.0, 0.5, -0.5]), dec, np.zeros((1, 3)))
    assert np.allclose(lam, [[0.0, 0.5, -0.5]])
