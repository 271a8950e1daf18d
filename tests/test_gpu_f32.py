"""fp32-state fast path: TV solution within 1e-4 relative of the reference
at matched iterations (north_star tolerance), and bitwise-exact f64 device
runs at BASELINE scale checked against the C oracle."""
import numpy as np
import pytest

import paracut_b200 as pc
from paracut_b200.instances import CONFIGS, make_instance
from conftest import golden_grid

pytestmark = pytest.mark.gpu


def _rel(x, ref):
    return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300))


def test_cfg1_f32_within_tolerance():
    g, d = golden_grid("cfg1.npz")
    g = pc.GridEnergy(g.dims, g.connectivity, g.w, g.dir_weights)
    res = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(max_iters=200, check_every=201, precision="f32"))
    x_ref = g.w - d["y_200"].sum(axis=0)
    x = g.w - res.dual_state.y.sum(axis=0)
    assert _rel(x, x_ref) <= 1e-4
    assert _rel(res.dual_state.z, d["z_200"]) <= 1e-4


@pytest.mark.parametrize("conn,dims,k", [("2D-8", (96, 80), 150), ("3D-6", (24, 20, 28), 150),
                                         ("2D-4", (128, 128), 300)])
def test_f32_vs_oracle(conn, dims, k):
    from oracle import oracle as orc
    spec = {"2D-4": CONFIGS["cfg2"], "2D-8": CONFIGS["cfg3"], "3D-6": CONFIGS["cfg4"]}[conn]
    g = make_instance(spec, seed=5, dims=dims)
    z_ref, y_ref, _ = orc.aar(g, k, threads=8)
    x_ref = g.w - y_ref.sum(axis=0)
    res = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(max_iters=k, check_every=k + 1, precision="f32"))
    x = g.w - res.dual_state.y.sum(axis=0)
    assert _rel(x, x_ref) <= 1e-4


def test_integer_variant_f32_exact_energy():
    # integer capacities: the eps-threshold rule certifies and hits the optimum
    g, d = golden_grid("eps_int.npz")
    g = pc.GridEnergy(g.dims, g.connectivity, g.w, g.dir_weights)
    res = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(max_iters=400, check_every=401, precision="f32",
                                   thresholds=(0.0, 1e-6, -1e-6, 1e-3, -1e-3)))
    assert res.certified
    assert res.energy == float(d["maxflow"])


def test_full_size_cfg4_f64_bitwise_vs_oracle():
    # BASELINE cfg4 geometry (256^3) for a few iterations: device f64 == C oracle
    from oracle import oracle as orc
    g = make_instance("cfg4", seed=0)
    k = 2
    z_ref, y_ref, _ = orc.aar(g, k, threads=orc.max_threads())
    res = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(max_iters=k, check_every=k + 1, precision="f64"))
    assert np.array_equal(res.dual_state.z, z_ref)
    assert np.array_equal(res.dual_state.y, y_ref)


def _weights_regime(rng, shapes, regime):
    out = []
    for s in shapes:
        if regime == "uniform":
            a = rng.uniform(0, 2, s)
        elif regime == "huge":
            a = rng.uniform(20, 80, s)
        elif regime == "zeros":
            a = rng.integers(0, 3, s).astype(float)
        else:
            a = np.abs(rng.normal(0, 0.5, s))
        out.append(a)
    return out


@pytest.mark.parametrize("regime", ["uniform", "huge", "zeros", "critical"])
@pytest.mark.parametrize("conn,dims", [("2D-4", (37, 290)), ("2D-8", (41, 75)),
                                       ("3D-6", (9, 70, 45)), ("2D-4", (1, 100)),
                                       ("3D-6", (130, 3, 1))])
def test_staged_shadow_matches_oracle_projection(conn, dims, regime):
    """pcb_shadow on the fp32 state == oracle Pi_K of the same z (fp64 arithmetic)."""
    from oracle import oracle as orc
    from paracut_b200 import _native
    from paracut_b200.graph import DIRECTIONS, direction_shape
    rng = np.random.default_rng(hash((conn, dims, regime)) % 2 ** 31)
    n = int(np.prod(dims))
    shapes = [direction_shape(dims, d) for d in DIRECTIONS[conn]]
    g = pc.GridEnergy(dims, conn, rng.normal(0, 3, n), _weights_regime(rng, shapes, regime))
    S = _native.GridSolver(g, precision="f32")
    z = rng.normal(0, 4, size=(S.r, n)) + rng.normal(0, 200, size=n)[None, :]
    S.set_z(z)
    z_used = S.get_z()
    y, _ = S.shadow(want_y=True)
    want = orc.project_K(orc.decompose(g), z_used)
    scale = max(1.0, float(np.max(np.abs(want))))
    assert np.max(np.abs(y - want)) <= 1e-9 * scale * 1e3


@pytest.mark.parametrize("conn,dims", [("2D-4", (64, 70)), ("2D-8", (50, 61)),
                                       ("3D-6", (12, 20, 33))])
def test_staged_step_matches_oracle_iteration(conn, dims):
    """a few fused fp32 iterations == the reference loop on the same start point."""
    from oracle import oracle as orc
    spec = {"2D-4": CONFIGS["cfg2_int"], "2D-8": CONFIGS["cfg3"], "3D-6": CONFIGS["cfg4"]}[conn]
    g = make_instance(spec, seed=11, dims=dims)
    from paracut_b200 import _native
    S = _native.GridSolver(g, precision="f32")
    S.init_cold()
    z0 = S.get_z()
    norms = S.run(5)
    z_gpu = S.get_z()
    z_ref, _, norms_ref = orc.aar(g, 5, z=z0, threads=4)
    assert _rel(z_gpu, z_ref) <= 1e-5
    assert np.allclose(norms, norms_ref, rtol=1e-4)


@pytest.mark.parametrize("target", ["1", "100000"])
@pytest.mark.parametrize("conn,dims", [("2D-4", (64, 520)), ("2D-8", (40, 333)),
                                       ("3D-6", (7, 9, 300))])
def test_intra_chain_split_matches_oracle(monkeypatch, target, conn, dims):
    """Chains cut into blocks joined at speculative merge points give the same
    prox (shadow to ~1e-9) and iterates (1e-4) as whole chains."""
    from oracle import oracle as orc
    from paracut_b200 import _native
    monkeypatch.setenv("PCB_SPLIT_TARGET", target)
    spec = {"2D-4": CONFIGS["cfg2_int"], "2D-8": CONFIGS["cfg3"], "3D-6": CONFIGS["cfg4"]}[conn]
    g = make_instance(spec, seed=3, dims=dims)
    S = _native.GridSolver(g, precision="f32")
    S.init_cold()
    S.run(7)
    z = S.get_z()
    y, _ = S.shadow(want_y=True)
    want = orc.project_K(orc.decompose(g), z)
    assert np.max(np.abs(y - want)) <= 1e-9 * max(1.0, float(np.max(np.abs(want)))) * 1e3
    k = 60
    z_ref, y_ref, _ = orc.aar(g, k, threads=4)
    res = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(max_iters=k, check_every=k + 1, precision="f32"))
    x_ref = g.w - y_ref.sum(axis=0)
    x = g.w - res.dual_state.y.sum(axis=0)
    assert _rel(x, x_ref) <= 1e-4


def test_integer_full_size_f32_reaches_exact_optimum_and_polish_certifies():
    """BASELINE cfg2 integer variant (1024^2): the f32 path's labelling has the
    same (integer) cut energy as the certified fp64 reference-exact run, and a
    short fp64 polish certifies it."""
    g = make_instance(CONFIGS["cfg2_int"], seed=0)
    thr = (0.0, 1e-6, -1e-6, 1e-3, -1e-3)
    r64 = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(max_iters=500, check_every=10, gap_tol=1e-6, thresholds=thr))
    assert r64.certified
    r32 = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(max_iters=500, check_every=501, precision="f32",
                                   thresholds=thr, polish_iters=100))
    assert r32.certified
    assert r32.energy == r64.energy
    assert g.energy(r32.labeling) == r64.energy


def test_stall_triggered_polish_certifies_before_max_iters():
    """polish_stall: once the fp32 gap stops halving, the fp64 polish starts
    early and certifies the same integer optimum (cfg2 integer variant)."""
    g = make_instance(CONFIGS["cfg2_int"], seed=0)
    thr = (0.0, 1e-6, -1e-6, 1e-3)
    r64 = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(max_iters=1000, check_every=10, thresholds=thr))
    assert r64.certified
    r32 = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(max_iters=4000, check_every=10, precision="f32",
                                   thresholds=thr, polish_iters=1000, polish_stall=10))
    assert r32.certified and r32.energy == r64.energy
    start = r32.monitor["polish_start"][0]
    assert start < 4000 and r32.iterations < 1500


def test_f32_warm_start_keeps_zigzag_border_nodes():
    """An AAR point of the exact path (2D-8) loads into the fp32 state and
    reads back unchanged, zig-zag border nodes included (their z is the
    drift: the fused state keeps no p there)."""
    from paracut_b200 import _native
    g = make_instance(CONFIGS["cfg3"], seed=2, dims=(40, 56))
    r64 = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(max_iters=30, check_every=31))
    z = r64.dual_state.z
    S = _native.GridSolver(g, precision="f32")
    S.set_z(z)
    assert np.max(np.abs(S.get_z() - z)) <= 1e-6 * np.max(np.abs(z))


@pytest.mark.parametrize("conn,dims,k", [("2D-4", (256, 256), 200), ("2D-8", (96, 80), 150),
                                         ("3D-6", (24, 20, 28), 150)])
def test_f64s_within_1e6_of_oracle(conn, dims, k):
    """The fp64 split mode (fast kernels, fp64 state and scans, chains split
    at merge points): within the north_star fp64 tolerance 1e-6 of the
    reference at matched iterations (cfg1's geometry first)."""
    from oracle import oracle as orc
    spec = {"2D-4": CONFIGS["cfg1"], "2D-8": CONFIGS["cfg3"], "3D-6": CONFIGS["cfg4"]}[conn]
    g = make_instance(spec, seed=5, dims=dims)
    z_ref, y_ref, norms_ref = orc.aar(g, k, threads=8)
    x_ref = g.w - y_ref.sum(axis=0)
    res = pc.solve(g, pc.decompose_grid(g),
                   pc.SolverConfig(max_iters=k, check_every=k + 1, precision="f64s"))
    x = g.w - res.dual_state.y.sum(axis=0)
    assert _rel(x, x_ref) <= 1e-6
    assert _rel(res.dual_state.z, z_ref) <= 1e-6
    assert np.allclose(res.monitor["aar_step_norm"], norms_ref, rtol=1e-6, atol=1e-9)


def test_clone_and_copy_state_device_handover():
    """pcb_clone + pcb_copy_state: the f64s handle built on the device from an
    f32 one carries the same instance and exactly the same z (p_j converted,
    drift copied), and its iterations match a host round trip (get_z/set_z)."""
    from paracut_b200 import _native
    from paracut_b200.instances import synth_image, energy_from_image
    g = energy_from_image(synth_image((40, 36, 28), 6, 3, 9, seed=7), "3D-6")
    S = _native.GridSolver(g, precision="f32")
    S.init_cold()
    S.run(30, norms=False)
    T = S.clone("f64s")
    T.copy_state(S)
    assert np.array_equal(T.get_z(), S.get_z())
    U = _native.GridSolver(g, precision="f64s")
    U.set_z(S.get_z())
    T.run(20, norms=False)
    U.run(20, norms=False)
    zt, zu = T.get_z(), U.get_z()
    assert np.max(np.abs(zt - zu)) <= 1e-9 * np.max(np.abs(zu))
    # the clone of a rescaled handle keeps the lambda = 1 weights as its base
    S.scale_pairwise(2.0)
    V = S.clone("f64s")
    V.scale_pairwise(1.0)
    W = _native.GridSolver(g, precision="f64s")
    for h in (V, W):
        h.init_cold()
        h.run(5, norms=False)
    assert np.array_equal(V.get_z(), W.get_z())


@pytest.mark.parametrize("precision", ["f32", "f64s"])
def test_graph_replay_equals_eager_iterations(precision):
    # plain iterations replay as CUDA graphs once a handle has run 64 of them
    # (pcb_set_graph_after); replays and eager launches are the same kernels
    from paracut_b200 import _native
    g = make_instance(CONFIGS["cfg4"], seed=3, dims=(40, 36, 44))
    out = []
    for after in (0, 1 << 30):  # graphs from the first block / never
        S = _native.GridSolver(g, precision=precision)
        S.set_graph_after(after)
        S.init_cold()
        norms = np.concatenate([S.run(24), S.run(5), S.run(16)])
        out.append((S.get_z(), norms))
        S.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    # default threshold: the first 64 iterations run eagerly, later blocks replay
    S = _native.GridSolver(g, precision=precision)
    S.init_cold()
    norms = np.concatenate([S.run(24), S.run(5), S.run(16), S.run(40)])
    S2 = _native.GridSolver(g, precision=precision)
    S2.set_graph_after(1 << 30)
    S2.init_cold()
    norms2 = S2.run(85)
    assert np.array_equal(S.get_z(), S2.get_z())
    assert np.array_equal(norms, norms2)
