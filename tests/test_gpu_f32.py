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
