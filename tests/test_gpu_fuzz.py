"""Randomized shapes and weights through both device paths against the C
oracle: odd and degenerate dims (partial warps, one-node chains, chains
shorter than a tile), zero weights (piece ends), integer data, forced
intra-chain splits and TMA / cp.async families.  f64 is bitwise, f32 and
f64s within the north_star tolerances (1e-4, 1e-6)."""
import numpy as np
import pytest

import paracut_b200 as pc
from paracut_b200.graph import DIRECTIONS, direction_shape

pytestmark = pytest.mark.gpu


def _random_instance(rng):
    conn = ("2D-4", "2D-8", "3D-6")[int(rng.integers(3))]
    if conn == "3D-6":
        dims = tuple(int(v) for v in rng.integers(1, 19, size=3))
    else:
        dims = tuple(int(v) for v in rng.integers(1, 90, size=2))
    n = int(np.prod(dims))
    integer = rng.random() < 0.4
    if integer:
        w = rng.integers(-10, 11, size=n).astype(np.float64)
        dws = [rng.integers(0, 6, size=direction_shape(dims, d)).astype(np.float64)
               for d in DIRECTIONS[conn]]
    else:
        w = rng.normal(0, 3, size=n)
        dws = [rng.uniform(0, 2, size=direction_shape(dims, d))
               * (rng.uniform(size=direction_shape(dims, d)) < 0.85) for d in DIRECTIONS[conn]]
    return pc.GridEnergy(dims, conn, w, dws)


@pytest.mark.parametrize("seed", range(64))
def test_random_instances_both_paths(monkeypatch, oracle_lib, seed):
    rng = np.random.default_rng(1000 + seed)
    g = _random_instance(rng)
    monkeypatch.setenv("PCB_SPLIT_TARGET", str(int(rng.choice([64, 512, 4096]))))
    k = int(rng.integers(1, 40))
    z_ref, y_ref, _ = oracle_lib.aar(g, k, threads=4)
    dec = pc.decompose_grid(g)
    r64 = pc.solve(g, dec, pc.SolverConfig(max_iters=k, check_every=k + 1))
    assert np.array_equal(r64.dual_state.z, z_ref), (g.connectivity, g.dims)
    assert np.array_equal(r64.dual_state.y, y_ref), (g.connectivity, g.dims)
    r32 = pc.solve(g, dec, pc.SolverConfig(max_iters=k, check_every=k + 1, precision="f32"))
    x_ref = g.w - y_ref.sum(axis=0)
    x = g.w - r32.dual_state.y.sum(axis=0)
    scale = max(float(np.max(np.abs(x_ref))), 1.0)
    assert float(np.max(np.abs(x - x_ref))) <= 1e-4 * scale, (g.connectivity, g.dims, k)
    # the fast fp64 mode (split chains, fp64 state and scans): 1e-6
    r64s = pc.solve(g, dec, pc.SolverConfig(max_iters=k, check_every=k + 1, precision="f64s"))
    xs = g.w - r64s.dual_state.y.sum(axis=0)
    assert float(np.max(np.abs(xs - x_ref))) <= 1e-6 * scale, (g.connectivity, g.dims, k)
    # checks every few iterations: the check-iteration update (tiled apply)
    # runs on non-zero states of every family layout
    ce = int(rng.integers(1, 5))
    r32c = pc.solve(g, dec, pc.SolverConfig(max_iters=k, check_every=ce, precision="f32"))
    if r32c.iterations != k:  # certified at an earlier check
        _, y_ref, _ = oracle_lib.aar(g, r32c.iterations, threads=4)
        x_ref = g.w - y_ref.sum(axis=0)
        scale = max(float(np.max(np.abs(x_ref))), 1.0)
    xc = g.w - r32c.dual_state.y.sum(axis=0)
    assert float(np.max(np.abs(xc - x_ref))) <= 1e-4 * scale, (g.connectivity, g.dims, k, ce)
