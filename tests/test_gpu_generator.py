"""GPU-resident instance construction: pcb_create_synthetic
builds the BASELINE instances in HBM bit for bit equal to the host reference
paracut_b200/instances.py (counter-based noise, series log / exp), and a solve
from the device-built instance equals the solve from host arrays."""
import time

import numpy as np
import pytest

import paracut_b200 as pc
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, DeviceGrid, make_instance

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,dims", [("cfg1", (64, 80)), ("cfg2_int", (96, 72)),
                                       ("cfg3", (50, 61)), ("cfg4", (20, 24, 28)),
                                       ("cfg5_int", (16, 18, 20)), ("cfg4", (1, 7, 9))])
def test_device_instance_bitwise_equals_host(name, dims):
    spec = CONFIGS[name]
    g = make_instance(spec, seed=7, dims=dims)
    dg = DeviceGrid(spec, seed=7, dims=dims)
    S = _native.GridSolver(dg, precision="f64")
    w, dws = S.get_instance(spec.connectivity)
    assert w.tobytes() == g.w.tobytes()
    for a, b in zip(dws, g.dir_weights):
        assert a.shape == b.shape and a.tobytes() == b.tobytes()


def test_full_size_baseline_instance_bitwise(capsys):
    """cfg4 at its full 256^3: device arrays equal the host generator's."""
    g = make_instance("cfg4", seed=0)
    w, dws = _native.GridSolver(DeviceGrid("cfg4", seed=0), precision="f32").get_instance("3D-6")
    assert w.tobytes() == g.w.tobytes()
    assert all(a.tobytes() == b.tobytes() for a, b in zip(dws, g.dir_weights))


def test_cfg5_created_on_device_in_under_a_second(capsys):
    dg = DeviceGrid("cfg5", seed=0)
    S = _native.GridSolver(dg, precision="f32")  # warm (lazy module load, pool)
    S.close()
    del S
    t0 = time.perf_counter()
    S = _native.GridSolver(DeviceGrid("cfg5", seed=0), precision="f32")
    S.synchronize()
    dt = time.perf_counter() - t0
    with capsys.disabled():
        print("\n[generator] cfg5 512^3 handle from the device generator: %.3f s" % dt)
    assert dt < 1.0


def test_solve_from_device_grid_matches_host_arrays():
    dims = (24, 20, 28)
    g = make_instance("cfg4", seed=3, dims=dims)
    dg = DeviceGrid("cfg4", seed=3, dims=dims)
    cfg = pc.SolverConfig(max_iters=60, check_every=20, precision="f32")
    a = pc.solve(g, pc.decompose_grid(g), cfg)
    b = pc.solve(dg, pc.decompose_grid(dg), cfg)
    assert np.array_equal(a.labeling, b.labeling) and a.energy == b.energy
    assert np.array_equal(a.dual_state.y, b.dual_state.y)
    assert b.dual_state.fingerprint == pc.instance_fingerprint(g)


@pytest.mark.parametrize("name,dims,P", [("cfg4", (16, 20, 24), 4), ("cfg2", (40, 56), 4)])
def test_rank_parts_generated_on_device(name, dims, P):
    """A sharded rank's slab and pencil built by pcb_create_synthetic_box equal
    the host reference make_part (and so the slices of the whole instance),
    and a sharded run over a DeviceGrid -- every rank generating only its own
    parts -- reproduces the sharded run over host arrays bit for bit."""
    from paracut_b200.distributed import LocalComm, ShardedAAR, SlabGeometry
    from paracut_b200.instances import make_part
    spec = CONFIGS[name]
    dg = DeviceGrid(spec, seed=4, dims=dims)
    geo = SlabGeometry(dims, spec.connectivity, P)
    for rk in range(P):
        for o, e, d, m in geo.parts(rk):
            ref = make_part(spec, 4, dims, o, e, d, m)
            w, dws = _native.GridSolver(dg.part(o, e, d, m), precision="f32").get_instance(
                spec.connectivity)
            assert w.tobytes() == ref.w.tobytes()
            assert all(a.tobytes() == b.tobytes() for a, b in zip(dws, ref.dir_weights))
    g = make_instance(spec, seed=4, dims=dims)
    backend = lambda sub: _native.GridSolver(sub, precision="f32")  # noqa: E731
    runs = []
    for inst in (g, dg):
        sh = ShardedAAR(inst, LocalComm(P), range(P), backend, device="cuda")
        sh.init_cold()
        norms = sh.run(20)
        runs.append((norms, sh.assemble(sh.local_z())))
    assert np.array_equal(runs[0][0], runs[1][0]) and np.array_equal(runs[0][1], runs[1][1])
