"""Slab-sharded AAR (paracut_b200.distributed): host-side logic on CPU over
gloo (world 2, CPU emulation of the per-rank kernels), and the real kernels
with P virtual ranks on one GPU."""
import os
import socket

import numpy as np
import pytest

from paracut_b200.distributed import LocalComm, ShardedAAR, SlabGeometry
from paracut_b200.instances import CONFIGS, make_instance

SPEC = {"2D-4": CONFIGS["cfg2"], "2D-8": CONFIGS["cfg3"], "3D-6": CONFIGS["cfg4"]}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, conn, dims, iters, q, overlap=False):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    from emu import EmuSolver
    from paracut_b200.distributed import TorchComm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = make_instance(SPEC[conn], seed=2, dims=dims)
        sh = ShardedAAR(g, TorchComm(), [rank], EmuSolver, overlap=overlap)
        sh.init_cold()
        norms = sh.run(iters)
        parts = sh.local_z()
        ys = sh.local_shadow()
        cert = sh.check((0.0, 1e-3))
        q.put((rank, parts, ys, norms, cert))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("conn,dims,overlap", [("3D-6", (6, 8, 5), False), ("2D-4", (12, 10), False),
                                               ("2D-8", (12, 10), False), ("3D-6", (6, 8, 5), True),
                                               ("2D-4", (12, 10), True), ("2D-8", (12, 10), True)])
def test_gloo_world2_matches_unsharded(conn, dims, overlap):
    import multiprocessing as mp
    from emu import EmuSolver
    iters = 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, conn, dims, iters, q, overlap))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = make_instance(SPEC[conn], seed=2, dims=dims)
    ref = EmuSolver(g)
    ref.init_cold()
    # unsharded reference in the same family order as the sharded run:
    # serial schedule: cross family first (FIRST), local families after, LAST =
    # last local one; overlapped schedule: local families first, cross last
    # (the natural order)
    from emu import ORDER
    cross = {"2D-4": 1, "2D-8": 1, "3D-6": 2}[conn]
    ORDER_SAVE = ORDER[conn]
    if overlap:
        ORDER[conn] = tuple(j for j in ORDER_SAVE if j != cross) + (cross,)
    else:
        ORDER[conn] = (cross,) + tuple(j for j in ORDER_SAVE if j != cross)
    try:
        ref_norms = ref.run(iters)
    finally:
        ORDER[conn] = ORDER_SAVE
    sh = ShardedAAR.__new__(ShardedAAR)  # only for assemble()
    from paracut_b200.graph import DIRECTIONS
    sh.g = g
    sh.geo = SlabGeometry(g.dims, conn, 2)
    sh.r = len(DIRECTIONS[conn])
    sh.cross = cross
    zparts, yparts = {}, {}
    for _, parts, ys, _, _ in res:
        zparts.update(parts)
        yparts.update(ys)
    z = sh.assemble(zparts)
    y = sh.assemble(yparts)
    z_ref = ref.get_z()
    y_ref, _ = ref.shadow()
    scale = np.max(np.abs(z_ref))
    # 2D-8: the straddling path's d joins the owner's fp32 accumulator after
    # the owner's own families (a different fp32 summation order), so the
    # iterates agree to fp32 rounding instead of exactly
    # the overlapped schedule adds the cross family's d to the local
    # families' fp32 sum after it was rounded to fp32 for the exchange (the
    # unsharded LAST role adds it unrounded): fp32-rounding agreement too
    tol = 1e-6 if (conn == "2D-8" or overlap) else 1e-9
    assert np.max(np.abs(z - z_ref)) <= tol * scale
    assert np.max(np.abs(y - y_ref)) <= tol * max(1.0, np.max(np.abs(y_ref)))
    for _, _, _, norms, _ in res:
        assert np.allclose(norms, ref_norms, rtol=tol)
    # sharded certificate (labels stay on their ranks, boundary planes
    # exchanged, partials summed) == the unsharded certificate
    e_ref, gap_ref, smooth_ref = ref.check(np.array([0.0, 1e-3]))
    for _, _, _, _, (e, gap, smooth) in res:
        assert np.allclose(e, e_ref, rtol=tol, atol=tol)
        assert np.allclose(gap, gap_ref, rtol=tol, atol=tol * max(1.0, abs(float(gap_ref[0]))))
        assert smooth == pytest.approx(smooth_ref, rel=tol, abs=tol)


def test_geometry_partition():
    geo = SlabGeometry((8, 6, 4), "3D-6", 4)
    assert geo.dz == 2 and geo.cp == 6 and geo.n_slab * 4 == 8 * 24
    g = make_instance(CONFIGS["cfg4"], seed=0, dims=(8, 6, 4))
    sg = geo.slab_grid(g, 1)
    assert sg.dims == (2, 6, 4)
    assert np.array_equal(sg.w, g.w.reshape(8, 24)[2:4].ravel())
    assert np.array_equal(sg.dir_weights[0], g.dir_weights[0][2:4])
    pg = geo.pencil_grid(g, 3)
    assert pg.dims == (8, 1, 6)
    assert np.array_equal(pg.w, g.w.reshape(8, 24)[:, 18:24].ravel())
    assert np.array_equal(pg.dir_weights[2].reshape(7, 6), g.dir_weights[2].reshape(7, 24)[:, 18:24])
    with pytest.raises(ValueError):
        SlabGeometry((8, 6, 4), "3D-6", 3)
    with pytest.raises(ValueError):
        SlabGeometry((8, 8), "2D-6", 2)
    # 2D-8 row slabs carry the next slab's first row (except the last rank)
    g8 = make_instance(CONFIGS["cfg3"], seed=0, dims=(8, 6))
    geo8 = SlabGeometry((8, 6), "2D-8", 2)
    s0, s1 = geo8.slab_grid(g8, 0), geo8.slab_grid(g8, 1)
    assert s0.dims == (5, 6) and s1.dims == (4, 6)
    assert np.array_equal(s0.w, g8.w[:30]) and np.array_equal(s1.w, g8.w[24:])
    assert not s0.dir_weights[0][4].any() and np.array_equal(s0.dir_weights[0][:4], g8.dir_weights[0][:4])
    assert np.array_equal(s0.dir_weights[2], g8.dir_weights[2][:4])  # incl. the straddling pair
    assert np.array_equal(s0.dir_weights[1], g8.dir_weights[1][:4])  # incl. the boundary columns


@pytest.mark.gpu
@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("conn,dims", [("3D-6", (32, 24, 40)), ("2D-4", (64, 96)),
                                       ("2D-8", (64, 96))])
def test_virtual_ranks_on_one_gpu_match_single(P, conn, dims, overlap):
    """P slab/pencil handle pairs on one device (LocalComm, no kernel waits on
    another) reproduce the single-handle f32 run."""
    import paracut_b200 as pc
    from paracut_b200 import _native
    g = make_instance(SPEC[conn], seed=4, dims=dims)
    k = 25
    sh = ShardedAAR(g, LocalComm(P), range(P),
                    lambda sub: _native.GridSolver(sub, precision="f32"), device="cuda",
                    overlap=overlap)
    sh.init_cold()
    norms = sh.run(k)
    z = sh.assemble(sh.local_z())
    y = sh.assemble(sh.local_shadow())
    S = _native.GridSolver(g, precision="f32")
    S.init_cold()
    ref_norms = S.run(k)
    z_ref = S.get_z()
    y_ref, _ = S.shadow(want_y=True)
    x = g.w - y.sum(axis=0)
    x_ref = g.w - y_ref.sum(axis=0)
    assert np.max(np.abs(x - x_ref)) <= 1e-5 * np.max(np.abs(x_ref))
    assert np.max(np.abs(z - z_ref)) <= 1e-6 * np.max(np.abs(z_ref))
    assert np.allclose(norms, ref_norms, rtol=1e-4)


@pytest.mark.gpu
@pytest.mark.parametrize("conn,dims", [("3D-6", (16, 20, 24)), ("2D-4", (40, 56)),
                                       ("2D-8", (32, 48))])
def test_nccl_world1_and_graph_capture_match_eager(conn, dims):
    """The TorchComm/NCCL code path (world 1 in-process) and a CUDA-graph
    capture of one iteration give the same iterates as LocalComm eager."""
    import torch
    import torch.distributed as dist
    from paracut_b200 import _native
    from paracut_b200.distributed import TorchComm
    g = make_instance(SPEC[conn], seed=6, dims=dims)
    backend = lambda sub: _native.GridSolver(sub, precision="f32")
    ref = ShardedAAR(g, LocalComm(1), [0], backend, device="cuda")
    ref.init_cold()
    ref.run(12, norms=False)
    z_ref = ref.assemble(ref.local_z())
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        sh = ShardedAAR(g, TorchComm(), [0], backend, device="cuda")
        sh.init_cold()
        sh.run(2, norms=True)
        sh.capture()          # runs 1 warm iteration, then records one
        sh.run_graph(9)       # 2 + 1 + 9 = 12 iterations
        torch.cuda.synchronize()
        z = sh.assemble(sh.local_z())
    finally:
        dist.destroy_process_group()
    assert np.array_equal(z, z_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("P,conn,dims", [(2, "3D-6", (16, 20, 24)), (4, "2D-4", (64, 48)),
                                         (4, "2D-8", (64, 48))])
def test_virtual_ranks_sharded_certificate_matches_single(P, conn, dims):
    """Sharded certificate (device shadows, fp64 transpose of the cross
    shadow, per-slab pcb_check, boundary planes) == the single handle's
    certificate of the same shadow."""
    from paracut_b200 import _native
    spec = {"2D-4": CONFIGS["cfg2_int"], "2D-8": CONFIGS["cfg3"], "3D-6": CONFIGS["cfg4"]}[conn]
    g = make_instance(spec, seed=5, dims=dims)
    sh = ShardedAAR(g, LocalComm(P), range(P),
                    lambda sub: _native.GridSolver(sub, precision="f32"), device="cuda")
    sh.init_cold()
    sh.run(30, norms=False)
    thr = np.array([0.0, 1e-6, -1e-6])
    e, gap, smooth = sh.check(thr)
    # the same shadow certified by one f64 handle from the assembled z
    S = _native.GridSolver(g, precision="f64")
    S.set_z(sh.assemble(sh.local_z()))
    S.shadow()
    e_ref, gap_ref, smooth_ref = S.check(thr)
    scale = max(1.0, np.max(np.abs(e_ref)))
    assert np.allclose(e, e_ref, rtol=0, atol=1e-6 * scale)
    assert np.allclose(gap, gap_ref, rtol=0, atol=1e-6 * scale)
    assert smooth == pytest.approx(smooth_ref, rel=1e-6)


@pytest.mark.gpu
def test_solve_sharded_certifies_integer_instance():
    from paracut_b200 import _native
    import paracut_b200 as pc
    from paracut_b200.distributed import solve_sharded
    g = make_instance(CONFIGS["cfg2_int"], seed=3, dims=(96, 80))
    cfg = pc.SolverConfig(gap_tol=1e-6, max_iters=4000, check_every=20,
                          thresholds=(0.0, 1e-6, -1e-6, 1e-3, -1e-3))
    trace, k, gap, energy, ok = solve_sharded(
        g, LocalComm(4), range(4), lambda sub: _native.GridSolver(sub, precision="f32"), cfg,
        device="cuda")
    ref = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(gap_tol=1e-6, max_iters=4000,
                                                           check_every=20,
                                                           thresholds=cfg.thresholds))
    assert ok and ref.certified
    assert energy == ref.energy  # integer instance: the same exact optimum


def test_local_ranks_2d8_halo_warm_start_and_certificate():
    """2D-8 row slabs with halo rows, P=3 virtual ranks on CPU (emulated
    kernels): a warm start from a global z, further iterations and the
    sharded certificate follow the unsharded run to fp32 rounding."""
    from emu import EmuSolver, ORDER
    from paracut_b200.distributed import LocalComm
    g = make_instance(CONFIGS["cfg3_int"] if "cfg3_int" in CONFIGS else CONFIGS["cfg3"],
                      seed=7, dims=(12, 12))
    save = ORDER["2D-8"]
    ORDER["2D-8"] = (1, 0, 2, 3)  # the sharded run's order: cross family first
    try:
        ref = EmuSolver(g)
        ref.init_cold()
        ref.run(5)
        z5 = ref.get_z()
        sh = ShardedAAR(g, LocalComm(3), range(3), EmuSolver)
        sh.set_z(z5)
        assert np.max(np.abs(sh.assemble(sh.local_z()) - z5)) <= 1e-6 * np.max(np.abs(z5))
        norms = sh.run(4)
        ref_norms = ref.run(4)
    finally:
        ORDER["2D-8"] = save
    z, z_ref = sh.assemble(sh.local_z()), ref.get_z()
    assert np.max(np.abs(z - z_ref)) <= 1e-6 * np.max(np.abs(z_ref))
    assert np.allclose(norms, ref_norms, rtol=1e-5)
    e, gap, smooth = sh.check((0.0, 1e-3))
    ref.shadow()
    e_ref, gap_ref, smooth_ref = ref.check(np.array([0.0, 1e-3]))
    assert np.allclose(e, e_ref, rtol=1e-6, atol=1e-6)
    assert np.allclose(gap, gap_ref, rtol=1e-6, atol=1e-6 * max(1.0, abs(float(gap_ref[0]))))
    assert smooth == pytest.approx(smooth_ref, rel=1e-6)


@pytest.mark.gpu
def test_virtual_ranks_2d8_warm_start_on_one_gpu():
    """2D-8 halo slabs from a warm start (set_z zeroes the halo row's row-chain
    state in the device family layout) follow the single handle."""
    from paracut_b200 import _native
    g = make_instance(CONFIGS["cfg3"], seed=9, dims=(48, 64))
    S = _native.GridSolver(g, precision="f32")
    S.init_cold()
    S.run(15)
    z15 = S.get_z()
    sh = ShardedAAR(g, LocalComm(4), range(4),
                    lambda sub: _native.GridSolver(sub, precision="f32"), device="cuda")
    sh.set_z(z15)
    assert np.max(np.abs(sh.assemble(sh.local_z()) - z15)) <= 1e-6 * np.max(np.abs(z15))
    norms = sh.run(20)
    ref_norms = S.run(20)
    z, z_ref = sh.assemble(sh.local_z()), S.get_z()
    assert np.max(np.abs(z - z_ref)) <= 1e-5 * np.max(np.abs(z_ref))
    assert np.allclose(norms, ref_norms, rtol=1e-4)
