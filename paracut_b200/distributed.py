"""Slab-sharded AAR across ranks -- fp32-state path.

The grid is cut along its slowest axis into P slabs (3D: z-planes, 2D: row
bands).  Chain families inside a slab (3D x and y lines, 2D rows) stay
local on a *slab handle*; the family that crosses slabs (3D z lines, 2D
columns) lives on a *pencil handle*: rank r owns all slabs' positions of
the column chunk [r*Cp, (r+1)*Cp) of the plane, so its chains are whole.
One iteration (the fused (p_j, c) form of solvers.py:295-298):

    pencil : sweep the cross family (FIRST, no update)      -> G_p = d_z
    A2A #1 : pencil -> slab transpose of d_z (fp32)         -> G_s
    slab   : sweep local families (G preset, LAST exports g) -> x, c (slab copy), g
    A2A #2 : slab -> pencil transpose of g (fp32)
    pencil : x -= g; c += (x - g)/r   (pencil copy of the drift)

so each iteration moves 2 * 4 bytes per node across ranks (both bounded
quantities; the divergent drift c never travels).

Overlapped schedule (``overlap=True``, the default on GPUs for 3D-6 and
2D-4): the slab sweeps do not wait for the cross family.  Two streams per
process -- S (slab compute) and C (pencil compute + NCCL):

    C: pencil sweep (FIRST, no update) -> d_z ; A2A #1           (record A)
    S: slab sweeps (FIRST x, MID y, no update) -> G_s = d_x + d_y
    S: wait A ; G_s += d_z ; apply_g (x, c, norm) ; pack g         (record J)
    C: wait J ; A2A #2 ; pencil apply_g

so A2A #1 and the pencil sweep run under the slab sweeps, and A2A #2 plus
the pencil update of iteration k run under the slab sweeps of k + 1.  The
per-node sum is d_x + d_y + d_z, the family order of the unsharded run.
2D-8 adds its two one-row halo exchanges on S: the straddling paths' d goes
up before the cross family's d is added, the owner's complete first-row g
comes back down before the slab update.

2D-8 row slabs: rows and zig-zag pairs inside a slab are local, the zig-zag
path of the pair straddling a boundary runs on the upper rank, whose handle
carries the next slab's first row as a halo (``SlabGeometry.halo``).  Its
iteration replaces the slab's LAST role by ``apply_g`` after two one-row
exchanges (the path's d up to the owner, the owner's complete g back down),
so the owner's and the halo's drift and primal stay bitwise equal; the
certificate moves the path's shadow up and the owner's full first-row shadow
down, and the halo's unary / dual terms are left to the owner
(``pcb_set_owned``).  Step norms are reduced
across ranks as partial sums of squares.  Communication goes through a
``comm`` object (``TorchComm`` over torch.distributed -- NCCL on GPUs, gloo
on CPU -- or ``LocalComm`` for P virtual ranks in one process), so the
same driver runs multi-process and single-process.

Certificates stay sharded (``check``): each handle computes its shadow,
the cross family's shadow moves pencil -> slab in one fp64 all-to-all, every
slab handle certifies its own nodes and intra-slab edges with the device
reductions (``pcb_check``), the cut across slab boundaries uses the next
rank's first label plane, and the per-rank cut, unary, dual and smooth-dual
partials are summed across ranks.  ``solve_sharded`` runs the reference
driver loop (checks every ``check_every``, stop at ``gap_tol``) on top.
"""
from __future__ import annotations

import numpy as np

from .graph import DIRECTIONS, GridEnergy, as_grid

CROSS = {"2D-4": 1, "2D-8": 1, "3D-6": 2}                # family that crosses slabs
LOCAL = {"2D-4": (0,), "2D-8": (0, 2, 3), "3D-6": (0, 1)}  # families inside a slab
# 2D-8: the zig-zag path of the row pair that straddles a slab boundary is
# swept by the upper slab's rank, whose handle carries the next slab's first
# row as a halo (row-direction weights zeroed there, so that row's row chains
# are inert singletons); the path's d / shadow on the halo row move to the
# owner and the owner's complete g / shadow come back.
HALO = {"2D-8"}
ZIGZAG_PHASE = {2: 0, 3: 1}  # 2D-8 family -> phase: node (row, x) of pair row - ((x + phase) & 1)


class SlabGeometry:
    """Which nodes a rank owns in slab and in pencil layout."""

    def __init__(self, dims, connectivity, world):
        if connectivity not in CROSS:
            raise ValueError("slab sharding supports 2D-4, 2D-8 and 3D-6 grids, not %r"
                             % connectivity)
        self.dims = tuple(int(d) for d in dims)
        self.conn = connectivity
        self.P = int(world)
        D0 = self.dims[0]
        self.plane = int(np.prod(self.dims[1:]))
        if D0 % self.P or self.plane % self.P:
            raise ValueError("world size %d must divide dims[0]=%d and the plane size %d"
                             % (self.P, D0, self.plane))
        self.dz = D0 // self.P
        self.cp = self.plane // self.P
        self.n_slab = self.dz * self.plane
        self.n_pencil = D0 * self.cp

    def halo(self, rank):
        """Rows of the next slab this rank's handle carries (2D-8: 1, except the last rank)."""
        return 1 if self.conn in HALO and rank < self.P - 1 else 0

    def slab_grid(self, g, rank):
        """GridEnergy of rank's slab (all directions sliced; the cross one is unused)."""
        if self.conn in HALO:
            return self._halo_slab_grid(g, rank)
        z0, z1 = rank * self.dz, (rank + 1) * self.dz
        dims = (self.dz,) + self.dims[1:]
        w = g.w.reshape(self.dims)[z0:z1].ravel()
        dws = []
        for d, a in zip(DIRECTIONS[self.conn], g.dir_weights):
            hi = z1 - abs(d[0]) if z1 - abs(d[0]) > z0 else z0
            dws.append(np.ascontiguousarray(a[z0:max(hi, z0)]))
        # the cross direction's slab slice keeps only intra-slab edges; unused
        k = CROSS[self.conn]
        dws[k] = np.ascontiguousarray(g.dir_weights[k][z0:z0 + max(self.dz - 1, 0)])
        return GridEnergy(dims, self.conn, np.ascontiguousarray(w), dws)

    def _halo_slab_grid(self, g, rank):
        """2D-8 row slab plus the next slab's first row: rows and zig-zag pairs
        of the slab, the straddling pair, and the column edges to the halo row
        (the slab's certificate counts them); the halo row's row edges are 0."""
        z0, h = rank * self.dz, self.dz + self.halo(rank)
        W = self.dims[1]
        w = np.ascontiguousarray(g.w.reshape(self.dims)[z0:z0 + h].ravel())
        rows = np.array(g.dir_weights[0][z0:z0 + h], dtype=np.float64)
        if self.halo(rank):
            rows[-1] = 0.0
        cols = np.ascontiguousarray(g.dir_weights[1][z0:z0 + h - 1])
        d1 = np.ascontiguousarray(g.dir_weights[2][z0:z0 + h - 1])
        d2 = np.ascontiguousarray(g.dir_weights[3][z0:z0 + h - 1])
        assert rows.shape == (h, W - 1) and cols.shape == (h - 1, W)
        return GridEnergy((h, W), self.conn, w, [rows, cols, d1, d2])

    def parts(self, rank):
        """(slab, pencil) of rank as boxes of the global grid for the device
        generator -- (origin, extent, handle dims, direction mask) each -- or
        None where the layout is not a box (2D-8 halo slabs; a pencil that is
        not whole rows of the plane)."""
        if self.conn in HALO:
            return None
        D0, rest = self.dims[0], self.dims[1:]
        k = CROSS[self.conn]
        slab = ((rank * self.dz,) + (0,) * len(rest), (self.dz,) + rest, (self.dz,) + rest, 0xF)
        if self.conn == "3D-6":
            D1, D2 = rest
            if self.cp % D2:
                return None
            rows = self.cp // D2
            pencil = ((0, rank * rows, 0), (D0, rows, D2), (D0, 1, self.cp), 1 << k)
        else:
            pencil = ((0, rank * self.cp), (D0, self.cp), (D0, self.cp), 1 << k)
        return slab, pencil

    def pencil_cols(self, rank):
        return np.arange(rank * self.cp, (rank + 1) * self.cp)

    def pencil_grid(self, g, rank):
        """Grid whose cross-family chains are rank's pencil columns (other families unused)."""
        cols = self.pencil_cols(rank)
        D0 = self.dims[0]
        k = CROSS[self.conn]
        w = g.w.reshape(D0, self.plane)[:, cols]
        a = g.dir_weights[k].reshape(D0 - 1, self.plane)[:, cols]
        if self.conn == "3D-6":
            dims = (D0, 1, self.cp)
            dws = [np.zeros((D0, 1, self.cp - 1)), np.zeros((D0, 0, self.cp)),
                   a.reshape(D0 - 1, 1, self.cp)]
        else:
            dims = (D0, self.cp)
            dws = [np.zeros((D0, self.cp - 1)), a.reshape(D0 - 1, self.cp)]
            if self.conn == "2D-8":
                dws += [np.zeros((D0 - 1, self.cp - 1)), np.zeros((D0 - 1, self.cp - 1))]
        return GridEnergy(dims, self.conn, np.ascontiguousarray(w.ravel()),
                          [np.ascontiguousarray(x) for x in dws])


class LocalComm:
    """P virtual ranks in one process (tensors of every rank on one device)."""

    def __init__(self, world):
        self.world = int(world)

    def all_to_all(self, sends, recvs):
        """sends[r]: tensor [P, ...] (chunk q goes to rank q); recvs[r][q] <- sends[q][r]."""
        for r in range(self.world):
            for q in range(self.world):
                recvs[r][q].copy_(sends[q][r])

    def send_next(self, sends, recvs):
        """recvs[r] <- sends[r - 1] (sends[P-1] and recvs[0] are None)."""
        for r in range(1, self.world):
            recvs[r].copy_(sends[r - 1])

    def send_prev(self, sends, recvs):
        """recvs[r] <- sends[r + 1] (sends[0] and recvs[P-1] are None)."""
        for r in range(self.world - 1):
            recvs[r].copy_(sends[r + 1])

    def all_sum(self, values):
        tot = np.zeros_like(np.asarray(values[0], dtype=np.float64))
        for v in values:  # rank order, like TorchComm
            tot = tot + np.asarray(v, dtype=np.float64)
        return [tot] * self.world


class TorchComm:
    """One rank per process over torch.distributed (NCCL for cuda tensors, gloo for cpu)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()

    def all_to_all(self, sends, recvs):
        (s,), (r,) = sends, recvs
        self.dist.all_to_all_single(r.view(-1), s.reshape(-1).contiguous())

    def _p2p(self, send, send_to, recv, recv_from):
        ops = []
        if send is not None:
            ops.append(self.dist.P2POp(self.dist.isend, send.contiguous(), send_to))
        if recv is not None:
            ops.append(self.dist.P2POp(self.dist.irecv, recv, recv_from))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def send_next(self, sends, recvs):
        (s,), (r,) = sends, recvs
        self._p2p(s, self.rank + 1, r, self.rank - 1)

    def send_prev(self, sends, recvs):
        (s,), (r,) = sends, recvs
        self._p2p(s, self.rank - 1, r, self.rank + 1)

    def all_sum(self, values):
        import torch
        (v,) = values
        t = torch.as_tensor(np.asarray(v, dtype=np.float64))
        if self.dist.get_backend() == "nccl":
            t = t.cuda()
        # deterministic: gather every rank's partials, sum in rank order
        parts = [torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t)
        tot = parts[0].clone()
        for q in parts[1:]:
            tot += q
        return [tot.cpu().numpy()]


def _wrap(dev_ptr, count, dtype, device):
    """torch tensor view of a handle's device buffer (__cuda_array_interface__)."""
    import torch

    class _CAI:
        pass

    o = _CAI()
    typestr = {np.float32: "<f4", np.float64: "<f8", np.uint8: "|u1"}[dtype]
    o.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                  "data": (int(dev_ptr), False), "version": 3}
    return torch.as_tensor(o, device=device)


class ShardedAAR:
    """Slab-sharded fixed-iteration AAR for the local ranks `ranks` of `comm`.

    backend(grid) must return a per-handle solver with the GridSolver
    interface (``_native.GridSolver`` with precision="f32", or a CPU
    emulation in tests).
    """

    def __init__(self, g, comm, ranks, backend, device=None, overlap=None):
        import torch
        from . import _native as N
        self.N = N
        g = as_grid(g)  # (a DeviceGrid passes through: ranks generate their parts)
        self.g = g
        self.comm = comm
        self.ranks = list(ranks)
        self.geo = SlabGeometry(g.dims, g.connectivity, comm.world)
        self.r = len(DIRECTIONS[g.connectivity])
        self.cross = CROSS[g.connectivity]
        self.slab, self.pencil = [], []
        self.halo = g.connectivity in HALO
        dev = getattr(g, "_is_device_grid", False)
        for rk in self.ranks:
            parts = self.geo.parts(rk) if dev else None
            if parts is not None:  # only the rank's slab and pencil, generated on its device
                (so, se, sd, sm), (po, pe, pd, pm) = parts
                s = backend(g.part(so, se, sd, sm))
                p = backend(g.part(po, pe, pd, pm))
            else:
                s = backend(self.geo.slab_grid(g, rk))
                p = backend(self.geo.pencil_grid(g, rk))
            s.set_family_mask(sum(1 << j for j in LOCAL[g.connectivity]))
            p.set_family_mask(1 << self.cross)
            if self.geo.halo(rk):
                s.set_owned(self.geo.n_slab)
            self.slab.append(s)
            self.pencil.append(p)
        W = self.geo.dims[-1]
        # zig-zag nodes of an owner's first row that lie on the straddling path
        self._straddle = {j: (np.arange(W) + ph) % 2 == 1 for j, ph in ZIGZAG_PHASE.items()}
        self.device = device
        # overlapped schedule (module docstring)
        self.overlap = True if overlap is None else bool(overlap)
        self._bufs = []
        for s, p in zip(self.slab, self.pencil):
            self._bufs.append(dict(Gs=self._tensor(s, N.BUF_G, np.float32),
                                   Gp=self._tensor(p, N.BUF_G, np.float32),
                                   Cp=self._tensor(p, N.BUF_C, np.float64),
                                   Ns=self._tensor(s, N.BUF_NORMS, np.float64),
                                   Np=self._tensor(p, N.BUF_NORMS, np.float64)))
        P, dz, cp = self.geo.P, self.geo.dz, self.geo.cp
        self._recv_s = [torch.empty((P, dz, cp), dtype=torch.float32, device=self._dev())
                        for _ in self.ranks]
        if self.overlap:  # packed g (slab -> pencil), separate from G_s so S can run ahead
            self._send_g = [torch.empty((P, dz, cp), dtype=torch.float32, device=self._dev())
                            for _ in self.ranks]
            # no halo: the slab sends the pencils their new drift (fp64) instead
            self._send_c = ([torch.empty((P, dz, cp), dtype=torch.float64, device=self._dev())
                             for _ in self.ranks] if not self.halo else None)
            self._streams = None
        if self.halo:
            self._hrow = [torch.empty(W, dtype=torch.float32, device=self._dev())
                          for _ in self.ranks]
            self._mask = {j: torch.as_tensor(m, device=self._dev())
                          for j, m in self._straddle.items()}

    def _dev(self):
        return self.device if self.device is not None else "cpu"

    def _tensor(self, h, which, dtype):
        if hasattr(h, "host_buffer"):  # CPU emulation
            import torch
            return torch.from_numpy(h.host_buffer(which))
        ptr, cnt = h.device_buffer(which)
        return _wrap(ptr, cnt, dtype, self._dev())

    # ---------------------------------------------------------------- state
    def init_cold(self):
        for s, p in zip(self.slab, self.pencil):
            s.init_cold()
            p.init_cold()

    def set_z(self, z):
        """Warm start from a global AAR point z (r, n), natural layout."""
        z = np.asarray(z, dtype=np.float64).reshape(self.r, self.g.dims[0], self.geo.plane)
        for i, rk in enumerate(self.ranks):
            z0, z1 = rk * self.geo.dz, (rk + 1) * self.geo.dz + self.geo.halo(rk)
            zs = np.ascontiguousarray(z[:, z0:z1])
            emu = hasattr(self.slab[i], "host_buffer")
            if self.halo and not emu:
                fix = self._halo_seam_z(z, zs, rk)
            self.slab[i].set_z(zs.reshape(self.r, -1))
            if self.halo:
                self._zero_halo_rows(i, rk)
                if not emu:
                    self._set_seam_x(i, fix)
            cols = self.geo.pencil_cols(rk)
            self.pencil[i].set_z(np.ascontiguousarray(z[:, :, cols].reshape(self.r, -1)))

    def _halo_seam_z(self, z, zs, rk):
        """On the seam rows (an owner's first row, a halo row) each slab handle
        lacks one zig-zag family that the global grid has there, and its
        set_z takes the drift from that border family.  Hand it the global
        drift (mean over families, the single handle's choice for these
        interior nodes); returns {local row: global primal X} to restore."""
        dz, W = self.geo.dz, self.geo.dims[-1]
        fix = {}
        seams = ([(0, True)] if rk > 0 else []) + ([(dz, False)] if self.geo.halo(rk) else [])
        for row, on_path in seams:
            zg = z[:, rk * dz + row]
            m = zg[0].copy()
            for j in range(1, self.r):
                m = m + zg[j]
            m = m / self.r
            for j, msk in self._straddle.items():
                lack = msk if on_path else ~msk  # nodes whose family-j state is elsewhere
                zs[j, row, lack] = m[lack]
            sp = np.zeros(W)
            for j in range(self.r):
                sp = sp + (zg[j] - m).astype(np.float32).astype(np.float64)
            w = self.g.w.reshape(self.g.dims)[rk * dz + row]
            fix[row] = (w - sp).astype(np.float32)
        return fix

    def _set_seam_x(self, i, fix):
        import torch
        W = self.geo.dims[-1]
        X = self._tensor(self.slab[i], self.N.BUF_X, np.float32)
        for row, x in fix.items():
            X[row * W:(row + 1) * W] = torch.as_tensor(x, device=self._dev())

    def _zero_halo_rows(self, i, rk):
        """The halo row's row chains are inert: their state stays 0 (its drift
        and primal keep the owner's values)."""
        h, ns, W = self.slab[i], self.geo.n_slab, self.geo.dims[-1]
        if hasattr(h, "host_buffer"):
            # CPU emulation keeps node-order state for every family, where the
            # device keeps none for zig-zag border nodes: zero what another
            # rank's path owns (halo row off the straddling path, the owner's
            # first row on it)
            if self.geo.halo(rk):
                h.p[0][ns:] = 0
                for j, m in self._straddle.items():
                    h.p[j][ns:][~m] = 0
            if rk > 0:
                for j, m in self._straddle.items():
                    h.p[j][:W][m] = 0
            return
        if not self.geo.halo(rk):
            return
        ptr, cnt = h.device_buffer(self.N.BUF_P)
        rows = ns // W + 1
        # family 0 (rows) in family layout [pos = x][chain = row]
        _wrap(ptr, cnt, np.float32, self._dev())[:rows * W].view(W, rows)[:, rows - 1].zero_()

    # ---------------------------------------------------------------- iterations
    def run(self, iters, norms=True):
        """iters fused iterations; returns ||z_{k+1} - z_k|| per iteration (all ranks).

        Per-iteration partial sums of squares stay on the device and are
        reduced across ranks once at the end, so the loop never syncs the host."""
        import torch
        N = self.N
        P, dz, cp = self.geo.P, self.geo.dz, self.geo.cp
        K = int(iters)
        acc = [torch.zeros(K, dtype=torch.float64, device=self._dev()) for _ in self.ranks]
        if self.overlap:
            self._run_overlap(K, acc)
        elif self.halo:
            self._run_halo(K, acc)
        for k in range(0 if (self.halo or self.overlap) else K):
            for i, p in enumerate(self.pencil):
                p.step(1, N.STEP_NO_UPDATE | N.STEP_NORM_RAW, norms=False)
                acc[i][k] += self._bufs[i]["Np"][0]
            # pencil -> slab: d of the cross family; chunk q = slab q's planes
            sends = [b["Gp"].view(P, dz, cp) for b in self._bufs]
            self.comm.all_to_all(sends, self._recv_s)
            for i, b in enumerate(self._bufs):
                b["Gs"].view(dz, P, cp).copy_(self._recv_s[i].transpose(0, 1))
            for i, s in enumerate(self.slab):
                s.step(1, N.STEP_G_PRESET | N.STEP_EXPORT_G | N.STEP_NORM_RAW, norms=False)
                acc[i][k] += self._bufs[i]["Ns"][0]
            # slab -> pencil: g (sum of all families' d); chunk q = pencil q's columns
            sends = [b["Gs"].view(dz, P, cp).transpose(0, 1).contiguous() for b in self._bufs]
            recvs = [b["Gp"].view(P, dz, cp) for b in self._bufs]
            self.comm.all_to_all(sends, recvs)
            for i, p in enumerate(self.pencil):
                if hasattr(p, "host_buffer"):
                    p.apply_g_host(self._bufs[i]["Gp"].numpy())
                else:
                    p.apply_g(self._bufs[i]["Gp"].data_ptr())
        if not norms:
            return None
        tot = self.comm.all_sum([a.cpu().numpy() for a in acc])
        return np.sqrt(np.maximum(np.asarray(tot[0], dtype=np.float64), 0.0))

    def _stream_pair(self):
        """(S, C) CUDA streams of the overlapped schedule, or (None, None) on CPU."""
        import torch
        if not (self.device is not None and str(self.device).startswith("cuda")):
            return None, None
        if self._streams is None:
            self._streams = (torch.cuda.Stream(), torch.cuda.Stream())
        return self._streams

    def _run_overlap(self, K, acc):
        """Overlapped iterations (module docstring): slab work on stream S, pencil
        sweep / update and both all-to-alls on stream C, joined by two events per
        iteration.  Forks from and joins back to the caller's current stream, so
        it runs eagerly and inside a CUDA-graph capture alike."""
        import contextlib
        import torch
        N = self.N
        P, dz, cp = self.geo.P, self.geo.dz, self.geo.cp
        ns, W = self.geo.n_slab, self.geo.dims[-1]
        first = [rk > 0 for rk in self.ranks]
        has_halo = [bool(self.geo.halo(rk)) for rk in self.ranks]
        S, C = self._stream_pair()
        cuda = S is not None

        def on(st):
            return torch.cuda.stream(st) if cuda else contextlib.nullcontext()

        acc_p = [torch.zeros_like(a) for a in acc]  # C-side partials (acc is S-side)
        if cuda:
            base = torch.cuda.current_stream()
            S.wait_stream(base)
            C.wait_stream(base)
            for s in self.slab:
                s.set_stream(S.cuda_stream)
            for p in self.pencil:
                p.set_stream(C.cuda_stream)
        try:
            for k in range(K):
                with on(C):  # cross family: d_z, then pencil -> slab
                    for i, p in enumerate(self.pencil):
                        p.step(1, N.STEP_NO_UPDATE | N.STEP_NORM_RAW, norms=False)
                        acc_p[i][k] += self._bufs[i]["Np"][0]
                    self.comm.all_to_all([b["Gp"].view(P, dz, cp) for b in self._bufs],
                                         self._recv_s)
                    ev_a = torch.cuda.Event() if cuda else None
                    if cuda:
                        ev_a.record(C)
                with on(S):  # local families while d_z is in flight
                    for i, s in enumerate(self.slab):
                        s.step(1, N.STEP_NO_UPDATE | N.STEP_NORM_RAW, norms=False)
                        acc[i][k] += self._bufs[i]["Ns"][0]
                    if self.halo:  # straddling paths' d on the halo row -> the owner's first row
                        self.comm.send_next(
                            [b["Gs"][ns:] if h else None for b, h in zip(self._bufs, has_halo)],
                            [hr if f else None for hr, f in zip(self._hrow, first)])
                        for i, b in enumerate(self._bufs):
                            if first[i]:
                                b["Gs"][:W] += self._hrow[i]
                    if cuda:
                        S.wait_event(ev_a)
                    if not self.halo:
                        # one fused pass: g = G + d_z into the send buffer, and the update
                        for i, (s, b) in enumerate(zip(self.slab, self._bufs)):
                            if hasattr(s, "host_buffer"):
                                s.apply_g_exchange_host(self._recv_s[i].numpy(),
                                                        self._send_c[i].numpy(), P, dz, cp)
                            else:
                                s.apply_g_exchange(self._recv_s[i].data_ptr(),
                                                   self._send_c[i].data_ptr(), P, dz, cp)
                            acc[i][k] += b["Ns"][1]
                    else:
                        for i, b in enumerate(self._bufs):
                            b["Gs"][:ns].view(dz, P, cp).add_(self._recv_s[i].transpose(0, 1))
                            self._send_g[i].copy_(b["Gs"][:ns].view(dz, P, cp).transpose(0, 1))
                        # the owner's complete first-row g -> the halo row
                        self.comm.send_prev(
                            [b["Gs"][:W] if f else None for b, f in zip(self._bufs, first)],
                            [b["Gs"][ns:] if h else None for b, h in zip(self._bufs, has_halo)])
                        for i, (s, b) in enumerate(zip(self.slab, self._bufs)):
                            if hasattr(s, "host_buffer"):
                                s.apply_g_host(b["Gs"].numpy())
                            else:
                                s.apply_g(b["Gs"].data_ptr())
                            acc[i][k] += b["Ns"][1]
                    ev_j = torch.cuda.Event() if cuda else None
                    if cuda:
                        ev_j.record(S)
                with on(C):  # slab -> pencil (under the next slab sweeps)
                    if cuda:
                        C.wait_event(ev_j)
                    if not self.halo:  # the new drift straight into the pencils' c
                        self.comm.all_to_all(self._send_c,
                                             [b["Cp"].view(P, dz, cp) for b in self._bufs])
                    else:  # g, then the pencil update
                        recvs = [b["Gp"].view(P, dz, cp) for b in self._bufs]
                        self.comm.all_to_all(self._send_g, recvs)
                        for i, p in enumerate(self.pencil):
                            if hasattr(p, "host_buffer"):
                                p.apply_g_host(self._bufs[i]["Gp"].numpy())
                            else:
                                p.apply_g(self._bufs[i]["Gp"].data_ptr())
        finally:
            if cuda:
                base.wait_stream(S)
                base.wait_stream(C)
                for h in self.slab + self.pencil:
                    h.set_stream(base.cuda_stream)
        if cuda:
            with torch.cuda.stream(base):
                for a, b in zip(acc, acc_p):
                    a += b
        else:
            for a, b in zip(acc, acc_p):
                a += b

    def _run_halo(self, K, acc):
        """2D-8 iterations: every slab-side update goes through apply_g once the
        halo row's g is complete, so the owner's and the halo's copies of the
        drift and primal stay bitwise equal."""
        N = self.N
        P, dz, cp, ns, W = self.geo.P, self.geo.dz, self.geo.cp, self.geo.n_slab, self.geo.dims[-1]
        first = [rk > 0 for rk in self.ranks]
        has_halo = [bool(self.geo.halo(rk)) for rk in self.ranks]
        for k in range(K):
            for i, p in enumerate(self.pencil):
                p.step(1, N.STEP_NO_UPDATE | N.STEP_NORM_RAW, norms=False)
                acc[i][k] += self._bufs[i]["Np"][0]
            sends = [b["Gp"].view(P, dz, cp) for b in self._bufs]
            self.comm.all_to_all(sends, self._recv_s)
            for i, b in enumerate(self._bufs):
                b["Gs"][:ns].view(dz, P, cp).copy_(self._recv_s[i].transpose(0, 1))
                b["Gs"][ns:].zero_()
            for i, s in enumerate(self.slab):
                s.step(1, N.STEP_G_PRESET | N.STEP_NO_UPDATE | N.STEP_NORM_RAW, norms=False)
                acc[i][k] += self._bufs[i]["Ns"][0]
            # halo up: the straddling paths' d on the halo row -> the owner's first row
            self.comm.send_next([b["Gs"][ns:] if h else None for b, h in zip(self._bufs, has_halo)],
                                [hr if f else None for hr, f in zip(self._hrow, first)])
            for i, b in enumerate(self._bufs):
                if first[i]:
                    b["Gs"][:W] += self._hrow[i]
            # slab -> pencil: the complete g of the owned rows
            sends = [b["Gs"][:ns].view(dz, P, cp).transpose(0, 1).contiguous() for b in self._bufs]
            recvs = [b["Gp"].view(P, dz, cp) for b in self._bufs]
            self.comm.all_to_all(sends, recvs)
            # halo down: the owner's complete g of its first row -> the halo row
            self.comm.send_prev([b["Gs"][:W] if f else None for b, f in zip(self._bufs, first)],
                                [b["Gs"][ns:] if h else None for b, h in zip(self._bufs, has_halo)])
            for i, (s, p) in enumerate(zip(self.slab, self.pencil)):
                if hasattr(s, "host_buffer"):
                    s.apply_g_host(self._bufs[i]["Gs"].numpy())
                    p.apply_g_host(self._bufs[i]["Gp"].numpy())
                else:
                    s.apply_g(self._bufs[i]["Gs"].data_ptr())
                    p.apply_g(self._bufs[i]["Gp"].data_ptr())
                acc[i][k] += self._bufs[i]["Ns"][1]

    # ---------------------------------------------------------------- certificates
    def _ybuf(self, h):
        if hasattr(h, "host_buffer"):  # CPU emulation
            import torch
            return torch.from_numpy(h.host_buffer(self.N.BUF_Y))
        ptr, cnt = h.device_buffer(self.N.BUF_Y)
        return _wrap(ptr, cnt, np.float64, self._dev())

    def _bitbuf(self, h):
        """Check labels of a slab handle on the device: uint8[n], bit t = threshold t."""
        if hasattr(h, "host_buffer"):  # CPU emulation
            import torch
            return torch.from_numpy(h.host_buffer(self.N.BUF_BITS))
        ptr, cnt = h.device_buffer(self.N.BUF_BITS)
        return _wrap(ptr, cnt, np.uint8, self._dev())

    def check(self, thresholds=(0.0,)):
        """Global (energies[T], gaps[T], smooth dual) of the current iterate;
        labels stay on their ranks (slab handles' check state)."""
        import torch
        thr = np.asarray(thresholds, dtype=np.float64)
        T = thr.size
        P, dz, cp, plane = self.geo.P, self.geo.dz, self.geo.cp, self.geo.plane
        ns, npn = self.geo.n_slab, self.geo.n_pencil
        x = self.cross
        for s, p in zip(self.slab, self.pencil):
            s.shadow()
            p.shadow()
        # slab handles hold ns (+ one halo row) nodes per family
        next_ = [ns + plane * self.geo.halo(rk) for rk in self.ranks]
        ys = [self._ybuf(s).view(self.r, ne) for s, ne in zip(self.slab, next_)]
        # the cross family's shadow: pencil (D0, cp) -> slab (dz, P * cp)
        sends = [self._ybuf(p)[x * npn:(x + 1) * npn].view(P, dz, cp) for p in self.pencil]
        recvs = [torch.empty((P, dz, cp), dtype=torch.float64, device=self._dev())
                 for _ in self.ranks]
        self.comm.all_to_all(sends, recvs)
        for y, rv in zip(ys, recvs):
            y[x, :ns].view(dz, P, cp).copy_(rv.transpose(0, 1))
        if self.halo:
            self._halo_shadow(ys)
        # per-rank certificate of the slab (its nodes, its intra-slab edges)
        a_b = np.asarray(self.g.dir_weights[x], dtype=np.float64).reshape(self.g.dims[0] - 1, plane)
        local = []
        for rk, s in zip(self.ranks, self.slab):
            e, gp, smooth = s.check(thr)
            local.append((rk, e, float(e[0] - gp[0]), float(smooth)))
        cut_b = [np.zeros(T) for _ in self.ranks]
        if not self.halo:
            # edges between a slab's last plane and the next slab's first: the
            # next rank sends its first plane of label bits (bit t = threshold t)
            bits = [self._bitbuf(s)[:ns] for s in self.slab]
            first = [torch.empty(plane, dtype=torch.uint8, device=b.device) for b in bits]
            self.comm.send_prev([b[:plane] if rk > 0 else None for b, rk in zip(bits, self.ranks)],
                                [f if rk < P - 1 else None for f, rk in zip(first, self.ranks)])
            tb = torch.arange(T, dtype=torch.uint8, device=bits[0].device)[:, None]
            for q, (rk, b, f) in enumerate(zip(self.ranks, bits, first)):
                if rk == P - 1:
                    continue
                diff = (((b[ns - plane:][None, :] >> tb) & 1) != ((f[None, :] >> tb) & 1))
                row = torch.as_tensor(a_b[(rk + 1) * dz - 1], device=b.device)
                cut_b[q] = (diff.to(torch.float64) @ row).cpu().numpy()
        parts = []
        for (rk, e, dual, smooth), cb in zip(local, cut_b):
            parts.append(np.concatenate([np.asarray(e, dtype=np.float64) + cb, [dual, smooth]]))
        tot = self.comm.all_sum(parts)[0]
        energies, dual, smooth = tot[:T], tot[T], tot[T + 1]
        return energies, energies - dual, smooth

    def _halo_shadow(self, ys):
        """2D-8: the straddling paths' shadow on a halo row joins the owner's
        first row; then the owner's complete first-row shadow (all families)
        becomes the halo row, so the halo's x and labels are the owner's."""
        import torch
        ns, W = self.geo.n_slab, self.geo.dims[-1]
        zz = list(ZIGZAG_PHASE)
        first = [rk > 0 for rk in self.ranks]
        has_halo = [bool(self.geo.halo(rk)) for rk in self.ranks]
        up = [torch.empty((len(zz), W), dtype=torch.float64, device=self._dev()) for _ in ys]
        self.comm.send_next([y[zz, ns:ns + W].contiguous() if h else None
                             for y, h in zip(ys, has_halo)],
                            [u if f else None for u, f in zip(up, first)])
        for y, u, f in zip(ys, up, first):
            if f:
                for t, j in enumerate(zz):
                    y[j, :W] = torch.where(self._mask[j], u[t], y[j, :W])
        down = [torch.empty((self.r, W), dtype=torch.float64, device=self._dev()) for _ in ys]
        self.comm.send_prev([y[:, :W].contiguous() if f else None for y, f in zip(ys, first)],
                            [d if h else None for d, h in zip(down, has_halo)])
        for y, d, h in zip(ys, down, has_halo):
            if h:
                y[:, ns:ns + W] = d

    def capture(self):
        """Record one fused iteration (norms off) as a CUDA graph; replay it with
        ``run_graph``.  Every handle launches on the capture stream, torch's
        transposes and the NCCL all-to-alls are captured with them, so an
        iteration costs one graph launch on the host."""
        import torch
        self.run(1, norms=False)  # warm: lazy setup and attributes outside capture
        torch.cuda.synchronize()
        self._gstream = torch.cuda.Stream()
        for h in self.slab + self.pencil:
            h.set_stream(self._gstream.cuda_stream)
        self._graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._graph, stream=self._gstream):
            self.run(1, norms=False)
        torch.cuda.synchronize()
        return self._graph

    def run_graph(self, iters):
        for _ in range(int(iters)):
            self._graph.replay()

    # ---------------------------------------------------------------- results (local ranks)
    def local_z(self):
        """{rank: (slab z of local families [len(LOCAL), n_slab], pencil z_cross [n_pencil])}."""
        res = {}
        loc = LOCAL[self.g.connectivity]
        for i, rk in enumerate(self.ranks):
            zs = self.slab[i].get_z()
            zp = self.pencil[i].get_z()
            res[rk] = (zs[list(loc)], zp[self.cross])
        return res

    def local_shadow(self):
        res = {}
        loc = LOCAL[self.g.connectivity]
        for i, rk in enumerate(self.ranks):
            ys, _ = self.slab[i].shadow(want_y=True)
            yp, _ = self.pencil[i].shadow(want_y=True)
            res[rk] = (ys[list(loc)], yp[self.cross])
        return res

    def assemble(self, parts):
        """Global (r, n) array from {rank: (slab local families, pencil cross)} of ALL ranks."""
        D0, plane = self.g.dims[0], self.geo.plane
        out = np.zeros((self.r, D0, plane))
        loc = LOCAL[self.g.connectivity]
        ns = self.geo.n_slab
        for rk, (sl, pe) in parts.items():
            z0, z1 = rk * self.geo.dz, (rk + 1) * self.geo.dz
            for t, j in enumerate(loc):
                out[j, z0:z1] = sl[t][:ns].reshape(self.geo.dz, plane)
            out[self.cross][:, self.geo.pencil_cols(rk)] = pe.reshape(D0, self.geo.cp)
        if self.g.connectivity in HALO:
            # the straddling paths' nodes of each first row live on the rank above
            W = self.g.dims[-1]
            for rk, (sl, _) in parts.items():
                if not self.geo.halo(rk):
                    continue
                z1 = (rk + 1) * self.geo.dz
                for t, j in enumerate(loc):
                    if j in ZIGZAG_PHASE:
                        m = (np.arange(W) + ZIGZAG_PHASE[j]) % 2 == 1
                        out[j, z1, m] = sl[t][ns:ns + W][m]
        return out.reshape(self.r, -1)


def solve_sharded(g, comm, ranks, backend, cfg, device=None):
    """AAR over slab shards with sharded certificates (the reference loop,
    solvers.py:272-307, checks every cfg.check_every, stop at cfg.gap_tol).

    Returns (trace, iterations, best_gap, best_energy, certified); trace rows
    are (k, gap, dual_objective, energy) of the threshold with the least gap.
    """
    from .solvers import GAP_SLACK
    sh = ShardedAAR(g, comm, ranks, backend, device=device)
    sh.init_cold()
    thr = np.asarray(cfg.thresholds, dtype=np.float64)
    trace, best_gap, best_e = [], np.inf, np.nan
    k = 0
    while True:
        if k % cfg.check_every == 0 or k >= cfg.max_iters:
            e, gp, smooth = sh.check(thr)
            t = int(np.argmin(gp))
            trace.append((k, float(gp[t]), float(smooth), float(e[t])))
            if gp[t] < best_gap:
                best_gap, best_e = float(gp[t]), float(e[t])
            if gp[t] <= cfg.gap_tol + GAP_SLACK or k >= cfg.max_iters:
                break
        nxt = min((k // cfg.check_every + 1) * cfg.check_every, cfg.max_iters)
        sh.run(nxt - k, norms=False)
        k = nxt
    return trace, k, best_gap, best_e, best_gap <= cfg.gap_tol + GAP_SLACK
