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
quantities; the divergent drift c never travels).  Step norms are reduced
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

CROSS = {"2D-4": 1, "3D-6": 2}          # family that crosses slabs
LOCAL = {"2D-4": (0,), "3D-6": (0, 1)}  # families inside a slab


class SlabGeometry:
    """Which nodes a rank owns in slab and in pencil layout."""

    def __init__(self, dims, connectivity, world):
        if connectivity not in CROSS:
            raise ValueError("slab sharding supports 2D-4 and 3D-6 grids, not %r" % connectivity)
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

    def slab_grid(self, g, rank):
        """GridEnergy of rank's slab (all directions sliced; the cross one is unused)."""
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
    typestr = {np.float32: "<f4", np.float64: "<f8"}[dtype]
    o.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                  "data": (int(dev_ptr), False), "version": 3}
    return torch.as_tensor(o, device=device)


class ShardedAAR:
    """Slab-sharded fixed-iteration AAR for the local ranks `ranks` of `comm`.

    backend(grid) must return a per-handle solver with the GridSolver
    interface (``_native.GridSolver`` with precision="f32", or a CPU
    emulation in tests).
    """

    def __init__(self, g, comm, ranks, backend, device=None):
        import torch
        from . import _native as N
        self.N = N
        g = as_grid(g)
        self.g = g
        self.comm = comm
        self.ranks = list(ranks)
        self.geo = SlabGeometry(g.dims, g.connectivity, comm.world)
        self.r = len(DIRECTIONS[g.connectivity])
        self.cross = CROSS[g.connectivity]
        self.slab, self.pencil = [], []
        for rk in self.ranks:
            s = backend(self.geo.slab_grid(g, rk))
            p = backend(self.geo.pencil_grid(g, rk))
            s.set_family_mask(sum(1 << j for j in LOCAL[g.connectivity]))
            p.set_family_mask(1 << self.cross)
            self.slab.append(s)
            self.pencil.append(p)
        self.device = device
        self._bufs = []
        for s, p in zip(self.slab, self.pencil):
            self._bufs.append(dict(Gs=self._tensor(s, N.BUF_G, np.float32),
                                   Gp=self._tensor(p, N.BUF_G, np.float32),
                                   Ns=self._tensor(s, N.BUF_NORMS, np.float64),
                                   Np=self._tensor(p, N.BUF_NORMS, np.float64)))
        P, dz, cp = self.geo.P, self.geo.dz, self.geo.cp
        self._recv_s = [torch.empty((P, dz, cp), dtype=torch.float32, device=self._dev())
                        for _ in self.ranks]

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
            z0, z1 = rk * self.geo.dz, (rk + 1) * self.geo.dz
            self.slab[i].set_z(np.ascontiguousarray(z[:, z0:z1].reshape(self.r, -1)))
            cols = self.geo.pencil_cols(rk)
            self.pencil[i].set_z(np.ascontiguousarray(z[:, :, cols].reshape(self.r, -1)))

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
        for k in range(K):
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

    # ---------------------------------------------------------------- certificates
    def _ybuf(self, h):
        if hasattr(h, "host_buffer"):  # CPU emulation
            import torch
            return torch.from_numpy(h.host_buffer(self.N.BUF_Y))
        ptr, cnt = h.device_buffer(self.N.BUF_Y)
        return _wrap(ptr, cnt, np.float64, self._dev())

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
        # the cross family's shadow: pencil (D0, cp) -> slab (dz, P * cp)
        sends = [self._ybuf(p)[x * npn:(x + 1) * npn].view(P, dz, cp) for p in self.pencil]
        recvs = [torch.empty((P, dz, cp), dtype=torch.float64, device=self._dev())
                 for _ in self.ranks]
        self.comm.all_to_all(sends, recvs)
        for s, rv in zip(self.slab, recvs):
            self._ybuf(s)[x * ns:(x + 1) * ns].view(dz, P, cp).copy_(rv.transpose(0, 1))
        # per-rank certificate of the slab (its nodes, its intra-slab edges)
        a_b = np.asarray(self.g.dir_weights[x], dtype=np.float64).reshape(self.g.dims[0] - 1, plane)
        firsts_local, local = [], []
        for rk, s in zip(self.ranks, self.slab):
            e, gp, smooth = s.check(thr)
            labs = np.stack([s.check_labels(t) for t in range(T)]).astype(np.float64)
            mine = np.zeros((P, T, plane))
            mine[rk] = labs[:, :plane]  # this slab's first label plane, for rank rk - 1
            firsts_local.append(mine)
            local.append((rk, e, float(e[0] - gp[0]), float(smooth), labs[:, -plane:]))
        firsts = self.comm.all_sum(firsts_local)[0]
        parts = []
        for rk, e, dual, smooth, last in local:
            cut_b = np.zeros(T)
            if rk < P - 1:  # edges between this slab's last plane and the next one's first
                cut_b = np.abs(last - firsts[rk + 1]) @ a_b[(rk + 1) * dz - 1]
            parts.append(np.concatenate([np.asarray(e, dtype=np.float64) + cut_b,
                                         [dual, smooth]]))
        tot = self.comm.all_sum(parts)[0]
        energies, dual, smooth = tot[:T], tot[T], tot[T + 1]
        return energies, energies - dual, smooth

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
        for rk, (sl, pe) in parts.items():
            z0, z1 = rk * self.geo.dz, (rk + 1) * self.geo.dz
            for t, j in enumerate(loc):
                out[j, z0:z1] = sl[t].reshape(self.geo.dz, plane)
            out[self.cross][:, self.geo.pencil_cols(rk)] = pe.reshape(D0, self.geo.cp)
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
