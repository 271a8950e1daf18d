"""CPU emulation of the fp32-state GridSolver interface (test infrastructure).

Same state, roles and rounding rules as the device fast path
(csrc/fast_sweep.cuh): p_j fp32, drift c fp64, primal X fp32, accumulator G
fp32; FIRST G = d, MID G += d, LAST g32 = fp32(G + d), X -= g32,
c = (z - p_old) + (X_new - g32)/r.  The per-family prox is the oracle's
(fp64).  Lets the slab-sharded driver run over gloo on CPU.
"""
import numpy as np

from oracle import oracle as orc

STEP_G_PRESET, STEP_NO_UPDATE, STEP_EXPORT_G, STEP_NORM_RAW = 1, 2, 4, 8
BUF_G, BUF_X, BUF_C, BUF_Y, BUF_NORMS, BUF_BITS = 0, 1, 2, 3, 4, 6
ORDER = {"2D-4": (0, 1), "2D-8": (0, 1, 2, 3), "3D-6": (0, 1, 2)}


class EmuSolver:
    def __init__(self, g):
        self.g = g
        self.classes = orc.decompose(g)
        self.r = len(self.classes)
        self.n = int(np.asarray(g.w).size)
        self.w = np.asarray(g.w, dtype=np.float64)
        self.mask = (1 << self.r) - 1
        self.p = np.zeros((self.r, self.n), np.float32)
        self.c = np.zeros(self.n)
        self.X = np.zeros(self.n, np.float32)
        self.G = np.zeros(self.n, np.float32)
        self.norms = np.zeros(2)
        self.n_own = self.n
        self.y = np.zeros((self.r, self.n))
        self.bits = None

    def host_buffer(self, which):
        if which == BUF_BITS:
            return self._packed_bits()
        return {BUF_G: self.G, BUF_X: self.X, BUF_C: self.c, BUF_Y: self.y.reshape(-1),
                BUF_NORMS: self.norms}[which]

    def _packed_bits(self):
        out = np.zeros(self.n, dtype=np.uint8)
        for t, lab in enumerate(self.bits):
            out |= (lab.astype(np.uint8) << t)
        return out

    def set_family_mask(self, mask):
        self.mask = mask

    def set_owned(self, n_own):
        self.n_own = int(n_own)

    def init_cold(self):
        self.p[:] = 0
        self.c[:] = self.w / self.r
        self.X[:] = self.w.astype(np.float32)

    def set_z(self, z):
        z = np.asarray(z, dtype=np.float64)
        m = z.mean(axis=0)
        self.p[:] = (z - m).astype(np.float32)
        self.c[:] = m
        self.X[:] = (self.w - self.p.astype(np.float64).sum(axis=0)).astype(np.float32)

    def get_z(self):
        return self.p.astype(np.float64) + self.c

    def _prox_proj(self, j, z):
        out = np.zeros(self.n)
        cls = self.classes[j]
        if cls.num_chains:
            orc.prox_chains(cls, z, out, True)
        return out

    def step(self, iters, flags, norms=True):
        out = np.zeros(int(iters))
        act = [j for j in ORDER[self.g.connectivity] if (self.mask >> j) & 1]
        preset = bool(flags & STEP_G_PRESET)
        noupd = bool(flags & STEP_NO_UPDATE)
        for k in range(int(iters)):
            nrm = 0.0
            if len(act) == 1 and not preset and not noupd:
                self.G[:] = 0
            for q, j in enumerate(act):
                if q == len(act) - 1 and not noupd:
                    role = "LAST"
                elif q == 0 and not preset and not (len(act) == 1 and not noupd):
                    role = "FIRST"
                else:
                    role = "MID"
                pold = self.p[j].copy()
                z = pold.astype(np.float64) + self.c
                pn = self._prox_proj(j, z)
                p32 = pn.astype(np.float32)
                d = p32.astype(np.float64) - pold.astype(np.float64)
                self.p[j] = p32
                nrm += float(d @ d)
                if role == "FIRST":
                    self.G[:] = d.astype(np.float32)
                elif role == "MID":
                    self.G[:] = (self.G.astype(np.float64) + d).astype(np.float32)
                else:
                    g32 = (self.G.astype(np.float64) + d).astype(np.float32)
                    g = g32.astype(np.float64)
                    xn = self.X.astype(np.float64) - g
                    self.X[:] = xn.astype(np.float32)
                    dcv = (xn - g) / self.r
                    self.c[:] = (z - pold.astype(np.float64)) + dcv
                    if flags & STEP_EXPORT_G:
                        self.G[:] = g32
                    nrm += float(np.sum(2.0 * dcv * g + self.r * dcv * dcv))
            out[k] = nrm if flags & STEP_NORM_RAW else np.sqrt(nrm)
            self.norms[0] = out[k]
        return out if norms else None

    def run(self, iters, norms=True):
        return self.step(iters, 0, norms)

    def apply_g_host(self, g):
        gd = np.asarray(g, dtype=np.float32).astype(np.float64)
        xn = self.X.astype(np.float64) - gd
        self.X[:] = xn.astype(np.float32)
        dcv = (xn - gd) * (1.0 / self.r)
        self.c += dcv
        o = self.n_own
        self.norms[1] = float(np.sum(2.0 * dcv[:o] * gd[:o] + self.r * dcv[:o] * dcv[:o]))

    def apply_g_exchange_host(self, recv, send, P, dz, cp):
        """pcb_apply_g_exchange: g = G + d_z (fp32), apply_g, new drift into send [P][dz][cp]."""
        g = (self.G.reshape(dz, P, cp) + np.asarray(recv, dtype=np.float32).reshape(P, dz, cp)
             .transpose(1, 0, 2)).astype(np.float32)
        self.apply_g_host(g.reshape(-1))
        send.reshape(P, dz, cp)[...] = self.c.reshape(dz, P, cp).transpose(1, 0, 2)

    def shadow(self, want_y=True, want_s=False):
        for j in range(self.r):
            if (self.mask >> j) & 1:
                self.y[j] = self._prox_proj(j, self.p[j].astype(np.float64) + self.c)
        return self.y.copy(), None

    def check(self, thr):
        """pcb_check on this handle's grid: per threshold energy over its own
        edges, gap = energy - sum min(s - w, 0), smooth dual."""
        s = self.y.sum(axis=0)
        x = self.w - s
        labs = (x[None, :] > np.asarray(thr)[:, None]).astype(np.uint8)
        self.bits = labs
        o = self.n_own  # halo nodes: labelled for the cut, their sums are the owner's
        e = np.array([orc.grid_tv(self.g, lab) - float(self.w[:o] @ lab[:o]) for lab in labs])
        d = (s - self.w)[:o]
        dual = float(np.minimum(d, 0.0).sum())
        smooth = 0.5 * float(self.w[:o] @ self.w[:o]) - 0.5 * float(d @ d)
        return e, e - dual, smooth

    def check_labels(self, t, packed=False):
        return self.bits[t]
