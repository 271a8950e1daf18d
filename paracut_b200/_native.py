"""ctypes binding of ``libparacut_b200.so`` (the C ABI in include/paracut_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA
device is visible, every entry point raises.  Build the library with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``python -m
paracut_b200.build``); the .so is written in-tree under ``paracut_b200/_lib``.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libparacut_b200.so")

PCB_E_ARG, PCB_E_CUDA, PCB_E_STATE, PCB_E_NOMEM = -1, -2, -3, -4
STEP_G_PRESET, STEP_NO_UPDATE, STEP_EXPORT_G, STEP_NORM_RAW = 1, 2, 4, 8
BUF_G, BUF_X, BUF_C, BUF_Y, BUF_NORMS, BUF_P, BUF_BITS = 0, 1, 2, 3, 4, 5, 6
ALG_BCD, ALG_AP, ALG_FISTA = 1, 2, 3
CONN_CODES = {"2D-4": 0, "2D-8": 1, "3D-6": 2}
PRECISIONS = {"f64": 0, "f32": 1, "f64s": 2}

_lib = None
_lock = threading.Lock()

P = ctypes.c_void_p
I64 = ctypes.c_int64
INT = ctypes.c_int
DBL_P = ctypes.POINTER(ctypes.c_double)


class NativeLibraryMissing(ImportError):
    pass


def _declare(L):
    L.pcb_last_error.restype = ctypes.c_char_p
    L.pcb_version.restype = INT
    L.pcb_device_count.argtypes = [ctypes.POINTER(INT)]
    L.pcb_prox_chains.argtypes = [P, P, P, I64, I64, I64, I64, I64, P, P, INT, INT]
    L.pcb_tv1d_prox_batch.argtypes = [P, P, P, I64, P, INT]
    L.pcb_create.argtypes = [P, INT, INT, INT, P, P, INT, ctypes.POINTER(P)]
    L.pcb_destroy.argtypes = [P]
    L.pcb_shape.argtypes = [P, ctypes.POINTER(INT), ctypes.POINTER(I64)]
    L.pcb_set_stream.argtypes = [P, ctypes.c_size_t]
    L.pcb_synchronize.argtypes = [P]
    L.pcb_init_cold.argtypes = [P]
    L.pcb_set_z.argtypes = [P, P]
    L.pcb_get_z.argtypes = [P, P]
    L.pcb_aar_run.argtypes = [P, I64, P]
    L.pcb_aar_step.argtypes = [P, I64, INT, P]
    L.pcb_set_family_mask.argtypes = [P, ctypes.c_uint]
    L.pcb_clone.argtypes = [P, INT, ctypes.POINTER(P)]
    L.pcb_copy_state.argtypes = [P, P]
    L.pcb_apply_g.argtypes = [P, ctypes.c_size_t]
    L.pcb_device_buffer.argtypes = [P, INT, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(I64)]
    L.pcb_shadow.argtypes = [P, P, P]
    L.pcb_apply.argtypes = [P, P]
    L.pcb_shadow_get.argtypes = [P, P]
    L.pcb_shadow_delta.argtypes = [P, P]
    L.pcb_check.argtypes = [P, INT, P, P, P, P]
    L.pcb_get_check.argtypes = [P, INT, P, INT, P]
    L.pcb_keep_best.argtypes = [P, INT]
    L.pcb_get_best.argtypes = [P, P, P]
    L.pcb_level_set.argtypes = [P, P, P, P]
    L.pcb_dual_init.argtypes = [P, INT, P]
    L.pcb_release_memory.argtypes = [INT]
    L.pcb_scale_pairwise.argtypes = [P, ctypes.c_double]
    L.pcb_create_from_file.argtypes = [ctypes.c_char_p, INT, INT, P, P, P, P]
    L.pcb_debug_counters.argtypes = [P, INT]
    L.pcb_dual_run.argtypes = [P, I64, P, P]
    L.pcb_project_K.argtypes = [P, P, P]
    L.pcb_project_L.argtypes = [P, P, P, INT, I64, P, P, INT]
    L.pcb_set_profiling.argtypes = [P, INT]
    L.pcb_set_graph_after.argtypes = [P, I64]
    L.pcb_profile_read.argtypes = [P, P, P]
    L.pcb_verify_stats.argtypes = [P, P, P, P, P, P]
    L.pcb_apply_g_exchange.argtypes = [P, ctypes.c_size_t, ctypes.c_size_t, INT, INT, INT]
    L.pcb_create_synthetic.argtypes = [P, INT, INT, INT, P, P, ctypes.c_uint64, ctypes.c_double,
                                       INT, INT, INT, P]
    L.pcb_get_instance.argtypes = [P, P, P]
    L.pcb_create_synthetic_box.argtypes = [P, INT, INT, P, P, P, ctypes.c_uint, INT, P, P,
                                           ctypes.c_uint64, ctypes.c_double, INT, INT, INT, P]
    L.pcb_jaccard_packed.argtypes = [P, P, I64, DBL_P]
    L.pcb_set_owned.argtypes = [P, I64]
    L.pcb_log_start.argtypes = [P]
    L.pcb_log_stop.argtypes = [P]
    L.pcb_log_norms.argtypes = [P, P, I64, ctypes.POINTER(I64)]
    L.pcb_log_labels.argtypes = [P, INT, ctypes.POINTER(I64)]
    L.pcb_log_label_get.argtypes = [P, I64, P]
    L.pcb_log_jaccard.argtypes = [P, P, P, I64]
    L.pcb_launch_count.argtypes = [P]
    L.pcb_launch_count.restype = I64
    L.pcb_reset_launch_count.argtypes = [P]
    L.pcb_reset_launch_count.restype = None


EXPORTS = ("pcb_last_error", "pcb_version", "pcb_device_count", "pcb_prox_chains",
           "pcb_tv1d_prox_batch", "pcb_create", "pcb_destroy", "pcb_shape", "pcb_set_stream",
           "pcb_synchronize", "pcb_init_cold", "pcb_set_z", "pcb_get_z", "pcb_aar_run",
           "pcb_aar_step", "pcb_set_family_mask", "pcb_apply_g", "pcb_device_buffer",
           "pcb_shadow", "pcb_shadow_get", "pcb_shadow_delta", "pcb_apply", "pcb_check", "pcb_get_check", "pcb_keep_best",
           "pcb_get_best", "pcb_level_set", "pcb_dual_init", "pcb_dual_run", "pcb_release_memory", "pcb_create_from_file", "pcb_scale_pairwise", "pcb_debug_counters", "pcb_project_K", "pcb_project_L", "pcb_set_profiling", "pcb_profile_read", "pcb_launch_count",
           "pcb_reset_launch_count", "pcb_jaccard_packed", "pcb_set_owned", "pcb_log_start",
           "pcb_log_stop", "pcb_log_norms", "pcb_log_labels", "pcb_log_label_get",
           "pcb_log_jaccard", "pcb_verify_stats", "pcb_create_synthetic", "pcb_get_instance",
           "pcb_apply_g_exchange", "pcb_create_synthetic_box", "pcb_clone", "pcb_copy_state",
           "pcb_set_graph_after")


def lib():
    """Load the native library (raises NativeLibraryMissing if it is not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise NativeLibraryMissing(
                        "paracut_b200 native library not built (%s); run "
                        "`python -m paracut_b200.build`" % LIB_PATH)
                L = ctypes.CDLL(LIB_PATH)
                _declare(L)
                _lib = L
    return _lib


def check(rc):
    if rc == 0:
        return
    msg = lib().pcb_last_error().decode(errors="replace")
    if rc == PCB_E_ARG:
        raise ValueError(msg)
    if rc == PCB_E_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError("paracut_b200: %s (code %d)" % (msg, rc))


def ptr(a):
    return None if a is None else a.ctypes.data_as(P)


def device_count():
    c = INT(0)
    check(lib().pcb_device_count(ctypes.byref(c)))
    return int(c.value)


def release_memory(device=0):
    """Return the device memory destroyed handles left in the reuse pool."""
    check(lib().pcb_release_memory(int(device)))


def debug_counters(reset=True):
    """Sweep counters of a -DPCB_COUNT build (zeros in the normal build)."""
    out = np.zeros(8, dtype=np.uint64)
    check(lib().pcb_debug_counters(ptr(out), int(bool(reset))))
    return out


_HUGE_MIN = 32 << 20


def jaccard_packed(pa, pb):
    """1 - |A & B| / |A | B| of two packbits labelings (host popcount in the library)."""
    pa = np.ascontiguousarray(pa, dtype=np.uint8)
    pb = np.ascontiguousarray(pb, dtype=np.uint8)
    if pa.shape != pb.shape:
        raise ValueError("packed labelings differ in length")
    out = ctypes.c_double()
    check(lib().pcb_jaccard_packed(ptr(pa), ptr(pb), pa.size, ctypes.byref(out)))
    return out.value


def _host_empty(shape, dtype=np.float64):
    """Uninitialised host array for a large device read-back.

    Backed by an anonymous mapping advised for transparent huge pages, so the
    first-touch faults of the copy-out are 2 MB ones instead of 4 KB ones
    (fresh np.empty memory faults at ~20 GB/s on the B200 hosts).  Small
    arrays are plain np.empty.
    """
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dt.itemsize
    if nbytes < _HUGE_MIN:
        return np.empty(shape, dtype=dt)
    import mmap
    mm = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    if hasattr(mm, "madvise") and hasattr(mmap, "MADV_HUGEPAGE"):
        try:
            mm.madvise(mmap.MADV_HUGEPAGE)
        except OSError:
            pass
    return np.frombuffer(mm, dtype=dt).reshape(shape)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class GridSolver:
    """Owns one device-resident grid instance + AAR state (pcb_solver*)."""

    def __init__(self, g, precision="f64", device=0):
        if precision not in PRECISIONS:
            raise ValueError("precision must be one of %r" % (tuple(PRECISIONS),))
        L = lib()
        self.precision = precision
        self.device = int(device)
        self.dims = tuple(int(d) for d in g.dims)
        dims = np.asarray(self.dims, dtype=np.int64)
        if getattr(g, "_is_device_grid", False):
            # GPU-resident construction: the generator builds the instance in HBM
            h = P()
            cen = _f64(g.centres.reshape(-1))
            rad = _f64(g.radii)
            box = getattr(g, "box", None)
            if box is None:
                check(L.pcb_create_synthetic(ptr(dims), len(self.dims), CONN_CODES[g.connectivity],
                                             int(rad.size), ptr(cen), ptr(rad),
                                             ctypes.c_uint64(int(g.seed)), float(g.lam),
                                             int(bool(g.integer)), PRECISIONS[precision],
                                             self.device, ctypes.byref(h)))
            else:
                gd, org, ext, mask = box
                gd, org, ext = (np.asarray(v, dtype=np.int64) for v in (gd, org, ext))
                check(L.pcb_create_synthetic_box(ptr(gd), len(gd), CONN_CODES[g.connectivity],
                                                 ptr(org), ptr(ext), ptr(dims), int(mask),
                                                 int(rad.size), ptr(cen), ptr(rad),
                                                 ctypes.c_uint64(int(g.seed)), float(g.lam),
                                                 int(bool(g.integer)), PRECISIONS[precision],
                                                 self.device, ctypes.byref(h)))
            self._h = h
            r, n = INT(0), I64(0)
            check(L.pcb_shape(h, ctypes.byref(r), ctypes.byref(n)))
            self.r, self.n = int(r.value), int(n.value)
            return
        if getattr(g, "_is_grid_file", False):
            # device ingest: the payload goes file -> pinned staging -> HBM
            h = P()
            check(L.pcb_create_from_file(os.fsencode(g.path), PRECISIONS[precision],
                                         self.device, ctypes.byref(h), None, None, None))
            self._h = h
            r, n = INT(0), I64(0)
            check(L.pcb_shape(h, ctypes.byref(r), ctypes.byref(n)))
            self.r, self.n = int(r.value), int(n.value)
            return
        w = _f64(g.w)
        dws = [_f64(a) for a in g.dir_weights]
        arr = (P * 4)(*([ptr(a) for a in dws] + [None] * (4 - len(dws))))
        self._keep = (dims, w, dws)
        h = P()
        check(L.pcb_create(ptr(dims), len(self.dims), CONN_CODES[g.connectivity],
                           PRECISIONS[precision], ptr(w), arr, self.device, ctypes.byref(h)))
        self._keep = None
        self._h = h
        r, n = INT(0), I64(0)
        check(L.pcb_shape(h, ctypes.byref(r), ctypes.byref(n)))
        self.r, self.n = int(r.value), int(n.value)

    def clone(self, precision):
        """A handle of the same instance in another precision, built on the
        device from this handle's arrays (pcb_clone); no AAR state yet."""
        if precision not in PRECISIONS:
            raise ValueError("precision must be one of %r" % (tuple(PRECISIONS),))
        h = P()
        check(lib().pcb_clone(self.handle, PRECISIONS[precision], ctypes.byref(h)))
        other = GridSolver.__new__(GridSolver)
        other.precision, other.device, other.dims = precision, self.device, self.dims
        other._h, other.r, other.n = h, self.r, self.n
        return other

    def copy_state(self, src):
        """The fused-form AAR state of another f32 / f64s handle of the same
        instance, device to device (pcb_copy_state)."""
        check(lib().pcb_copy_state(self.handle, src.handle))

    # -- lifecycle
    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            lib().pcb_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        if not self._h:
            raise RuntimeError("solver handle is closed")
        return self._h

    # -- state
    def set_stream(self, stream_ptr):
        check(lib().pcb_set_stream(self.handle, int(stream_ptr)))

    def set_graph_after(self, iters):
        """Plain iterations replay as CUDA graphs once the handle has run
        ``iters`` of them eagerly (default 64; 0: from the first block)."""
        check(lib().pcb_set_graph_after(self.handle, int(iters)))

    def synchronize(self):
        check(lib().pcb_synchronize(self.handle))

    def init_cold(self):
        check(lib().pcb_init_cold(self.handle))

    def set_z(self, z):
        z = _f64(z)
        if z.shape != (self.r, self.n):
            raise ValueError("warm start shape %r, expected %r" % (z.shape, (self.r, self.n)))
        check(lib().pcb_set_z(self.handle, ptr(z)))

    def get_z(self):
        z = _host_empty((self.r, self.n))
        check(lib().pcb_get_z(self.handle, ptr(z)))
        return z

    def run(self, iters, norms=True):
        out = np.empty(max(int(iters), 1)) if norms else None
        check(lib().pcb_aar_run(self.handle, int(iters), ptr(out)))
        return out[:int(iters)] if norms else None

    def step(self, iters, flags, norms=True):
        """pcb_aar_step: fused iterations with sharding flags (STEP_*)."""
        out = np.empty(max(int(iters), 1)) if norms else None
        check(lib().pcb_aar_step(self.handle, int(iters), int(flags), ptr(out)))
        return out[:int(iters)] if norms else None

    def set_family_mask(self, mask):
        check(lib().pcb_set_family_mask(self.handle, int(mask)))

    def apply_g(self, g_dev_ptr):
        check(lib().pcb_apply_g(self.handle, int(g_dev_ptr)))

    def apply_g_exchange(self, recv_ptr, send_ptr, P, dz, cp):
        """g = G + received d_z, into the send buffer and applied (pcb_apply_g_exchange)."""
        check(lib().pcb_apply_g_exchange(self.handle, int(recv_ptr), int(send_ptr), int(P),
                                         int(dz), int(cp)))

    def set_owned(self, n_own):
        """Nodes [n_own, n) are halo copies owned by another shard (pcb_set_owned)."""
        check(lib().pcb_set_owned(self.handle, int(n_own)))

    def device_buffer(self, which):
        """(device pointer, element count) of a handle buffer (BUF_*)."""
        p_, n_ = ctypes.c_size_t(0), I64(0)
        check(lib().pcb_device_buffer(self.handle, int(which), ctypes.byref(p_), ctypes.byref(n_)))
        return int(p_.value), int(n_.value)

    def shadow(self, want_y=False, want_s=False):
        y = _host_empty((self.r, self.n)) if want_y else None
        s = _host_empty((self.n,)) if want_s else None
        check(lib().pcb_shadow(self.handle, ptr(y), ptr(s)))
        return y, s

    def shadow_get(self):
        y = _host_empty((self.r, self.n))
        check(lib().pcb_shadow_get(self.handle, ptr(y)))
        return y

    def shadow_delta(self):
        d = np.empty(1)
        check(lib().pcb_shadow_delta(self.handle, ptr(d)))
        return float(d[0])

    def apply(self, norm=True):
        """One AAR update from the current shadow; its step norm (None when
        norm=False: with the solve log on it is logged on the device)."""
        if not norm:
            check(lib().pcb_apply(self.handle, None))
            return None
        out = np.empty(1)
        check(lib().pcb_apply(self.handle, ptr(out)))
        return float(out[0])

    # ---- solve log (pcb_log_*): step norms and check labelings kept on the
    # device until the solve ends
    def log_start(self):
        check(lib().pcb_log_start(self.handle))

    def log_stop(self):
        check(lib().pcb_log_stop(self.handle))

    def log_norms(self):
        cnt = I64(0)
        check(lib().pcb_log_norms(self.handle, None, 0, ctypes.byref(cnt)))
        out = np.empty(max(int(cnt.value), 1))
        check(lib().pcb_log_norms(self.handle, ptr(out), int(cnt.value), ctypes.byref(cnt)))
        return out[:int(cnt.value)]

    def log_labels(self, t):
        """Append the current check's packed labels (threshold t); returns the slot."""
        slot = I64(0)
        check(lib().pcb_log_labels(self.handle, int(t), ctypes.byref(slot)))
        return int(slot.value)

    def log_label_get(self, slot):
        out = np.empty((self.n + 7) // 8, dtype=np.uint8)
        check(lib().pcb_log_label_get(self.handle, int(slot), ptr(out)))
        return out

    def log_jaccard(self, ref_packed, count):
        ref = np.ascontiguousarray(ref_packed, dtype=np.uint8)
        if ref.size != (self.n + 7) // 8:
            raise ValueError("packed reference has %d bytes, expected %d" % (ref.size, (self.n + 7) // 8))
        out = np.empty(max(int(count), 1))
        check(lib().pcb_log_jaccard(self.handle, ptr(ref), ptr(out), int(count)))
        return out[:int(count)]

    def check(self, thresholds):
        thr = _f64(thresholds)
        T = thr.size
        e, gp, d = np.empty(T), np.empty(T), np.empty(1)
        check(lib().pcb_check(self.handle, T, ptr(thr), ptr(e), ptr(gp), ptr(d)))
        return e, gp, float(d[0])

    def check_labels(self, t, packed=False):
        nb = (self.n + 7) // 8 if packed else self.n
        lab = np.empty(nb, dtype=np.uint8)
        check(lib().pcb_get_check(self.handle, int(t), ptr(lab), int(bool(packed)), None))
        return lab

    def check_x(self, t=0):
        x = _host_empty((self.n,))
        check(lib().pcb_get_check(self.handle, int(t), None, 0, ptr(x)))
        return x

    def keep_best(self, t):
        check(lib().pcb_keep_best(self.handle, int(t)))

    def get_best(self, labels=True, x=True, labels_out=None):
        """(labels uint8, x fp64) of the kept best iterate; either may be skipped (None).
        ``labels_out``: a uint8 host array of n entries to fill (e.g. one whose
        pages were touched while the device was busy)."""
        lab = None
        if labels:
            ok = (isinstance(labels_out, np.ndarray) and labels_out.dtype == np.uint8
                  and labels_out.shape == (self.n,) and labels_out.flags.c_contiguous)
            lab = labels_out if ok else _host_empty((self.n,), np.uint8)
        xv = _host_empty((self.n,)) if x else None
        check(lib().pcb_get_best(self.handle, ptr(lab) if labels else None,
                                 ptr(xv) if x else None))
        return lab, xv

    def scale_pairwise(self, factor):
        """Pairwise weights := factor * creation weights; AAR state kept."""
        check(lib().pcb_scale_pairwise(self.handle, float(factor)))

    def dual_init(self, alg, y0=None):
        """Start a BCD/AP/FISTA iterate (ALG_*) from y0 (r, n) or zeros."""
        ya = None
        if y0 is not None:
            ya = _f64(y0)
            if ya.shape != (self.r, self.n):
                raise ValueError("expected shape %r" % ((self.r, self.n),))
        check(lib().pcb_dual_init(self.handle, int(alg), ptr(ya)))

    def dual_run(self, iters, stop=False):
        """iters scheme iterations -> (monitor[iters], stop quantity[iters] or None)."""
        mon = np.empty(max(int(iters), 0))
        st = np.empty_like(mon) if stop else None
        check(lib().pcb_dual_run(self.handle, int(iters), ptr(mon), ptr(st)))
        return mon, st

    def level_set(self, x=None):
        """Best level set {x > u} of x (host array) or of the current check's x.

        Returns (u, energy); u = -inf for the all-ones labeling.
        """
        xa = None
        if x is not None:
            xa = _f64(x)
            if xa.shape != (self.n,):
                raise ValueError("length mismatch")
        u, e = ctypes.c_double(0.0), ctypes.c_double(0.0)
        check(lib().pcb_level_set(self.handle, ptr(xa), ctypes.byref(u), ctypes.byref(e)))
        return float(u.value), float(e.value)

    def project_K(self, v):
        v = _f64(v)
        if v.shape != (self.r, self.n):
            raise ValueError("expected shape %r" % ((self.r, self.n),))
        out = np.empty_like(v)
        check(lib().pcb_project_K(self.handle, ptr(v), ptr(out)))
        return out

    def set_profiling(self, on):
        check(lib().pcb_set_profiling(self.handle, int(bool(on))))

    def get_instance(self, connectivity):
        """(w, dir_weights) of the handle's instance, copied to the host."""
        from .graph import DIRECTIONS, direction_shape
        w = np.empty(self.n)
        dws = [np.empty(direction_shape(self.dims, d)) for d in DIRECTIONS[connectivity]]
        arr = (P * 4)(*([ptr(a) for a in dws] + [None] * (4 - len(dws))))
        check(lib().pcb_get_instance(self.handle, ptr(w), arr))
        return w, dws

    def verify_stats(self, scans=False):
        """(modes, verified sweeps, repaired chains[, scan sweeps, changed
        chains]) per family (pcb_verify_stats)."""
        modes = np.zeros(self.r, dtype=np.int32)
        out = [np.zeros(self.r, dtype=np.int64) for _ in range(4)]
        check(lib().pcb_verify_stats(self.handle, ptr(modes), *[ptr(a) for a in out]))
        return (modes, *out) if scans else (modes, out[0], out[1])

    def profile_read(self):
        ms = np.zeros(self.r)
        cnt = np.zeros(self.r, dtype=np.int64)
        check(lib().pcb_profile_read(self.handle, ptr(ms), ptr(cnt)))
        return ms, cnt

    def launch_count(self):
        return int(lib().pcb_launch_count(self.handle))

    def reset_launch_count(self):
        lib().pcb_reset_launch_count(self.handle)


def prox_chains(node_idx, chain_ptr, edge_w, c_lo, c_hi, v, out, as_projection, device=0):
    """GPU replacement of _kernels.prox_chains (in-place on ``out``)."""
    node_idx = np.ascontiguousarray(node_idx, dtype=np.int64)
    chain_ptr = np.ascontiguousarray(chain_ptr, dtype=np.int64)
    edge_w = _f64(edge_w)
    v = _f64(v)
    if out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a contiguous float64 array")
    check(lib().pcb_prox_chains(ptr(node_idx), ptr(chain_ptr),
                                ptr(edge_w) if edge_w.size else None, int(c_lo), int(c_hi),
                                v.size, node_idx.size, edge_w.size, ptr(v), ptr(out),
                                int(bool(as_projection)), int(device)))


def tv1d_batch(s, a, ptr_, device=0):
    s = _f64(s)
    a = _f64(a)
    ptr_ = np.ascontiguousarray(ptr_, dtype=np.int64)
    x = np.empty_like(s)
    check(lib().pcb_tv1d_prox_batch(ptr(s), ptr(a) if a.size else None, ptr(ptr_),
                                    ptr_.size - 1, ptr(x), int(device)))
    return x


def project_L_general(w, degree, support, v, device=0):
    """Pi_L for an arbitrary (hand-built) decomposition (projections.py:107-122)."""
    w = _f64(w)
    v = _f64(v)
    degree = np.ascontiguousarray(degree, dtype=np.int64)
    support = np.ascontiguousarray(support, dtype=np.uint8)
    r, n = v.shape
    out = np.empty_like(v)
    check(lib().pcb_project_L(ptr(w), ptr(degree), ptr(support), int(r), int(n), ptr(v),
                              ptr(out), int(device)))
    return out
