"""Seeded synthetic grid instances for BASELINE.json's five configurations.

The reference ships no generator for these (its ``random_grid``,
``graph.py:271-277``, is uniform noise); BASELINE.json describes the images
only in words, so every unstated choice is fixed here and documented in
DESIGN.md ("Synthetic inputs"):

* RNG: shape centres (uniform over the continuous box ``[0, dim)`` per axis),
  then radii (uniform ``[rmin, rmax]``) from ``numpy.random.default_rng(seed)``;
  the iid N(0, 0.15^2) noise field from a counter-based stream (``noise``:
  Philox-4x32-10 + inverse normal CDF), reproduced bit for bit by the device
  generator (``pcb_create_synthetic``).
* Image: background 0.3; every node whose centre-distance is <= radius is
  set to 0.7 (later shapes overwrite earlier ones, which is a no-op because
  all shapes carry the same value).
* Unaries ``w = 10 (I - 0.5)``; pairwise ``lambda * exp(-(I_i - I_j)^2 /
  (2 * 0.1^2))`` per direction of ``DIRECTIONS`` (exp by ``series_exp``);
  2D-8 diagonals scaled by ``1/sqrt(2)``.
* Integer variant: ``w = clip(rint(w), -10, 10)`` and
  ``a = rint(5 * lambda * exp(...))`` (numpy ``rint`` = round half to even).
* lambda path: ``GridEnergy.scaled_pairwise(lambda)`` of the lambda = 1
  instance (graph.py:182-187), warm-started with ``force_warm=True``.

Shape loops touch only each shape's bounding box, so a 4096^2 image with
128 disks or a 512^3 volume with 512 balls builds in seconds.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from .graph import DIRECTIONS, GridEnergy, direction_slices

SIGMA_NOISE = 0.15
SIGMA_EDGE = 0.1


@dataclass(frozen=True)
class InstanceSpec:
    name: str
    dims: tuple
    connectivity: str
    shapes: int
    rmin: float
    rmax: float
    iters: int
    dtype: str            # compute/storage precision the config names
    lam: float = 1.0
    integer: bool = False


# BASELINE.json "configs", in order.  cfg3's radius is unstated there; the
# survey's suggestion U[20,120] (same as cfg2) is used.
CONFIGS = {
    "cfg1": InstanceSpec("cfg1", (256, 256), "2D-4", 8, 10, 40, 200, "f64"),
    "cfg2": InstanceSpec("cfg2", (1024, 1024), "2D-4", 32, 20, 120, 500, "f32"),
    "cfg2_f64": InstanceSpec("cfg2_f64", (1024, 1024), "2D-4", 32, 20, 120, 500, "f64"),
    "cfg2_int": InstanceSpec("cfg2_int", (1024, 1024), "2D-4", 32, 20, 120, 500, "f64",
                             integer=True),
    "cfg3": InstanceSpec("cfg3", (4096, 4096), "2D-8", 128, 20, 120, 1000, "f32"),
    "cfg4": InstanceSpec("cfg4", (256, 256, 256), "3D-6", 64, 8, 40, 500, "f32"),
    "cfg5": InstanceSpec("cfg5", (512, 512, 512), "3D-6", 512, 8, 40, 300, "f32"),
    "cfg5_int": InstanceSpec("cfg5_int", (512, 512, 512), "3D-6", 512, 8, 40, 300, "f32",
                             integer=True),
}

LAMBDA_PATH = (0.25, 0.5, 1.0, 2.0, 4.0)


# ------------------------------------------------------------------ noise
#
# The N(0, 0.15^2) noise is a counter-based stream: node i's value comes from
# Philox-4x32-10 (Salmon et al., SC'11) at counter (i, 0, NOISE_STREAM, 0)
# under key = seed, turned into a 53-bit uniform u in (0, 1) and mapped through
# the inverse normal CDF (Wichura's AS241, PPND16).  Every step is integer
# arithmetic or IEEE-exact fp64 (+ - * / sqrt, frexp / ldexp / rint) in a
# fixed order -- log and exp are evaluated by the series below rather than by
# libm -- so the device generator (csrc/generator.cuh, built with
# -fmad=false) reproduces these arrays bit for bit, and any node can be
# generated independently.

NOISE_STREAM = 0x6E6F6973
_M0, _M1, _W0, _W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85
_U32 = np.uint64(0xFFFFFFFF)
LN2 = 0.6931471805599453
LN2_HI, LN2_LO = 6.93147180369123816490e-01, 1.90821492927058770002e-10
INV2S2 = 1.0 / (2.0 * SIGMA_EDGE * SIGMA_EDGE)
# PPND16 coefficients (Wichura 1988), numerator / denominator, lowest degree first
_PA = (3.3871328727963666080e0, 1.3314166789178437745e+2, 1.9715909503065514427e+3,
       1.3731693765509461125e+4, 4.5921953931549871457e+4, 6.7265770927008700853e+4,
       3.3430575583588128105e+4, 2.5090809287301226727e+3)
_PB = (1.0, 4.2313330701600911252e+1, 6.8718700749205790830e+2, 5.3941960214247511077e+3,
       2.1213794301586595867e+4, 3.9307895800092710610e+4, 2.8729085735721942674e+4,
       5.2264952788528545610e+3)
_PC = (1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0,
       3.64784832476320460504e0, 1.27045825245236838258e0, 2.41780725177450611770e-1,
       2.27238449892691845833e-2, 7.74545014278341407640e-4)
_PD = (1.0, 2.05319162663775882187e0, 1.67638483018380384940e0, 6.89767334985100004550e-1,
       1.48103976427480074590e-1, 1.51986665636164571966e-2, 5.47593808499534494600e-4,
       1.05075007164441684324e-9)
_PE = (6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0,
       2.96560571828504891230e-1, 2.65321895265761230930e-2, 1.24266094738807843860e-3,
       2.71155556874348757815e-5, 2.01033439929228813265e-7)
_PF = (1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1, 1.48753612908506148525e-2,
       7.86869131145613259100e-4, 1.84631831751005468180e-5, 1.42151175831644588870e-7,
       2.04426310338993978564e-15)


def _philox(c0, c1, c2, c3, k0, k1):
    """Philox-4x32-10 on uint64 arrays holding 32-bit words."""
    for rnd in range(10):
        if rnd:
            k0 = (k0 + _W0) & 0xFFFFFFFF
            k1 = (k1 + _W1) & 0xFFFFFFFF
        p0 = c0 * np.uint64(_M0)
        p1 = c2 * np.uint64(_M1)
        c0, c1, c2, c3 = ((p1 >> np.uint64(32)) ^ c1 ^ np.uint64(k0), p1 & _U32,
                          (p0 >> np.uint64(32)) ^ c3 ^ np.uint64(k1), p0 & _U32)
    return c0, c1, c2, c3


def _poly(c, r):
    v = c[7]
    for k in range(6, -1, -1):
        v = v * r + c[k]
    return v


def series_log(x):
    """log(x), x > 0: frexp reduction and the atanh series (IEEE ops only)."""
    m, e = np.frexp(x)
    small = m < 0.7071067811865476
    m = np.where(small, m * 2.0, m)
    e = np.where(small, e - 1, e).astype(np.float64)
    f = m - 1.0
    s = f / (2.0 + f)
    t = s * s
    P = 1.0 / 25.0
    for k in range(11, -1, -1):
        P = P * t + 1.0 / (2 * k + 1)
    return e * LN2 + 2.0 * s * P


def series_exp(x):
    """exp(x), x <= 0: ln 2 reduction and a degree-14 Taylor polynomial (0 below -700)."""
    x = np.asarray(x, dtype=np.float64)
    k = np.rint(x / LN2)
    r = (x - k * LN2_HI) - k * LN2_LO
    P = 1.0 / math.factorial(14)
    for n in range(13, -1, -1):
        P = P * r + 1.0 / math.factorial(n)
    return np.where(x < -700.0, 0.0, np.ldexp(P, np.where(x < -700.0, 0, k).astype(np.int64)))


def inverse_normal(u):
    """PPND16 (AS241): the standard normal quantile of u in (0, 1)."""
    q = u - 0.5
    r = 0.180625 - q * q
    central = q * _poly(_PA, r) / _poly(_PB, r)
    rr = np.sqrt(-series_log(np.where(q < 0, u, 1.0 - u)))
    r1 = rr - 1.6
    r2 = rr - 5.0
    tail = np.where(rr <= 5.0, _poly(_PC, r1) / _poly(_PD, r1), _poly(_PE, r2) / _poly(_PF, r2))
    tail = np.where(q < 0, -tail, tail)
    return np.where(np.abs(q) <= 0.425, central, tail)


def noise(seed, start, count):
    """N(0, 1) values of nodes [start, start + count) for `seed`."""
    return noise_at(seed, np.arange(start, start + count, dtype=np.uint64))


def noise_at(seed, i):
    """N(0, 1) values of the global node indices i (uint64 array) for `seed`."""
    i = np.asarray(i, dtype=np.uint64)
    count = i.size
    k0, k1 = int(seed) & 0xFFFFFFFF, (int(seed) >> 32) & 0xFFFFFFFF
    o0, o1, _, _ = _philox(i & _U32, i >> np.uint64(32),
                           np.full(count, NOISE_STREAM, np.uint64), np.zeros(count, np.uint64),
                           k0, k1)
    u = ((o0 >> np.uint64(5)).astype(np.float64) * 67108864.0
         + (o1 >> np.uint64(6)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)
    return inverse_normal(u)


def shapes_of(dims, shapes, rmin, rmax, seed):
    """Shape centres (uniform over the continuous box) then radii, from
    numpy default_rng(seed)."""
    rng = np.random.default_rng(seed)
    dims = tuple(int(d) for d in dims)
    centres = rng.uniform(0.0, 1.0, size=(shapes, len(dims))) * np.asarray(dims, dtype=np.float64)
    radii = rng.uniform(rmin, rmax, size=shapes)
    return centres, radii


def synth_image(dims, shapes, rmin, rmax, seed):
    """Background 0.3, ``shapes`` disks/balls of value 0.7, plus N(0, 0.15^2)."""
    dims = tuple(int(d) for d in dims)
    nd = len(dims)
    centres, radii = shapes_of(dims, shapes, rmin, rmax, seed)
    img = np.full(dims, 0.3, dtype=np.float64)
    for c, rad in zip(centres, radii):
        lo = [max(0, int(math.floor(c[a] - rad))) for a in range(nd)]
        hi = [min(dims[a], int(math.ceil(c[a] + rad)) + 1) for a in range(nd)]
        if any(h <= l for l, h in zip(lo, hi)):
            continue
        axes = [np.arange(l, h, dtype=np.float64) - c[a]
                for a, (l, h) in enumerate(zip(lo, hi))]
        d2 = np.zeros([h - l for l, h in zip(lo, hi)])
        for a, ax in enumerate(axes):
            shape = [1] * nd
            shape[a] = ax.size
            d2 = d2 + (ax * ax).reshape(shape)
        box = tuple(slice(l, h) for l, h in zip(lo, hi))
        sub = img[box]
        sub[d2 <= rad * rad] = 0.7
    flat = img.reshape(-1)
    _chunked(flat.size, lambda s0, cnt: flat.__setitem__(
        slice(s0, s0 + cnt), flat[s0:s0 + cnt] + SIGMA_NOISE * noise(seed, s0, cnt)))
    return img


def _chunked(n, fn, chunk=1 << 21):
    """fn(start, count) over [0, n) in chunks on host threads (numpy ufuncs
    release the GIL); chunks are independent, so the result does not depend
    on the thread count."""
    starts = list(range(0, n, chunk))
    if len(starts) <= 1:
        for s0 in starts:
            fn(s0, min(chunk, n - s0))
        return
    with ThreadPoolExecutor(max_workers=min(len(starts), os.cpu_count() or 1)) as ex:
        list(ex.map(lambda s0: fn(s0, min(chunk, n - s0)), starts))


def make_part(spec, seed, gdims, origin, extent, dims, dir_mask=0xF, lam=None):
    """Host reference of pcb_create_synthetic_box: the box [origin, origin +
    extent) of the global instance (gdims), as a GridEnergy of `dims` (the
    box's nodes in C order), with the box's internal edges of the directions
    in dir_mask and zero weights elsewhere.  Equals slicing make_instance."""
    if isinstance(spec, str):
        spec = CONFIGS[spec]
    gdims = tuple(int(d) for d in gdims)
    nd = len(gdims)
    centres, radii = shapes_of(gdims, spec.shapes, spec.rmin, spec.rmax, seed)
    ext = tuple(int(e) for e in extent)
    org = tuple(int(o) for o in origin)
    img = np.full(ext, 0.3, dtype=np.float64)
    for c, rad in zip(centres, radii):
        lo = [max(max(0, int(math.floor(c[a] - rad))), org[a]) for a in range(nd)]
        hi = [min(min(gdims[a], int(math.ceil(c[a] + rad)) + 1), org[a] + ext[a])
              for a in range(nd)]
        if any(h <= l for l, h in zip(lo, hi)):
            continue
        axes = [np.arange(l, h, dtype=np.float64) - c[a] for a, (l, h) in enumerate(zip(lo, hi))]
        d2 = np.zeros([h - l for l, h in zip(lo, hi)])
        for a, ax in enumerate(axes):
            shape = [1] * nd
            shape[a] = ax.size
            d2 = d2 + (ax * ax).reshape(shape)
        box = tuple(slice(l - o, h - o) for l, h, o in zip(lo, hi, org))
        sub = img[box]
        sub[d2 <= rad * rad] = 0.7
    flat = img.reshape(-1)

    def add_noise(s0, cnt):  # box flat index -> global node index, per chunk
        t = np.arange(s0, s0 + cnt, dtype=np.int64)
        gi = np.zeros(cnt, dtype=np.uint64)
        coords = []
        for a in range(nd - 1, -1, -1):
            coords.append(t % ext[a] + org[a])
            t = t // ext[a]
        for a, c in zip(range(nd), reversed(coords)):
            gi = gi * np.uint64(gdims[a]) + c.astype(np.uint64)
        flat[s0:s0 + cnt] += SIGMA_NOISE * noise_at(seed, gi)

    _chunked(flat.size, add_noise)
    full = energy_from_image(img, spec.connectivity, lam=spec.lam if lam is None else lam,
                             integer=spec.integer)
    dims = tuple(int(d) for d in dims)
    dws = []
    for k, (d, a) in enumerate(zip(DIRECTIONS[spec.connectivity], full.dir_weights)):
        shape = tuple(s - abs(o) for s, o in zip(dims, d))
        dws.append(a.reshape(shape) if (dir_mask >> k) & 1 else np.zeros(shape))
    return GridEnergy(dims, spec.connectivity, full.w, dws)


def energy_from_image(img, connectivity, lam=1.0, integer=False):
    """GridEnergy with the BASELINE.json unary/pairwise formulas."""
    dims = img.shape
    w = 10.0 * (img - 0.5)
    if integer:
        w = np.clip(np.rint(w), -10.0, 10.0)
    dw = []
    for k, d in enumerate(DIRECTIONS[connectivity]):
        sa, sb = direction_slices(dims, d)
        diff = np.ascontiguousarray(img[sa] - img[sb])
        a = np.empty_like(diff)
        fd, fa = diff.reshape(-1), a.reshape(-1)
        diag = connectivity == "2D-8" and k >= 2

        def edge(s0, cnt, fd=fd, fa=fa, diag=diag):
            dd = fd[s0:s0 + cnt]
            v = series_exp(-(dd * dd) * INV2S2)
            if diag:
                v = v * (1.0 / math.sqrt(2.0))
            fa[s0:s0 + cnt] = np.rint(5.0 * lam * v) if integer else lam * v

        _chunked(fd.size, edge)
        dw.append(a)
    return GridEnergy(dims, connectivity, np.ascontiguousarray(w.ravel()), dw)


def make_instance(spec, seed=0, lam=None, dims=None):
    """Build the GridEnergy for an InstanceSpec (optionally resized for tests)."""
    if isinstance(spec, str):
        spec = CONFIGS[spec]
    dims = tuple(dims) if dims is not None else spec.dims
    img = synth_image(dims, spec.shapes, spec.rmin, spec.rmax, seed)
    return energy_from_image(img, spec.connectivity,
                             lam=spec.lam if lam is None else lam,
                             integer=spec.integer)


def algorithmic_bytes(g, r, bytes_per_elem):
    """B = b * ((2r + 1) n + |E|) per AAR iteration."""
    nedges = sum(int(np.count_nonzero(a)) for a in g.dir_weights)
    return bytes_per_elem * ((2 * r + 1) * g.n + nedges)


class DeviceGrid:
    """A BASELINE instance generated in device memory (pcb_create_synthetic).

    ``GridSolver`` (and so ``solve``) builds its handle from it on the GPU --
    image, noise, unaries and edge weights never exist on the host; the arrays
    equal ``make_instance(spec, seed)`` bit for bit.  ``w``, ``dir_weights``,
    ``energy`` and the fingerprint copy the instance back on first use."""

    _is_device_grid = True

    def __init__(self, spec, seed=0, lam=None, dims=None, device=0):
        if isinstance(spec, str):
            spec = CONFIGS[spec]
        self.spec, self.seed = spec, int(seed)
        self.dims = tuple(int(d) for d in (dims if dims is not None else spec.dims))
        self.connectivity = spec.connectivity
        self.lam = spec.lam if lam is None else float(lam)
        self.integer = bool(spec.integer)
        self.device = int(device)
        self.centres, self.radii = shapes_of(self.dims, spec.shapes, spec.rmin, spec.rmax,
                                             self.seed)
        self.n = int(np.prod(self.dims))
        self._grid = None

    def part(self, origin, extent, dims, dir_mask=0xF):
        """The box [origin, origin + extent) as a device grid of `dims`
        (pcb_create_synthetic_box; a sharded rank's slab or pencil)."""
        return DeviceGridPart(self, origin, extent, dims, dir_mask)

    def load(self):
        """The instance with host arrays (generated on the device, copied back)."""
        if self._grid is None:
            from ._native import GridSolver
            S = GridSolver(self, precision="f32", device=self.device)  # (no fp64 hull spill)
            w, dws = S.get_instance(self.connectivity)
            S.close()
            self._grid = GridEnergy(self.dims, self.connectivity, w, dws)
        return self._grid

    @property
    def w(self):
        return self.load().w

    @property
    def dir_weights(self):
        return self.load().dir_weights

    @property
    def num_edges(self):
        return self.load().num_edges

    def tv(self, x):
        return self.load().tv(x)

    def energy(self, x):
        return self.load().energy(x)

    def edge_arrays(self):
        return self.load().edge_arrays()

    def scaled_pairwise(self, factor):
        return self.load().scaled_pairwise(factor)

    def _fingerprint(self):
        from .graph import instance_fingerprint
        return instance_fingerprint(self.load())


class DeviceGridPart(DeviceGrid):
    """A box of a DeviceGrid's global instance, generated on the device
    (equals make_part / slicing make_instance)."""

    def __init__(self, parent, origin, extent, dims, dir_mask=0xF):
        self.spec, self.seed = parent.spec, parent.seed
        self.connectivity, self.lam, self.integer = parent.connectivity, parent.lam, parent.integer
        self.device = parent.device
        self.centres, self.radii = parent.centres, parent.radii
        self.dims = tuple(int(d) for d in dims)
        self.n = int(np.prod(self.dims))
        self.box = (tuple(parent.dims), tuple(int(o) for o in origin),
                    tuple(int(e) for e in extent), int(dir_mask))
        self._grid = None


class HostPartsGrid(DeviceGrid):
    """Like DeviceGrid for a sharded run, but each rank's slab and pencil are
    generated on the host (make_part) and uploaded: the rank holds host arrays
    of its own part only, never of the whole instance."""

    def part(self, origin, extent, dims, dir_mask=0xF):
        key = (tuple(origin), tuple(extent), tuple(dims), int(dir_mask))
        cache = self.__dict__.setdefault("_parts", {})
        if key not in cache:  # built once: a rank's host-side input arrays
            cache[key] = make_part(self.spec, self.seed, self.dims, origin, extent, dims,
                                   dir_mask, lam=self.lam)
        return cache[key]
