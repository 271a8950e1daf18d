"""Seeded synthetic grid instances for BASELINE.json's five configurations.

The reference ships no generator for these (its ``random_grid``,
``graph.py:271-277``, is uniform noise); BASELINE.json describes the images
only in words, so every unstated choice is fixed here and documented in
DESIGN.md ("Synthetic inputs"):

* RNG: ``numpy.random.default_rng(seed)``; draw order is all shape centres
  (uniform over the continuous box ``[0, dim)`` per axis), then all radii
  (uniform ``[rmin, rmax]``), then the iid N(0, 0.15^2) noise field in C order.
* Image: background 0.3; every node whose centre-distance is <= radius is
  set to 0.7 (later shapes overwrite earlier ones, which is a no-op because
  all shapes carry the same value).
* Unaries ``w = 10 (I - 0.5)``; pairwise ``lambda * exp(-(I_i - I_j)^2 /
  (2 * 0.1^2))`` per direction of ``DIRECTIONS``; 2D-8 diagonals scaled by
  ``1/sqrt(2)``.
* Integer variant: ``w = clip(rint(w), -10, 10)`` and
  ``a = rint(5 * lambda * exp(...))`` (numpy ``rint`` = round half to even).
* lambda path: ``GridEnergy.scaled_pairwise(lambda)`` of the lambda = 1
  instance (graph.py:182-187), warm-started with ``force_warm=True``.

Shape loops touch only each shape's bounding box, so a 4096^2 image with
128 disks or a 512^3 volume with 512 balls builds in seconds.
"""
from __future__ import annotations

import math
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


def synth_image(dims, shapes, rmin, rmax, seed):
    """Background 0.3, ``shapes`` disks/balls of value 0.7, plus N(0, 0.15^2)."""
    rng = np.random.default_rng(seed)
    dims = tuple(int(d) for d in dims)
    nd = len(dims)
    centres = rng.uniform(0.0, 1.0, size=(shapes, nd)) * np.asarray(dims, dtype=np.float64)
    radii = rng.uniform(rmin, rmax, size=shapes)
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
    img += rng.normal(0.0, SIGMA_NOISE, size=dims)
    return img


def energy_from_image(img, connectivity, lam=1.0, integer=False):
    """GridEnergy with the BASELINE.json unary/pairwise formulas."""
    dims = img.shape
    w = 10.0 * (img - 0.5)
    if integer:
        w = np.clip(np.rint(w), -10.0, 10.0)
    dw = []
    inv2s2 = 1.0 / (2.0 * SIGMA_EDGE * SIGMA_EDGE)
    for k, d in enumerate(DIRECTIONS[connectivity]):
        sa, sb = direction_slices(dims, d)
        diff = img[sa] - img[sb]
        a = np.exp(-(diff * diff) * inv2s2)
        if connectivity == "2D-8" and k >= 2:
            a = a * (1.0 / math.sqrt(2.0))
        if integer:
            a = np.rint(5.0 * lam * a)
        else:
            a = lam * a
        dw.append(np.ascontiguousarray(a))
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
