"""Grid cut instances: the data the B200 path consumes.

Mirrors the reference energy model (``graph.py:116-213``) for the grid case
only, which is all the AAR hot path uses:

    E(x) = sum_{ij} a_ij |x_i - x_j| - sum_i w_i x_i,   a_ij >= 0,

with nodes in C order of ``dims`` and one dense weight array per edge
direction (``DIRECTIONS``; zero entries are absent edges).  Differences from
the reference are deliberate and do not change any value:

* the flat, lexsorted edge list (``graph.py:152-161``, 13 s at 4096^2 2D-8)
  is built lazily, only if ``edge_arrays()`` is called;
* ``tv``/``energy`` keep the reference's per-direction formula so host-side
  certificates agree with it to rounding.

``instance_fingerprint`` reproduces ``graph.py:195-213`` byte for byte, so a
``DualState`` saved by either implementation warm-starts the other.
"""
from __future__ import annotations

import hashlib

import numpy as np

CONNECTIVITIES = ("2D-4", "2D-8", "3D-6")

# Offsets per connectivity; line directions first (fastest axis first), then
# the two 2D diagonals.  Same order as graph.py:24-28 and the file format.
DIRECTIONS = {
    "2D-4": ((0, 1), (1, 0)),
    "2D-8": ((0, 1), (1, 0), (1, 1), (1, -1)),
    "3D-6": ((0, 0, 1), (0, 1, 0), (1, 0, 0)),
}


def direction_shape(dims, d):
    return tuple(int(s) - abs(int(k)) for s, k in zip(dims, d))


def direction_slices(dims, d):
    """(sa, sb): grid[sa] and grid[sb] are the two ends of every d-edge."""
    sa, sb = [], []
    for s, k in zip(dims, d):
        if k >= 0:
            sa.append(slice(0, s - k))
            sb.append(slice(k, s))
        else:
            sa.append(slice(-k, s))
            sb.append(slice(0, s + k))
    return tuple(sa), tuple(sb)


class GridEnergy:
    """Binary cut energy on a 2D/3D grid (reference ``GridEnergy`` surface)."""

    def __init__(self, dims, connectivity, w, dir_weights):
        if connectivity not in CONNECTIVITIES:
            raise ValueError("unsupported connectivity %r" % (connectivity,))
        dims = tuple(int(s) for s in dims)
        dirs = DIRECTIONS[connectivity]
        if len(dims) != len(dirs[0]):
            raise ValueError("dims rank does not match connectivity")
        if any(s < 1 for s in dims):
            raise ValueError("dims must be positive")
        n = int(np.prod(dims))
        w = np.ascontiguousarray(w, dtype=np.float64)
        if w.shape != (n,):
            raise ValueError("w length must equal product of dims")
        if len(dir_weights) != len(dirs):
            raise ValueError("expected %d direction arrays" % len(dirs))
        arrs = []
        for d, arr in zip(dirs, dir_weights):
            arr = np.ascontiguousarray(arr, dtype=np.float64)
            want = direction_shape(dims, d)
            if arr.shape != want:
                raise ValueError("direction %r weights must have shape %r" % (d, want))
            if arr.size and np.any(arr < 0):
                raise ValueError("edge weights must be nonnegative")
            arrs.append(arr)
        self.dims = dims
        self.connectivity = connectivity
        self.w = w
        self.dir_weights = arrs
        self._edges = None

    @property
    def n(self):
        return self.w.size

    @property
    def num_edges(self):
        return int(sum(np.count_nonzero(a) for a in self.dir_weights))

    def edge_arrays(self):
        """Sorted (i, j, a) with i < j, a > 0 -- built on first use only."""
        if self._edges is None:
            grid = np.arange(self.n, dtype=np.int64).reshape(self.dims)
            ei, ej, ea = [], [], []
            for d, arr in zip(DIRECTIONS[self.connectivity], self.dir_weights):
                sa, sb = direction_slices(self.dims, d)
                a, b = grid[sa].ravel(), grid[sb].ravel()
                keep = arr.ravel() > 0.0
                ei.append(np.minimum(a, b)[keep])
                ej.append(np.maximum(a, b)[keep])
                ea.append(arr.ravel()[keep])
            ei = np.concatenate(ei) if ei else np.zeros(0, np.int64)
            ej = np.concatenate(ej) if ej else np.zeros(0, np.int64)
            ea = np.concatenate(ea) if ea else np.zeros(0)
            order = np.lexsort((ej, ei))
            self._edges = (ei[order], ej[order], ea[order])
        return self._edges

    def direction_pairs(self, k):
        grid = np.arange(self.n, dtype=np.int64).reshape(self.dims)
        sa, sb = direction_slices(self.dims, DIRECTIONS[self.connectivity][k])
        return grid[sa].ravel(), grid[sb].ravel()

    def tv(self, x):
        """f(x) = sum a_ij |x_i - x_j|, per-direction like graph.py:169-180."""
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError("length mismatch")
        xg = x.reshape(self.dims)
        total = 0.0
        for d, arr in zip(DIRECTIONS[self.connectivity], self.dir_weights):
            if arr.size == 0:
                continue
            sa, sb = direction_slices(self.dims, d)
            total += float((np.abs(xg[sa] - xg[sb]) * arr).sum())
        return total

    def energy(self, x):
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError("length mismatch")
        return self.tv(x) - float(self.w @ x)

    def scaled_pairwise(self, factor):
        """The lambda-path instance: every a_ij times ``factor``."""
        if factor < 0:
            raise ValueError("scale factor must be nonnegative")
        return GridEnergy(self.dims, self.connectivity, self.w.copy(),
                          [a * factor for a in self.dir_weights])


def energy(g, x):
    """E(x) = f(x) - w.x for binary x."""
    return g.energy(x)


def tv_value(g, x):
    return g.tv(x)


def instance_fingerprint(g):
    """sha256 over topology + pairwise weights (unaries excluded), as graph.py:195-213."""
    fp = getattr(g, "_fingerprint", None)
    if callable(fp):  # file-backed grids hash the payload without loading it
        return fp()
    h = hashlib.sha256()
    if hasattr(g, "dims"):
        h.update(("grid:%s:%r" % (g.connectivity, tuple(g.dims))).encode())
        for arr in g.dir_weights:
            h.update(np.ascontiguousarray(arr, dtype=np.float64).tobytes())
    else:
        h.update(("cut:%d" % g.n).encode())
        h.update(np.ascontiguousarray(g.edge_i, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(g.edge_j, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(g.edge_a, dtype=np.float64).tobytes())
    return h.hexdigest()


def as_grid(g):
    """Accept our GridEnergy or any object with the reference's grid fields."""
    if (isinstance(g, GridEnergy) or getattr(g, "_is_grid_file", False)
            or getattr(g, "_is_device_grid", False)):
        return g
    for attr in ("dims", "connectivity", "w", "dir_weights"):
        if not hasattr(g, attr):
            raise ValueError("the B200 path needs a grid instance (dims, "
                             "connectivity, w, dir_weights)")
    return GridEnergy(g.dims, g.connectivity, g.w, g.dir_weights)


class CutInstance:
    """General (non-grid) cut instance, host only (reference graph.py:42-113).

    The device path needs a grid; this class carries DIMACS instances through
    the file formats and the small verification helpers.  Edges are stored
    sorted by (i, j), i < j, positive weights only; duplicates are rejected.
    """

    def __init__(self, w, edges):
        self.w = np.ascontiguousarray(w, dtype=np.float64)
        if self.w.ndim != 1 or self.w.size < 1:
            raise ValueError("w must be a nonempty 1D vector")
        n = self.w.size
        if len(edges) == 0:
            e = np.zeros((0, 3))
        else:
            e = np.asarray(edges, dtype=np.float64).reshape(-1, 3)
        i, j, a = e[:, 0].astype(np.int64), e[:, 1].astype(np.int64), np.ascontiguousarray(e[:, 2])
        if np.any(a < 0):
            raise ValueError("edge weights must be nonnegative")
        lo, hi = np.minimum(i, j), np.maximum(i, j)
        if np.any(lo < 0) or np.any(hi >= n) or np.any(lo == hi):
            raise ValueError("edge endpoints out of bounds or self-loop")
        pos = a > 0.0
        lo, hi, a = lo[pos], hi[pos], a[pos]
        order = np.lexsort((hi, lo))
        self.edge_i = np.ascontiguousarray(lo[order])
        self.edge_j = np.ascontiguousarray(hi[order])
        self.edge_a = np.ascontiguousarray(a[order])
        if self.edge_i.size > 1:
            same = (self.edge_i[1:] == self.edge_i[:-1]) & (self.edge_j[1:] == self.edge_j[:-1])
            if np.any(same):
                raise ValueError("duplicate edges")

    @property
    def n(self):
        return self.w.size

    @property
    def num_edges(self):
        return self.edge_i.size

    def edge_arrays(self):
        return self.edge_i, self.edge_j, self.edge_a

    def tv(self, x):
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError("length mismatch")
        if self.edge_i.size == 0:
            return 0.0
        return float(np.abs(x[self.edge_i] - x[self.edge_j]) @ self.edge_a)

    def energy(self, x):
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError("length mismatch")
        return self.tv(x) - float(self.w @ x)

    def scaled_pairwise(self, factor):
        if factor < 0:
            raise ValueError("scale factor must be nonnegative")
        return CutInstance(self.w.copy(), np.column_stack([self.edge_i, self.edge_j,
                                                           self.edge_a * factor]))
