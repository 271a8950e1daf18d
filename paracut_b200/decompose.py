"""Chain decompositions (reference ``decompose.py`` surface).

On the B200 path a grid decomposition is *structural*: every family is a
regular set of lines (rows/columns, 3D axis lines) or 2D-8 zig-zag paths,
and the device kernels derive chain membership from indices
(``node(c, i)``).  Zero-weight edges split chains
on the fly inside the prox kernel exactly where the reference splits them
(decompose.py:101-139), and zig-zag border nodes are edgeless singletons
(decompose.py:153-183), so degree = r on every node.

``GridDecomposition.classes`` materialises the reference's CSR
``ChainClass`` objects lazily, for callers that inspect them; the solver
never needs them.  ``ChainClass``/``ChainDecomposition`` also accept
hand-built CSR decompositions (``project_K``/``project_L`` then run the
CSR kernel ``pcb_prox_chains``).
"""
from __future__ import annotations

import numpy as np

from .graph import GridEnergy, as_grid

FAMILY_NAMES = {
    "2D-4": ("rows", "cols"),
    "2D-8": ("rows", "cols", "zigzag0", "zigzag1"),
    "3D-6": ("x", "y", "z"),
}


class Chain:
    """A weighted path: node ids plus one nonnegative weight per edge (tv1d.py:23-39)."""

    def __init__(self, node_ids, weights):
        self.node_ids = np.ascontiguousarray(node_ids, dtype=np.int64)
        self.weights = np.ascontiguousarray(weights, dtype=np.float64)
        if self.node_ids.ndim != 1 or self.node_ids.size < 1:
            raise ValueError("chain needs at least one node")
        if self.weights.shape != (self.node_ids.size - 1,):
            raise ValueError("need exactly one weight per chain edge")
        if np.unique(self.node_ids).size != self.node_ids.size:
            raise ValueError("chain nodes must be distinct")
        if self.weights.size and self.weights.min() < 0:
            raise ValueError("chain weights must be nonnegative")

    def __len__(self):
        return self.node_ids.size


class ChainClass:
    """Vertex-disjoint chains of one class in CSR form (decompose.py:29-80)."""

    def __init__(self, n, node_idx, chain_ptr, edge_w):
        self.n = int(n)
        self.node_idx = np.ascontiguousarray(node_idx, dtype=np.int64)
        self.chain_ptr = np.ascontiguousarray(chain_ptr, dtype=np.int64)
        self.edge_w = np.ascontiguousarray(edge_w, dtype=np.float64)
        self.support = np.zeros(self.n, dtype=bool)
        self.support[self.node_idx] = True

    @property
    def num_chains(self):
        return self.chain_ptr.size - 1

    @property
    def num_edges(self):
        return self.edge_w.size

    @property
    def chains(self):
        out = []
        for c in range(self.num_chains):
            b, e = self.chain_ptr[c], self.chain_ptr[c + 1]
            out.append(Chain(self.node_idx[b:e], self.edge_w[b - c:e - c - 1]))
        return out

    def _seam_mask(self):
        keep = np.ones(max(self.node_idx.size - 1, 0), dtype=bool)
        if self.num_chains > 1:
            keep[self.chain_ptr[1:-1] - 1] = False
        return keep

    def tv(self, x):
        if self.node_idx.size < 2:
            return 0.0
        dw = np.zeros(self.node_idx.size - 1)
        dw[self._seam_mask()] = self.edge_w
        return float(np.abs(np.diff(np.asarray(x)[self.node_idx])) @ dw)

    def edge_pairs(self):
        if self.num_chains == 0:
            return (np.zeros(0, np.int64), np.zeros(0, np.int64), self.edge_w)
        keep = self._seam_mask()
        return self.node_idx[:-1][keep], self.node_idx[1:][keep], self.edge_w


class ChainDecomposition:
    """f = sum_j f_j over r CSR classes (decompose.py:83-98)."""

    def __init__(self, n, classes):
        self.n = int(n)
        self.classes = list(classes)
        self.support = (np.stack([c.support for c in self.classes]) if self.classes
                        else np.zeros((0, self.n), dtype=bool))
        self.degree = self.support.sum(axis=0).astype(np.int64)

    @property
    def r(self):
        return len(self.classes)

    def tv(self, x):
        return sum(c.tv(x) for c in self.classes)


def _csr_from_lines(n, nodes, wts, leftover=None):
    nodes = np.asarray(nodes, dtype=np.int64)
    wts = np.asarray(wts, dtype=np.float64)
    ptr = [np.zeros(1, np.int64)]
    edge_w = np.zeros(0)
    if nodes.size:
        nl, L = nodes.shape
        starts = np.arange(1, nl, dtype=np.int64) * L
        if L > 1:
            zr, zc = np.nonzero(wts == 0.0)
            cuts = zr * L + zc + 1
            edge_w = wts[wts != 0.0]
        else:
            cuts = np.zeros(0, np.int64)
        ptr.append(np.append(np.union1d(starts, cuts), nl * L).astype(np.int64))
    idx = [nodes.ravel()]
    if leftover is not None and len(leftover):
        single = np.asarray(leftover, dtype=np.int64)
        idx.append(single)
        ptr.append(nodes.size + 1 + np.arange(single.size, dtype=np.int64))
    return ChainClass(n, np.concatenate(idx), np.concatenate(ptr), edge_w)


class GridDecomposition(ChainDecomposition):
    """Structural decomposition of a grid instance (what the kernels consume)."""

    def __init__(self, g):
        self.grid = g
        self.n = g.n
        self.connectivity = g.connectivity
        self.dims = tuple(g.dims)
        self.families = FAMILY_NAMES[g.connectivity]
        self._classes = None

    @property
    def r(self):
        return len(self.families)

    @property
    def degree(self):
        return np.full(self.n, self.r, dtype=np.int64)

    @property
    def support(self):
        return np.ones((self.r, self.n), dtype=bool)

    @property
    def classes(self):
        """Reference-layout CSR classes, built on first access (not used by the solver)."""
        if self._classes is None:
            self._classes = _materialise(self.grid)
        return self._classes

    def tv(self, x):
        return self.grid.tv(x)


def _line(g, axis, k):
    grid = np.arange(g.n, dtype=np.int64).reshape(g.dims)
    L = g.dims[axis]
    nodes = np.moveaxis(grid, axis, -1).reshape(-1, L)
    wm = (np.zeros((nodes.shape[0], 0)) if L < 2
          else np.moveaxis(g.dir_weights[k], axis, -1).reshape(-1, L - 1))
    return _csr_from_lines(g.n, nodes, wm)


def _zigzag(g, phase):
    H, W = g.dims
    if H < 2 or W < 2:
        return _csr_from_lines(g.n, np.zeros((0, 0), np.int64), np.zeros((0, 0)),
                               leftover=np.arange(g.n))
    cols = np.arange(W, dtype=np.int64)
    par = cols % 2
    base = np.arange(H - 1, dtype=np.int64)[:, None]
    rows = base + par[None, :] if phase == 0 else base + 1 - par[None, :]
    nodes = rows * W + cols[None, :]
    even = ((cols[:-1] % 2) == 0)[None, :]
    d1, d2 = g.dir_weights[2], g.dir_weights[3]
    wm = np.where(even, d1, d2) if phase == 0 else np.where(even, d2, d1)
    cov = np.zeros(g.n, dtype=bool)
    cov[nodes.ravel()] = True
    return _csr_from_lines(g.n, nodes, wm, leftover=np.flatnonzero(~cov))


def _materialise(g):
    if g.connectivity == "2D-4":
        return [_line(g, 1, 0), _line(g, 0, 1)]
    if g.connectivity == "2D-8":
        return [_line(g, 1, 0), _line(g, 0, 1), _zigzag(g, 0), _zigzag(g, 1)]
    return [_line(g, 2, 0), _line(g, 1, 1), _line(g, 0, 2)]


def decompose_grid(g):
    """Chain decomposition of a grid energy (decompose.py:186-200)."""
    if not isinstance(g, GridEnergy):
        try:
            g = as_grid(g)
        except ValueError:
            raise ValueError("chain decomposition requires a grid instance")
    return GridDecomposition(g)


def validate(dec, g, rng=None, report=None):
    """Decomposition invariants against the grid (decompose.py:203-260 checks).

    Every class partitions the nodes, the chain edges of all classes are the
    grid's positive edges exactly once with their weights, and
    sum_j f_j(x) = f(x) on random vectors (relative 1e-10).  Returns a bool;
    diagnostics go to ``report`` (a list) when given.
    """
    problems = []
    lo_all, hi_all, a_all = [], [], []
    for k, cls in enumerate(dec.classes):
        if np.unique(cls.node_idx).size != cls.node_idx.size:
            problems.append("class %d: chains share a vertex" % k)
        if cls.node_idx.size != g.n:
            problems.append("class %d: chains do not partition every node" % k)
        ei, ej, ea = cls.edge_pairs()
        if ea.size and ea.min() <= 0:
            problems.append("class %d: nonpositive chain edge weight" % k)
        lo_all.append(np.minimum(ei, ej))
        hi_all.append(np.maximum(ei, ej))
        a_all.append(np.asarray(ea, dtype=np.float64))
    lo = np.concatenate(lo_all) if lo_all else np.zeros(0, np.int64)
    hi = np.concatenate(hi_all) if hi_all else np.zeros(0, np.int64)
    a = np.concatenate(a_all) if a_all else np.zeros(0)
    order = np.lexsort((hi, lo))
    lo, hi, a = lo[order], hi[order], a[order]
    if lo.size > 1 and np.any((lo[1:] == lo[:-1]) & (hi[1:] == hi[:-1])):
        problems.append("an edge appears in more than one chain")
    gi, gj, ga = g.edge_arrays()
    if lo.size != gi.size or not (np.array_equal(lo, gi) and np.array_equal(hi, gj)):
        problems.append("chain edges do not match the grid edges")
    elif not np.array_equal(a, ga):
        problems.append("chain edge weights altered")
    rng = np.random.default_rng(0) if rng is None else rng
    for _ in range(3):
        x = rng.normal(size=g.n)
        f, fj = g.tv(x), sum(c.tv(x) for c in dec.classes)
        if abs(f - fj) > 1e-10 * max(1.0, abs(f)):
            problems.append("sum of class TVs %r differs from f(x) %r" % (fj, f))
            break
    if report is not None:
        report.extend(problems)
    return not problems
