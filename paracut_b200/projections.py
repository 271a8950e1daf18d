"""Geometric operators Pi_K, Pi_L on the device (reference projections.py).

``project_K`` runs the fp64 chain-prox kernels (bitwise equal to the
reference's numba kernels); ``project_L`` runs the closed-form average on
the device.  Inside ``solve_aar`` neither is called: the fused sweep
kernels apply both per iteration.
"""
from __future__ import annotations

import numpy as np

from . import _native
from .decompose import ChainDecomposition, GridDecomposition


class DualState:
    """Solver dual variables y (in K), lam (in L), AAR point z (projections.py:28-44).

    Fields are (r, n) float64 arrays or None.  States returned by the B200
    solver keep y/z and the instance fingerprint on the device until first
    read (see ``solvers._DeviceDualState``); reading them gives plain arrays.
    """

    def __init__(self, y=None, lam=None, z=None, fingerprint=None):
        self.y = y
        self.lam = lam
        self.z = z
        self.fingerprint = fingerprint

    def copy(self):
        cp = lambda a: None if a is None else np.array(a, copy=True)
        return DualState(cp(self.y), cp(self.lam), cp(self.z), self.fingerprint)


class ChainPool:
    """Accepted for API compatibility (projections.py:47-86): the device kernels
    already run every chain of a family concurrently, so no host pool exists."""

    def __init__(self, threads=1):
        self.threads = max(1, int(threads))

    def run_class(self, cls, v, out, as_projection=True):
        if cls.num_chains:
            _native.prox_chains(cls.node_idx, cls.chain_ptr, cls.edge_w, 0, cls.num_chains,
                                v, out, as_projection)

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


_solver_cache = {}


def _grid_solver(dec):
    key = id(dec)
    ent = _solver_cache.get(key)
    if ent is None or ent[0] is not dec:
        _solver_cache.clear()
        ent = (dec, _native.GridSolver(dec.grid, precision="f64"))
        _solver_cache[key] = ent
    return ent[1]


def project_K(dec, v, pool=None):
    """out_j = Pi_{K_j}(v_j) = v_j - prox_{f_j}(v_j); 0 off the class support."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    if isinstance(dec, GridDecomposition):
        return _grid_solver(dec).project_K(v)
    out = np.zeros_like(v)
    for j, cls in enumerate(dec.classes):
        if cls.num_chains:
            _native.prox_chains(cls.node_idx, cls.chain_ptr, cls.edge_w, 0, cls.num_chains,
                                v[j], out[j], True)
    return out


def project_L(w, dec, v):
    """lam_j = (v_j + (w - sum_k v_k) / d) * support_j (projections.py:107-122)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    return _native.project_L_general(w, dec.degree, dec.support, v)


def reflect_K(dec, v, pool=None):
    return 2.0 * project_K(dec, v, pool) - v


def reflect_L(w, dec, v):
    return 2.0 * project_L(w, dec, v) - v


def aggregate(y):
    """s = sum_j y_j in class order (projections.py:133-137)."""
    y = np.asarray(y)
    if y.shape[0] == 0:
        return np.zeros(y.shape[1])
    return y.sum(axis=0)


__all__ = ["DualState", "ChainPool", "project_K", "project_L", "reflect_K", "reflect_L",
           "aggregate", "ChainDecomposition"]
