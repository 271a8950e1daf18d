"""Public weighted 1D-TV prox on the device (reference tv1d.py surface).

``tv1d_prox`` validates exactly like tv1d.py:42-69 and then runs the
taut-string kernel (bitwise equal to the reference on fp64 inputs);
``tv1d_prox_batch`` solves many independent signals in one launch.
``chain_dual_feasible`` is the reference's membership test (a checker, not
on the solver path).
"""
from __future__ import annotations

import numpy as np

from . import _native
from .decompose import Chain

DUAL_FEAS_TOL = 1e-9


def tv1d_prox(signal, weights):
    """argmin_x 0.5||x - signal||^2 + sum_i weights_i |x_{i+1} - x_i|."""
    s = np.ascontiguousarray(signal, dtype=np.float64)
    a = np.ascontiguousarray(weights, dtype=np.float64)
    if s.ndim != 1 or s.size == 0:
        raise ValueError("signal must be a nonempty 1D vector")
    m = s.size
    if a.shape != (m - 1,):
        raise ValueError("expected %d weights, got %r" % (m - 1, a.shape))
    if a.size and a.min() < 0:
        raise ValueError("weights must be nonnegative")
    return _native.tv1d_batch(s, a, np.array([0, m], dtype=np.int64))


def tv1d_prox_batch(signals, weights):
    """Prox of every (signal, weights) pair; lists in, list of arrays out."""
    sig = [np.ascontiguousarray(s, dtype=np.float64) for s in signals]
    wts = [np.ascontiguousarray(a, dtype=np.float64) for a in weights]
    if len(sig) != len(wts):
        raise ValueError("signals and weights differ in length")
    for s, a in zip(sig, wts):
        if s.ndim != 1 or s.size == 0:
            raise ValueError("signal must be a nonempty 1D vector")
        if a.shape != (s.size - 1,):
            raise ValueError("expected %d weights, got %r" % (s.size - 1, a.shape))
        if a.size and a.min() < 0:
            raise ValueError("weights must be nonnegative")
    if not sig:
        return []
    ptr = np.cumsum([0] + [s.size for s in sig]).astype(np.int64)
    x = _native.tv1d_batch(np.concatenate(sig),
                           np.concatenate(wts) if sum(a.size for a in wts) else np.zeros(0),
                           ptr)
    return [x[ptr[c]:ptr[c + 1]] for c in range(len(sig))]


def chain_dual_feasible(y, weights, tol=DUAL_FEAS_TOL):
    """|partial sums| <= weights and total 0, within tol (tv1d.py:72-88)."""
    y = np.asarray(y, dtype=np.float64)
    a = np.asarray(weights, dtype=np.float64)
    if y.ndim != 1 or y.size == 0 or a.shape != (y.size - 1,):
        raise ValueError("length mismatch")
    t = np.cumsum(y)
    if abs(t[-1]) > tol:
        return False
    if a.size == 0:
        return True
    return bool(np.all(np.abs(t[:-1]) <= a + tol))


__all__ = ["Chain", "tv1d_prox", "tv1d_prox_batch", "chain_dual_feasible", "DUAL_FEAS_TOL"]
