"""AAR solver driver on the B200 path (reference solvers.py surface).

``solve(g, dec, cfg)`` / ``solve_aar`` keep the reference's configuration,
result, trace, best-iterate, stopping and warm-start semantics
(solvers.py:33-209, 272-307); every iteration runs on the device:

* plain iterations between checks: ``pcb_aar_run`` (fused prox sweeps plus
  the reflect/average update, step norms accumulated on the device);
* check iterations: ``pcb_shadow`` (y = Pi_K(z)), ``pcb_check`` (threshold,
  cut, unary and dual reductions for up to 8 thresholds in one pass), then
  ``pcb_apply`` (z update from that shadow) if the loop continues.

Precision: ``SolverConfig.precision="f64"`` (default) keeps z in fp64 and
reproduces the reference iterates bit for bit; ``"f32"`` stores the bounded
shadows in fp32 with an fp64 drift vector (SURVEY 8(a) a6 fused form) and
computes every prox in fp64 -- the fast path for large grids; ``"f64s"`` is
that fused form with fp64 state and fp64 scans, chains split at merge points
(not bitwise, ~1e-12 relative to the reference) -- the fast fp64 path, and the
one for small grids whose few chains leave the bitwise kernel latency bound.

Extensions (defaults give the reference's behaviour): ``thresholds`` lists
extra primal thresholds evaluated in the same pass; each check keeps the
smallest-gap one (ties -> earlier entry), which certifies integer instances
with exact-zero plateaus; ``level_sets=True`` adds, at
every check, the best level set of x (best_level_set_gap, certify.py:50-65,
as one device sort), which is never worse than any threshold.

The other dual schemes ("bcd", "ap", "fista") run on the same exact fp64
kernels (``pcb_dual_init`` / ``pcb_dual_run``) with the reference's loop,
monitors and dual_tol rules; their iterates are bitwise the reference's.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .certify import jaccard_distance, jaccard_packed
from .decompose import ChainDecomposition, GridDecomposition
from .graph import as_grid, instance_fingerprint
from .projections import DualState

ALGORITHMS = ("bcd", "ap", "aar", "fista")
GAP_SLACK = 1e-6
PRECISIONS = ("f64", "f32", "f64s")
MAX_THRESHOLDS = 8


@dataclass
class SolverConfig:
    algorithm: str = "aar"
    max_iters: int = 20000
    gap_tol: float = 0.0
    dual_tol: float = 0.0
    threads: int = 1
    check_every: int = 10
    warm_start: DualState | None = None
    force_warm: bool = False
    reference: np.ndarray | None = None
    # --- B200 extensions
    precision: str = "f64"
    thresholds: tuple = (0.0,)
    device: int = 0
    polish_iters: int = 0   # f32 runs that end uncertified: up to this many f64 iterations
    polish_stall: int = 0   # f32: start the polish early once the best gap has not halved
                            # over this many checks (0: only at max_iters)
    polish_precision: str = "f64s"  # the polish's fp64 mode: "f64s" (fast split
                                    # kernels) or "f64" (bitwise reference kernels)
    polish_gap: float = 0.0  # f32 + polish_stall: stall only counts once the best gap is at
                             # most this (0: any gap), so a plateau far above the fp32
                             # noise floor keeps the cheaper f32 iterations going
    level_sets: bool = False  # each check also tries the best level set of x (on the device)

    def __post_init__(self):
        if self.algorithm not in ALGORITHMS:
            raise ValueError("unknown algorithm %r" % (self.algorithm,))
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.gap_tol < 0 or self.dual_tol < 0:
            raise ValueError("tolerances must be >= 0")
        if self.threads < 1 or self.check_every < 1:
            raise ValueError("threads and check_every must be >= 1")
        if self.polish_precision not in ("f64", "f64s"):
            raise ValueError("polish_precision must be 'f64' or 'f64s'")
        if self.precision not in PRECISIONS:
            raise ValueError("precision must be one of %r" % (PRECISIONS,))
        if self.polish_iters < 0 or self.polish_stall < 0 or self.polish_gap < 0:
            raise ValueError("polish_iters, polish_stall and polish_gap must be >= 0")
        thr = tuple(float(t) for t in self.thresholds)
        if not 1 <= len(thr) <= MAX_THRESHOLDS:
            raise ValueError("1..%d thresholds supported" % MAX_THRESHOLDS)
        if self.level_sets and len(thr) >= MAX_THRESHOLDS:
            raise ValueError("level_sets needs a free threshold slot (<= %d thresholds)"
                             % (MAX_THRESHOLDS - 1))
        self.thresholds = thr


@dataclass
class TraceRow:
    iteration: int
    gap: float
    dual_objective: float
    energy: float
    jaccard: float
    wall_s: float


@dataclass
class SolveResult:
    labeling: np.ndarray
    tv_solution: np.ndarray
    energy: float
    gap: float
    iterations: int
    certified: bool
    dual_state: DualState
    trace: list
    wall_time: float
    algorithm: str
    monitor: dict = field(default_factory=dict)
    threshold: float = 0.0   # primal threshold of the reported labeling (extension)


class _DeviceSolveResult(SolveResult):
    """SolveResult whose tv_solution (n fp64, the largest read-back) is copied
    from the device on first access; the handle that kept the best iterate is
    held until then.  Used only when that handle is private to the solve."""

    @property
    def tv_solution(self):
        if self._x is None and self._xsrc is not None:
            _, self._x = self._xsrc.get_best(labels=False, x=True)
            self._xsrc = None
        return self._x

    @tv_solution.setter
    def tv_solution(self, v):
        self._x = v
        if v is not None:
            self._xsrc = None


def threshold(x):
    """x_i > 0 -> 1, else 0 (strict; solvers.py:81-83)."""
    return (np.asarray(x) > 0).astype(np.uint8)


def level_sets(x):
    """Nested labelings thresholding x above each of its values (solvers.py:86-97)."""
    x = np.asarray(x, dtype=np.float64)
    labs = [np.ones(x.size, dtype=np.uint8)]
    for v in np.unique(x):
        labs.append((x > v).astype(np.uint8))
    return labs


class _DeviceDualState(DualState):
    """DualState whose y/z stay on the device until first read."""

    def __init__(self, solver, g):
        self._solver = solver
        self._g = g
        self._y = self._z = self._fp = None
        self.lam = None

    def _fetch(self):
        if self._solver is not None:
            self._y = self._solver.shadow_get()
            self._z = self._solver.get_z()
            self._solver = None

    @property
    def y(self):
        self._fetch()
        return self._y

    @y.setter
    def y(self, v):
        self._fetch()
        self._y = v

    @property
    def z(self):
        self._fetch()
        return self._z

    @z.setter
    def z(self, v):
        self._fetch()
        self._z = v

    @property
    def fingerprint(self):
        if self._fp is None and self._g is not None:
            self._fp = instance_fingerprint(self._g)
        return self._fp

    @fingerprint.setter
    def fingerprint(self, v):
        self._fp = v
        self._g = None


class _Driver:
    """Per-solve bookkeeping mirroring solvers.py:124-209."""

    def __init__(self, g, dec, cfg, solver=None):
        if not isinstance(dec, (GridDecomposition, ChainDecomposition)) or dec.n != g.n:
            raise ValueError("decomposition does not match the instance")
        if not isinstance(dec, GridDecomposition):
            raise ValueError("the B200 solver needs a grid decomposition (decompose_grid)")
        self.g = g
        self.cfg = cfg
        self.r = dec.r
        self.shape = (dec.r, g.n)
        self.trace = []
        self.monitor = {}
        self.best_gap = np.inf
        self.best_energy = np.nan
        self.best_t = 0
        self.best_thr = float(cfg.thresholds[0])
        self.best_packed = None
        self.iterations = 0
        self.stopped = False
        self._labs = []
        self.thr = np.asarray(cfg.thresholds, dtype=np.float64)
        self.owned = solver is None  # handles created here serve this solve only
        self.solver = (solver if solver is not None else
                       _native.GridSolver(g, precision=cfg.precision, device=cfg.device))
        self.best_solver = None
        self.kmax = cfg.max_iters
        self.stall = 0  # > 0: leave the loop once the best gap stalls for this many checks
        self._best_hist = []
        self.log = False  # solve log on the device (start_log)
        self._lab_buf = None  # the result's labeling, pages touched ahead (prefault_labels)
        self.t0 = time.perf_counter()

    def prefault_labels(self):
        """Allocate the result's label array and touch its pages now.  Called
        right after iterations were queued on the device, so the first-touch
        page faults (the larger part of the final read-back of a fresh array)
        run on the host while the device works."""
        if self._lab_buf is None:
            self._lab_buf = np.empty(self.g.n, dtype=np.uint8)
            self._lab_buf.fill(0)

    def start_log(self):
        """Keep step norms and check labelings on the device (pcb_log_*): a check
        cycle then syncs the host once, for the certificate it must act on."""
        self.log = True
        self.solver.log_start()

    def flush_norms(self):
        """Move the current handle's logged step norms into the monitor."""
        if self.log:
            self.record("aar_step_norm", self.solver.log_norms())
            self.solver.log_stop()

    def switch_solver(self, S):
        """Continue on another handle (fp64 polish), keeping the log going."""
        self.flush_norms()
        self.solver = S
        if self.log:
            S.log_start()

    def warm_or_cold(self):
        ws = self.cfg.warm_start
        if ws is None:
            self.solver.init_cold()
            return
        fp = instance_fingerprint(self.g)
        if ws.fingerprint is not None and ws.fingerprint != fp and not self.cfg.force_warm:
            raise ValueError("warm start fingerprint does not match instance")
        for name in ("z", "y"):
            v = getattr(ws, name, None)
            if v is not None:
                if v.shape != self.shape:
                    raise ValueError("warm start shape %r, expected %r" % (v.shape, self.shape))
                self.solver.set_z(np.asarray(v, dtype=np.float64))
                return
        self.solver.init_cold()

    def record(self, name, values):
        self.monitor.setdefault(name, []).extend(float(v) for v in np.atleast_1d(values))

    def check(self, k):
        thr = self.thr
        energies, gaps, dual = self.solver.check(thr)
        if self.cfg.level_sets:
            # best level set of this x (one device sort), certified by a second
            # pass of the same deterministic reductions as the thresholds
            u, _ = self.solver.level_set()
            if not np.any(thr == u):
                thr = np.append(thr, u)
                energies, gaps, dual = self.solver.check(thr)
        t = int(np.argmin(gaps))  # first minimum: threshold 0 wins ties
        gap, en = float(gaps[t]), float(energies[t])
        jac = np.nan
        packed = None
        if self.cfg.reference is not None:
            lab = self.solver.check_labels(t)
            jac = jaccard_distance(lab, self.cfg.reference)
        elif self.log:
            packed = (self.solver, self.solver.log_labels(t))
            self._labs.append(packed)
        else:
            packed = self.solver.check_labels(t, packed=True)
            self._labs.append(packed)
        self.trace.append(TraceRow(k, gap, dual, en, jac, time.perf_counter() - self.t0))
        if gap < self.best_gap:
            self.best_gap = gap
            self.best_energy = en
            self.best_t = t
            self.best_thr = float(thr[t])
            self.best_packed = packed
            self.solver.keep_best(t)
            self.best_solver = self.solver
        self.iterations = k
        if gap <= self.cfg.gap_tol + GAP_SLACK:
            self.stopped = True
        self._best_hist.append(self.best_gap)
        return self.stopped

    POLISH_NEAR = 10.0  # a best gap within this factor of the tolerance hands over at once

    def stalled(self):
        """The best gap has not halved over the last `stall` checks -- or it is
        already within POLISH_NEAR of the tolerance, where only the fp32
        state's noise floor can separate it from a certificate (cfg4: 1.3e-6
        against 1e-6), so waiting for the stall to show buys nothing."""
        h, w = self._best_hist, self.stall
        if w > 0 and h and h[-1] <= self.POLISH_NEAR * (self.cfg.gap_tol + GAP_SLACK):
            return True
        if w > 0 and self.cfg.polish_gap > 0 and not h[-1] <= self.cfg.polish_gap:
            return False
        return w > 0 and len(h) > w and not h[-1] <= 0.5 * h[-1 - w]

    def due(self, k):
        return k % self.cfg.check_every == 0 or k >= self.kmax

    def next_due(self, k):
        ce = self.cfg.check_every
        return min(((k // ce) + 1) * ce, self.kmax)

    def warm_y(self):
        """Warm-start iterate for the y-based schemes (warm_or("y"), solvers.py:150-165)."""
        ws = self.cfg.warm_start
        if ws is None:
            return None
        fp = instance_fingerprint(self.g)
        if ws.fingerprint is not None and ws.fingerprint != fp and not self.cfg.force_warm:
            raise ValueError("warm start fingerprint does not match instance")
        for name in ("y", "z"):
            v = getattr(ws, name, None)
            if v is not None:
                if v.shape != self.shape:
                    raise ValueError("warm start shape %r, expected %r" % (v.shape, self.shape))
                return np.asarray(v, dtype=np.float64)
        return None

    def finish(self, state=None):
        wall = time.perf_counter() - self.t0
        src = self.best_solver or self.solver
        lazy_x = self.owned  # no later solve reuses the handle: x on first access
        lab, x = src.get_best(labels=True, x=not lazy_x, labels_out=self._lab_buf)
        self._lab_buf = None
        certified = self.best_gap <= self.cfg.gap_tol + GAP_SLACK
        if self.cfg.reference is None and self.log:
            self.flush_norms()
            # jaccard against the best labeling, every logged slot of every
            # handle in one device pass each
            ref = self.best_packed[0].log_label_get(self.best_packed[1]) if self._labs else None
            jac = {}
            for h, _ in self._labs:
                if id(h) not in jac:
                    cnt = sum(1 for h2, _ in self._labs if h2 is h)
                    jac[id(h)] = h.log_jaccard(ref, cnt)
            for row, (h, slot) in zip(self.trace, self._labs):
                row.jaccard = float(jac[id(h)][slot])
        elif self.cfg.reference is None:
            for row, packed in zip(self.trace, self._labs):
                row.jaccard = jaccard_packed(packed, self.best_packed)
        elif self.log:
            self.flush_norms()
        if state is None:
            state = _DeviceDualState(self.solver, self.g)
        cls = _DeviceSolveResult if lazy_x else SolveResult
        res = cls(labeling=lab, tv_solution=x, energy=self.best_energy,
                  gap=self.best_gap, iterations=self.iterations, certified=certified,
                  dual_state=state, trace=self.trace, wall_time=wall,
                  algorithm=self.cfg.algorithm, monitor=self.monitor,
                  threshold=self.best_thr)
        if lazy_x:
            res._xsrc = src
        return res


def solve_aar(g, dec, cfg, _solver=None, _resident=False, _make64=None):
    """Averaged alternating reflections on the device (solvers.py:272-307).

    (_solver, _resident, _make64: used by solve_path to run on a resident
    instance whose AAR state continues from the previous solve.)"""
    if _solver is None:
        g = as_grid(g)
    drv = _Driver(g, dec, cfg, solver=_solver)
    if not _resident:
        drv.warm_or_cold()
    S = drv.solver
    k = 0
    if cfg.dual_tol > 0:
        have_prev = False
        while True:
            delta = S.shadow_delta()
            if drv.due(k) and drv.check(k):
                break
            if k >= cfg.max_iters:
                break
            drv.record("aar_step_norm", S.apply())
            k += 1
            if have_prev and delta <= cfg.dual_tol:
                S.shadow()
                drv.check(k)
                break
            have_prev = True
        return drv.finish()
    polish = cfg.precision == "f32" and cfg.polish_iters > 0
    if polish:
        drv.stall = cfg.polish_stall
    drv.start_log()
    k = _loop(drv, S, k)
    drv.stall = 0
    if polish and not drv.stopped:
        # fp32 state leaves a ~1e-5 floor on the discrete gap of large instances;
        # continue in fp64 (the split fast kernels by default) from the same
        # AAR point to certify
        # the polish handle is built from the f32 one on the device, and the
        # state moves over device to device (no host round trip)
        S64 = _make64() if _make64 is not None else S.clone(cfg.polish_precision)
        if cfg.polish_precision == "f64s":
            S64.copy_state(S)
        else:  # the bitwise kernels keep z_j themselves
            S64.set_z(S.get_z())
        drv.switch_solver(S64)
        drv.kmax = k + cfg.polish_iters
        drv.record("polish_start", k)
        # iteration k was just checked (its trace row stays): update first
        _loop(drv, S64, k, checked=k)
    return drv.finish()


def _loop(drv, S, k, checked=None):
    """Plain iterations between checks, shadow + certificate + update at checks.
    ``checked``: an iteration already certified (its check is not repeated)."""
    while True:
        if drv.due(k):
            S.shadow()
            if k != checked and (drv.check(k) or k >= drv.kmax or drv.stalled()):
                return k
            if drv.log:
                S.apply(norm=False)
            else:
                drv.record("aar_step_norm", S.apply())
            k += 1
        else:
            nxt = drv.next_due(k)
            if drv.log:
                S.run(nxt - k, norms=False)  # queued; the host is free until the next check
                drv.prefault_labels()
            else:
                drv.record("aar_step_norm", S.run(nxt - k))
            k = nxt


class _ScaledGrid:
    """g.scaled_pairwise(factor) without materialising it: structure for the
    decomposition, weights and fingerprint computed on first use."""

    def __init__(self, base, factor):
        self._base, self._factor = base, float(factor)
        self.dims, self.connectivity, self.n = tuple(base.dims), base.connectivity, base.n
        self._grid = None

    def _load(self):
        if self._grid is None:
            self._grid = self._base.scaled_pairwise(self._factor)
        return self._grid

    @property
    def w(self):
        return self._base.w

    @property
    def dir_weights(self):
        return self._load().dir_weights

    def tv(self, x):
        return self._load().tv(x)

    def energy(self, x):
        return self._load().energy(x)

    def _fingerprint(self):
        return instance_fingerprint(self._load())


def solve_path(g, lambdas, cfg, keep_states=True):
    """Warm-started lambda path on one resident device instance.

    Same results as the reference usage::

        res = None
        for lam in lambdas:
            res = solve(g.scaled_pairwise(lam), dec,
                        replace(cfg, warm_start=res and res.dual_state, force_warm=True))

    but the instance is uploaded once: each step rescales the pairwise
    weights on the device from the lambda = 1 copy (``pcb_scale_pairwise``)
    and the AAR state simply continues (the warm start, bitwise in f64).
    AAR only.  Returns the list of SolveResults; with ``keep_states=False``
    only the last one carries a dual state (the others skip the read-back).
    """
    import dataclasses
    if cfg.algorithm != "aar":
        raise ValueError("solve_path runs the AAR scheme")
    if cfg.dual_tol > 0:
        raise ValueError("solve_path: dual_tol stopping is not supported")
    g = as_grid(g)
    S = _native.GridSolver(g, precision=cfg.precision, device=cfg.device)
    out = []
    for i, lam in enumerate(lambdas):
        if lam < 0:
            raise ValueError("scale factor must be nonnegative")
        S.scale_pairwise(lam)
        gl = _ScaledGrid(g, lam)
        c = cfg if i == 0 else dataclasses.replace(cfg, warm_start=None, force_warm=True)

        def make64():  # S holds this lambda's weights: the clone copies them
            return S.clone(cfg.polish_precision)
        res = solve_aar(gl, GridDecomposition(gl), c, _solver=S, _resident=i > 0,
                        _make64=make64)
        if i + 1 < len(lambdas):  # the device state moves on: freeze this step's
            if keep_states:
                st = res.dual_state
                res.dual_state = DualState(y=st.y, z=st.z, fingerprint=st.fingerprint)
            else:
                res.dual_state = None
        out.append(res)
    return out


def _solve_dual(g, dec, cfg, alg, monitor_name):
    """Shared loop of the y-based schemes (solvers.py:219-243, 251-269, 318-341)."""
    if cfg.precision != "f64":
        raise ValueError("precision=%r: the fp32-state path is AAR-only" % (cfg.precision,))
    g = as_grid(g)
    drv = _Driver(g, dec, cfg)
    S = drv.solver
    S.dual_init(alg, drv.warm_y())
    k = 0
    stepped = False
    while True:
        if drv.due(k) and drv.check(k):
            break
        if k >= cfg.max_iters:
            break
        if cfg.dual_tol > 0:
            mon, stop = S.dual_run(1, stop=True)
            drv.record(monitor_name, mon)
            k += 1
            stepped = True
            if stop[0] <= cfg.dual_tol:
                drv.check(k)
                break
        else:
            nxt = drv.next_due(k)
            mon, _ = S.dual_run(nxt - k)
            drv.record(monitor_name, mon)
            k = nxt
            stepped = True
    lam = S.get_z() if (alg == _native.ALG_AP and stepped) else None
    state = DualState(y=S.shadow_get(), lam=lam, fingerprint=instance_fingerprint(g))
    return drv.finish(state)


def solve_bcd(g, dec, cfg):
    """Cyclic block projections y_j <- Pi_{K_j}(w - sum_{k != j} y_k) (solvers.py:212-243)."""
    return _solve_dual(g, dec, cfg, _native.ALG_BCD, "dual_objective")


def solve_ap(g, dec, cfg):
    """Alternating projections between K and L (solvers.py:246-269)."""
    return _solve_dual(g, dec, cfg, _native.ALG_AP, "ap_distance")


def solve_fista(g, dec, cfg):
    """Accelerated projected gradient on the smooth dual, step 1/r (solvers.py:310-341)."""
    return _solve_dual(g, dec, cfg, _native.ALG_FISTA, "dual_objective")

_SOLVERS = {"bcd": solve_bcd, "ap": solve_ap, "aar": solve_aar, "fista": solve_fista}


def solve(g, dec, cfg):
    """Dispatch on cfg.algorithm (solvers.py:348-350)."""
    return _SOLVERS[cfg.algorithm](g, dec, cfg)
