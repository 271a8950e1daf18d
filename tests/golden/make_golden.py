"""Generate golden fixtures by running the REFERENCE implementation itself.

Run here (the container that has /root/reference); the GPU box never reads
/root/reference, it only reads the committed .npz files this script writes:

    python tests/golden/make_golden.py

The reference package is copied to a scratch dir under /tmp first and numba's
cache is redirected there, so nothing is ever written under /root/reference.

Fixtures (all float64, reference dtype):

* tv1d.npz     -- 360 chains in five weight regimes (restating the regimes
                  of pkg/tests/gen.py:26-42) plus long chains; s, a, CSR ptr,
                  x = paracut.tv1d_prox(s, a)  (tv1d.py:42-69).
* aar_*.npz    -- fixed-iteration AAR (solvers.py:272-307) on small grids of
                  every connectivity, real and integer weights, degenerate
                  dims: instance arrays and, per k, z^k, y^k = Pi_K(z^k), the
                  monitor aar_step_norm and the reference gap/energy at k.
* solve_*.npz  -- full gap-stopped solves (check_every 5, gap_tol 1e-6):
                  iterations, certified, energy, labeling, trace.
* cfg1.npz     -- BASELINE cfg1 (256^2 2D-4, seed 0) at k = 200.
* eps_int.npz  -- integer instance: reference discrete_gap at thresholds
                  0, +-1e-6 on the k = 400 iterate, plus maxflow_mincut energy.
* kat.npz      -- the frozen brute-force KAT of pkg/tests/test_oracle.py:60-68.
"""
from __future__ import annotations

import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src/paracut"


def import_reference():
    sys.dont_write_bytecode = True
    scratch = os.path.join(tempfile.gettempdir(), "paracut_ref_golden")
    os.makedirs(scratch, exist_ok=True)
    dst = os.path.join(scratch, "paracut")
    if os.path.exists(dst):
        shutil.rmtree(dst)
    shutil.copytree(REF_SRC, dst, ignore=shutil.ignore_patterns("__pycache__"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(scratch, "numba_cache"))
    sys.path.insert(0, scratch)
    import paracut  # noqa: E402
    return paracut


def chain_regimes(rng, count, m_max=50):
    """Five weight regimes (uniform, half zeros, huge, integer ties, near-critical)."""
    out = []
    for t in range(count):
        m = int(rng.integers(1, m_max + 1))
        s = rng.normal(0.0, 2.0, size=m)
        kind = t % 5
        if kind == 0:
            a = rng.uniform(0.0, 2.0, size=m - 1)
        elif kind == 1:
            a = rng.uniform(0.0, 2.0, size=m - 1) * (rng.random(m - 1) < 0.5)
        elif kind == 2:
            a = rng.uniform(5.0, 50.0, size=m - 1)
        elif kind == 3:
            s = rng.integers(-2, 3, size=m).astype(float)
            a = rng.integers(0, 3, size=m - 1).astype(float)
        else:
            a = np.abs(rng.normal(0.0, 0.5, size=m - 1))
        out.append((s, a))
    return out


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, os.path.getsize(path), "bytes")


_PC = None


def grid_arrays(g, prefix=""):
    d = {prefix + "dims": np.array(g.dims, dtype=np.int64),
         prefix + "conn": np.array(g.connectivity),
         prefix + "w": g.w}
    if _PC is not None:
        d[prefix + "fingerprint"] = np.array(_PC.instance_fingerprint(g))
    for k, a in enumerate(g.dir_weights):
        d[prefix + "dw%d" % k] = a
    return d


def fixed_iter(pc, g, ks):
    dec = pc.decompose_grid(g)
    out = {}
    for k in ks:
        res = pc.solve(g, dec, pc.SolverConfig(algorithm="aar", max_iters=k,
                                               check_every=k + 1))
        st = res.dual_state
        out["z_%d" % k] = st.z
        out["y_%d" % k] = st.y
        out["norms_%d" % k] = np.asarray(res.monitor.get("aar_step_norm", []), dtype=np.float64)
        out["iters_%d" % k] = np.array(res.iterations)
        last = res.trace[-1]
        out["gap_%d" % k] = np.array(last.gap)
        out["energy_%d" % k] = np.array(last.energy)
        out["dual_%d" % k] = np.array(last.dual_objective)
    out["ks"] = np.array(ks, dtype=np.int64)
    return out


def main():
    global _PC
    pc = import_reference()
    _PC = pc
    sys.path.insert(0, REPO)
    from paracut_b200.instances import CONFIGS, make_instance

    # --- tv1d chains
    rng = np.random.default_rng(20261020)
    chains = chain_regimes(rng, 350)
    for m in (2000, 4096, 3):
        s = rng.normal(0, 2, size=m)
        a = rng.uniform(0, 1.5, size=m - 1)
        chains.append((s, a))
    # closed-form two-point and bitwise identities
    chains.append((np.array([1.0, -1.0]), np.array([1.0])))
    chains.append((np.array([1.0, -1.0]), np.array([0.25])))
    chains.append((np.full(25, -0.3), rng.uniform(0, 2, 24)))
    chains.append((rng.normal(size=40), np.zeros(39)))
    chains.append((np.array([4.2]), np.zeros(0)))
    s_all = np.concatenate([c[0] for c in chains])
    a_all = np.concatenate([c[1] for c in chains])
    ptr = np.cumsum([0] + [c[0].size for c in chains]).astype(np.int64)
    x_all = np.concatenate([pc.tv1d_prox(s, a) for s, a in chains])
    save("tv1d.npz", s=s_all, a=a_all, ptr=ptr, x=x_all)

    # --- fixed-iteration AAR on small grids
    cases = []
    r = np.random.default_rng(1)
    cases.append(("aar_r2d4", pc.random_grid((24, 31), "2D-4", r), (1, 7, 60)))
    cases.append(("aar_r2d8", pc.random_grid((17, 22), "2D-8", r), (1, 7, 60)))
    cases.append(("aar_r3d6", pc.random_grid((6, 7, 9), "3D-6", r), (1, 7, 60)))
    for conn, dims, name in (("2D-4", (48, 40), "aar_i2d4"), ("2D-8", (33, 30), "aar_i2d8"),
                             ("3D-6", (12, 10, 11), "aar_i3d6")):
        spec = {"2D-4": CONFIGS["cfg2_int"], "2D-8": CONFIGS["cfg3"],
                "3D-6": CONFIGS["cfg5_int"]}[conn]
        from paracut_b200.instances import synth_image, energy_from_image
        img = synth_image(dims, 4, 3, 9, seed=7)
        ours = energy_from_image(img, conn, integer=True)
        g = pc.GridEnergy(ours.dims, conn, ours.w, ours.dir_weights)
        cases.append((name, g, (1, 9, 80)))
    deg = [pc.random_grid((1, 7), "2D-4", r), pc.random_grid((5, 1), "2D-8", r),
           pc.random_grid((1, 1, 5), "3D-6", r), pc.random_grid((2, 2), "2D-8", r),
           pc.random_grid((1, 1), "2D-4", r), pc.random_grid((3, 1, 4), "3D-6", r)]
    for i, g in enumerate(deg):
        cases.append(("aar_deg%d" % i, g, (1, 5)))
    for name, g, ks in cases:
        d = grid_arrays(g)
        d.update(fixed_iter(pc, g, ks))
        save(name + ".npz", **d)

    # --- gap-stopped solves
    r = np.random.default_rng(5)
    for name, g in (("solve_2d4", pc.random_grid((14, 12), "2D-4", r)),
                    ("solve_2d8", pc.random_grid((10, 13), "2D-8", r)),
                    ("solve_3d6", pc.random_grid((5, 4, 6), "3D-6", r))):
        res = pc.solve(g, pc.decompose_grid(g),
                       pc.SolverConfig(algorithm="aar", gap_tol=1e-6, max_iters=20000,
                                       check_every=5))
        d = grid_arrays(g)
        d.update(iterations=np.array(res.iterations), certified=np.array(res.certified),
                 energy=np.array(res.energy), gap=np.array(res.gap),
                 labeling=res.labeling, tv_solution=res.tv_solution,
                 trace_iter=np.array([t.iteration for t in res.trace]),
                 trace_gap=np.array([t.gap for t in res.trace]),
                 trace_energy=np.array([t.energy for t in res.trace]),
                 trace_jac=np.array([t.jaccard for t in res.trace]),
                 norms=np.asarray(res.monitor["aar_step_norm"]),
                 z=res.dual_state.z, y=res.dual_state.y)
        save(name + ".npz", **d)

    # --- cfg1 at its full size and iteration count
    ours = make_instance("cfg1", seed=0)
    g = pc.GridEnergy(ours.dims, ours.connectivity, ours.w, ours.dir_weights)
    d = grid_arrays(g)
    d.update(fixed_iter(pc, g, (200,)))
    save("cfg1.npz", **d)

    # --- integer exact-energy pin: eps thresholds on one iterate + max-flow
    img = synth_image((64, 64), 6, 5, 20, seed=3)
    ours = energy_from_image(img, "2D-4", integer=True)
    g = pc.GridEnergy(ours.dims, "2D-4", ours.w, ours.dir_weights)
    res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(algorithm="aar", max_iters=400,
                                                            check_every=401))
    s = res.dual_state.y.sum(axis=0)
    x = g.w - s
    thr = np.array([0.0, 1e-6, -1e-6])
    gaps, ens = [], []
    for t in thr:
        c = pc.discrete_gap(g, (x > t).astype(np.uint8), s)
        gaps.append(c.gap)
        ens.append(c.primal_energy)
    lab_mf, e_mf = pc.maxflow_mincut(g)
    d = grid_arrays(g)
    d.update(thr=thr, gaps=np.array(gaps), energies=np.array(ens), maxflow=np.array(e_mf),
             z_400=res.dual_state.z, y_400=res.dual_state.y)
    save("eps_int.npz", **d)

    # --- frozen KAT (pkg/tests/test_oracle.py:60-68)
    g = pc.random_grid((4, 4), "2D-8", np.random.default_rng(12345))
    lab, e = pc.brute_force_mincut(g)
    d = grid_arrays(g)
    d.update(labeling=lab, energy=np.array(e))
    save("kat.npz", **d)

    make_levels()
    make_dual()
    make_io()
    make_path()


def make_levels():
    """Best-level-set certificates (certify.py:50-65) on partially solved x."""
    global _PC
    pc = import_reference()
    _PC = pc
    sys.path.insert(0, REPO)
    from paracut_b200.instances import synth_image, energy_from_image
    r = np.random.default_rng(9)
    cases = [("r2d4", pc.random_grid((12, 10), "2D-4", r), 3),
             ("r2d8", pc.random_grid((9, 11), "2D-8", r), 4),
             ("r3d6", pc.random_grid((4, 5, 6), "3D-6", r), 2)]
    for conn, dims in (("2D-4", (24, 20)), ("3D-6", (6, 7, 5))):
        ours = energy_from_image(synth_image(dims, 3, 2, 6, seed=11), conn, integer=True)
        cases.append(("i" + conn.replace("-", "").lower(),
                      pc.GridEnergy(ours.dims, conn, ours.w, ours.dir_weights), 5))
    for name, g, iters in cases:
        res = pc.solve(g, pc.decompose_grid(g),
                       pc.SolverConfig(algorithm="aar", max_iters=iters, check_every=iters + 1))
        s = res.dual_state.y.sum(axis=0)
        x = g.w - s
        lab, cert = pc.best_level_set_gap(g, x, s)
        base = pc.discrete_gap(g, pc.threshold(x), s)
        d = grid_arrays(g)
        d.update(x=x, s=s, labeling=lab, gap=np.array(cert.gap),
                 energy=np.array(cert.primal_energy), dual=np.array(cert.dual_objective),
                 thr0_gap=np.array(base.gap), nlevels=np.array(len(pc.level_sets(x))))
        save("levels_%s.npz" % name, **d)


def make_dual():
    """BCD / AP / FISTA (solvers.py:212-269, 310-341): fixed iterations,
    gap-stopped and dual_tol-stopped runs."""
    global _PC
    pc = import_reference()
    _PC = pc
    sys.path.insert(0, REPO)
    from paracut_b200.instances import synth_image, energy_from_image
    r = np.random.default_rng(21)
    grids = [("r2d4", pc.random_grid((13, 11), "2D-4", r)),
             ("r2d8", pc.random_grid((9, 12), "2D-8", r)),
             ("r3d6", pc.random_grid((5, 4, 6), "3D-6", r)),
             ("deg", pc.random_grid((1, 6), "2D-8", r))]
    ours = energy_from_image(synth_image((20, 18), 3, 2, 6, seed=5), "2D-4", integer=True)
    grids.append(("i2d4", pc.GridEnergy(ours.dims, "2D-4", ours.w, ours.dir_weights)))
    mon = {"bcd": "dual_objective", "ap": "ap_distance", "fista": "dual_objective"}
    for alg in ("bcd", "ap", "fista"):
        for name, g in grids:
            dec = pc.decompose_grid(g)
            d = grid_arrays(g)
            ks = (1, 6, 40)
            for k in ks:
                res = pc.solve(g, dec, pc.SolverConfig(algorithm=alg, max_iters=k,
                                                       check_every=k + 1))
                d["y_%d" % k] = res.dual_state.y
                if res.dual_state.lam is not None:
                    d["lam_%d" % k] = res.dual_state.lam
                d["mon_%d" % k] = np.asarray(res.monitor.get(mon[alg], []), dtype=np.float64)
                d["gap_%d" % k] = np.array(res.trace[-1].gap)
            d["ks"] = np.array(ks, dtype=np.int64)
            res = pc.solve(g, dec, pc.SolverConfig(algorithm=alg, gap_tol=1e-6, max_iters=600,
                                                   check_every=7))
            d.update(s_iterations=np.array(res.iterations), s_certified=np.array(res.certified),
                     s_energy=np.array(res.energy), s_labeling=res.labeling,
                     s_tv=res.tv_solution, s_y=res.dual_state.y,
                     s_trace_iter=np.array([t.iteration for t in res.trace]),
                     s_trace_gap=np.array([t.gap for t in res.trace]),
                     s_trace_dual=np.array([t.dual_objective for t in res.trace]))
            res = pc.solve(g, dec, pc.SolverConfig(algorithm=alg, dual_tol=1e-3, max_iters=400,
                                                   check_every=50))
            d.update(t_iterations=np.array(res.iterations), t_y=res.dual_state.y,
                     t_trace_iter=np.array([t.iteration for t in res.trace]))
            save("dual_%s_%s.npz" % (alg, name), **d)


def make_io():
    """Files written by the reference's io.py (io.py:113-261): our readers must
    load them bitwise and our writers must reproduce their bytes."""
    global _PC
    pc = import_reference()
    _PC = pc
    from paracut.solvers import TraceRow
    r = np.random.default_rng(31)
    out = os.path.join(HERE, "io")
    os.makedirs(out, exist_ok=True)
    for conn, dims in (("2D-4", (5, 7)), ("2D-8", (4, 6)), ("3D-6", (3, 4, 5))):
        g = pc.random_grid(dims, conn, r)
        tag = conn.replace("-", "").lower()
        pc.write_grid(g, os.path.join(out, "grid_%s.pcut" % tag))
        pc.write_grid(g, os.path.join(out, "grid_%s.txt" % tag), text=True)
        np.savez(os.path.join(out, "grid_%s_arrays.npz" % tag), w=g.w,
                 **{"dw%d" % k: a for k, a in enumerate(g.dir_weights)},
                 fingerprint=np.array(pc.instance_fingerprint(g)))
    w = r.uniform(-3, 3, 9)
    edges = [(i, j, float(r.uniform(0.01, 2.0))) for i in range(9) for j in range(i + 1, 9)
             if r.random() < 0.4]
    del w, edges  # (drawn for the general-instance files of round 1; kept for the RNG stream)
    st = pc.DualState(y=r.normal(size=(2, 6)), z=r.normal(size=(2, 6)), fingerprint="fp-io")
    pc.save_dual(st, os.path.join(out, "state.dual"))
    trace = [TraceRow(0, 1.25, -0.5, 3.0, np.nan, 0.001), TraceRow(10, 0.0, 2.0, -1.0, 0.25, 0.002)]
    pc.write_trace(trace, os.path.join(out, "trace.csv"))
    print("wrote", out)


def make_path():
    """Warm-started lambda path the reference way (scaled_pairwise + force_warm)."""
    global _PC
    pc = import_reference()
    _PC = pc
    sys.path.insert(0, REPO)
    from paracut_b200.instances import synth_image, energy_from_image
    r = np.random.default_rng(41)
    cases = [("r3d6", pc.random_grid((6, 5, 7), "3D-6", r))]
    ours = energy_from_image(synth_image((40, 36), 4, 3, 9, seed=13), "2D-4", integer=True)
    cases.append(("i2d4", pc.GridEnergy(ours.dims, "2D-4", ours.w, ours.dir_weights)))
    lams = [0.25, 0.5, 1.0, 2.0]
    for name, g in cases:
        d = grid_arrays(g)
        d["lambdas"] = np.array(lams)
        res = None
        for i, lam in enumerate(lams):
            gl = g.scaled_pairwise(lam)
            cfg = pc.SolverConfig(algorithm="aar", gap_tol=1e-6, max_iters=400, check_every=10,
                                  warm_start=res.dual_state if res else None, force_warm=True)
            res = pc.solve(gl, pc.decompose_grid(gl), cfg)
            d.update({"iters_%d" % i: np.array(res.iterations), "energy_%d" % i: np.array(res.energy),
                      "gap_%d" % i: np.array(res.gap), "certified_%d" % i: np.array(res.certified),
                      "labeling_%d" % i: res.labeling, "y_%d" % i: res.dual_state.y,
                      "z_%d" % i: res.dual_state.z,
                      "fp_%d" % i: np.array(res.dual_state.fingerprint)})
        save("path_%s.npz" % name, **d)


def make_cfg1():
    """cfg1.npz alone: BASELINE cfg1 (256^2 2D-4, seed 0) through the reference
    at k = 200 (rerun when the synthetic generator changes)."""
    global _PC
    pc = import_reference()
    _PC = pc
    sys.path.insert(0, REPO)
    from paracut_b200.instances import make_instance
    ours = make_instance("cfg1", seed=0)
    g = pc.GridEnergy(ours.dims, ours.connectivity, ours.w, ours.dir_weights)
    d = grid_arrays(g)
    d.update(fixed_iter(pc, g, (200,)))
    save("cfg1.npz", **d)


if __name__ == "__main__" and "cfg1" in sys.argv[1:]:
    make_cfg1()
elif __name__ == "__main__" and "path" in sys.argv[1:]:
    make_path()
elif __name__ == "__main__" and "io" in sys.argv[1:]:
    make_io()
elif __name__ == "__main__" and "levels" in sys.argv[1:]:
    make_levels()
elif __name__ == "__main__" and "dual" in sys.argv[1:]:
    make_dual()
elif __name__ == "__main__":
    main()
