#!/usr/bin/env python
"""Benchmark of the AAR chain-prox hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--impl ours|reference]

A *step* is one AAR iteration (every chain family's exact weighted 1D-TV prox
plus the reflect/average/primal update and the step-norm monitor) over the
whole grid of BASELINE.json's workload (default cfg4: 3D-6 256^3, fp32 state).
``value`` = grid-node prox updates per second = r * n * K * N / t, with t the
max over ranks of the CUDA-event time of K steps on data resident in HBM
(working set > L2, so no flush is needed).  ``e2e`` runs the same K steps
through the public API ``paracut_b200.solve`` from host numpy arrays in
pinned memory (upload, cold start, shadow + certificate at k=0 and k=K, the
labeling read back; the fp64 TV solution is copied only when the caller
reads ``tv_solution``), wall clock.  ``roofline`` covers the dominant kernel
(the chain family prox kernel with the largest share of the step), timed
live with CUDA events around each launch inside the timed region.
``cpu_baseline`` is the oracle's C restatement of the reference loop (bitwise
equal to it) on the same instance, all host threads and one thread, with
the CPU time to cut extrapolated from the GPU solve's iteration count.
``time_to_cut`` is the
metric's second half: wall time of ``paracut_b200.solve`` from host arrays to a
certified optimal cut (gap <= 1e-6 at a check, checks every 10 iterations).

N > 1 (torchrun, NCCL): the ONE workload instance is slab-sharded across the
ranks (paracut_b200.distributed.ShardedAAR): local chain families on a slab
handle, the cross-slab family on a pencil handle, two NCCL all-to-alls of
fp32 per iteration ("scaling": "strong", whole-job updates/s).
``--impl reference`` times the CPU reference port on rank 0 only; other
ranks exit 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-node TV-prox updates/sec per AAR iteration"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--precision", default=None, choices=(None, "f32", "f64", "f64s"))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--sharded", action="store_true",
                    help="run the slab-sharded NCCL path even at world size 1 (test of the N>1 path)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ttc", action="store_true", help="skip the time-to-optimal-cut solves")
    ap.add_argument("--cpu-iters", type=int, default=3)
    ap.add_argument("--path", action="store_true",
                    help="time BASELINE's warm-started lambda path (cfg5: 5 x 300 iterations) "
                         "through paracut_b200.solve_path instead of the step")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons; only samples whose timestamp falls
    inside [mark_start, mark_end] (the timed region) are kept."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        import datetime
        sm, smax, reasons, allsm = [], [], set(), []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                v, vmax = float(parts[1]), float(parts[2])
            except ValueError:
                continue
            allsm.append(v)
            # keep the timed region, with a 50 ms guard for the sampling period
            if self.t0 is not None and not (self.t0 - 0.05 <= ts <= self.t1 + 0.05):
                continue
            sm.append(v)
            smax.append(vmax)
            for nm, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def cpu_port_rate(g, iters, threads, warm=1, runner=None):
    """(updates/s, seconds per iteration) of the oracle's C port of the
    reference loop (bitwise the reference's fp64 arithmetic, OpenMP over
    chains) on the whole workload instance with `threads` host threads."""
    from oracle import oracle as orc
    run = runner if runner is not None else orc.AARRunner(g, threads=threads)
    run.threads = int(threads)
    if warm:
        run.run(warm, final_shadow=False)
    t0 = time.perf_counter()
    run.run(iters, final_shadow=False)
    dt = time.perf_counter() - t0
    return run.r * run.n * iters / dt, dt / iters, run


def cpu_baseline(g, workload, iters_all=3, iters_one=1, ttc_iters=None):
    """The reference arithmetic on this box's host cores, same instance as the
    GPU line: all cores and one core, plus the CPU time to a certified cut
    extrapolated from the per-iteration time (the GPU solve's iteration count
    to its certificate; checks every 10 iterations not counted)."""
    from oracle import oracle as orc
    tmax = orc.max_threads()
    rate, spi, run = cpu_port_rate(g, iters_all, tmax)
    rate1, spi1, _ = cpu_port_rate(g, iters_one, 1, warm=0, runner=run)
    out = {"value": rate, "unit": "updates/s", "cores": tmax, "kind": "port",
           "sample": ("%s %s (the whole %s instance), %d AAR iterations on %d threads and %d on "
                      "1 thread after one warm-up iteration; oracle/paracut_oracle.c: the "
                      "reference loop in its fp64 operation order, OpenMP over chains"
                      % (g.connectivity, "x".join(map(str, g.dims)), workload, iters_all, tmax,
                         iters_one)),
           "s_per_iter": spi, "one_core": {"value": rate1, "unit": "updates/s", "cores": 1,
                                           "s_per_iter": spi1}}
    if ttc_iters:
        out["time_to_cut"] = {"value": spi * ttc_iters, "unit": "s", "cores": tmax,
                              "iterations": int(ttc_iters), "extrapolated": True,
                              "one_core_value": spi1 * ttc_iters,
                              "rule": "per-iteration time x the GPU solve's iterations to its "
                                      "certificate (check iterations not counted)"}
    return out


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args, world, rank):
    """The reference's CPU implementation of the path (its loop in the
    reference's fp64 operation order: oracle/paracut_oracle.c) on the box's
    host cores, on the SAME workload instance as our arm; rank 0 only."""
    from paracut_b200.instances import CONFIGS, make_instance
    if rank != 0:
        return
    from oracle import oracle as orc
    spec = CONFIGS[args.workload]
    g = make_instance(spec, seed=args.seed)
    threads = orc.max_threads()
    run = orc.AARRunner(g, threads=threads)
    run.run(max(args.warmup, 1), final_shadow=False)
    t0 = time.perf_counter()
    run.run(args.steps, final_shadow=False)
    dt = time.perf_counter() - t0
    value = run.r * run.n * args.steps / dt
    desc = ("%s %s, the whole %s instance (seed %d), fp64 (the reference is fp64-only); each "
            "step one AAR iteration on %d threads" % (g.connectivity, "x".join(map(str, g.dims)),
                                                      args.workload, args.seed, threads))
    line = {
        "metric": METRIC, "value": value, "unit": "updates/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE.json generator)",
        "config": {"workload": args.workload, "dims": list(spec.dims),
                   "connectivity": spec.connectivity, "r": run.r, "n": run.n,
                   "step": "1 AAR iteration"},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": threads, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_sharded(args, world, rank, local):
    """N > 1: one instance, slab-sharded over the ranks (strong scaling)."""
    import torch
    import torch.distributed as dist
    from paracut_b200 import _native
    from paracut_b200.distributed import ShardedAAR, TorchComm
    from paracut_b200.graph import DIRECTIONS
    from paracut_b200.instances import CONFIGS, DeviceGrid, HostPartsGrid, make_instance

    torch.cuda.set_device(local)
    if "MASTER_ADDR" not in os.environ:  # --sharded without torchrun: world of one
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = CONFIGS[args.workload]
    # every rank builds only its own slab and pencil: on its GPU for the timed
    # run (pcb_create_synthetic_box), from host arrays of its parts for e2e;
    # 2D-8 halo slabs fall back to the whole host instance
    halo = spec.connectivity == "2D-8"
    g = make_instance(spec, seed=args.seed) if halo else DeviceGrid(spec, seed=args.seed,
                                                                    device=local)
    r, n = len(DIRECTIONS[spec.connectivity]), int(np.prod(spec.dims))
    backend = lambda sub: _native.GridSolver(sub, precision="f32", device=local)
    sh = ShardedAAR(g, TorchComm(), [rank], backend, device="cuda")
    sh.init_cold()
    sh.run(args.warmup, norms=False)
    mode = "cuda-graph"
    try:
        sh.capture()  # one iteration as a graph (handles, transposes, NCCL all-to-alls)
        sh.run_graph(2)
    except Exception as e:  # capture unsupported here: time the eager loop instead
        mode = "eager (graph capture failed: %s)" % (str(e).splitlines()[0][:80],)
        for h in sh.slab + sh.pencil:
            h.set_stream(0)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    handles = sh.slab + sh.pencil
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    clocks.mark_start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream()  # CUDAGraph.replay launches on the current stream
    ev0.record(stream)
    if mode == "cuda-graph":
        sh.run_graph(args.steps)
    else:
        sh.run(args.steps, norms=False)
    ev1.record(stream)
    ev1.synchronize()
    clocks.mark_end()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    # graph replays carry no per-launch events: time the family kernels (and
    # count this library's launches per iteration) over a few eager iterations
    torch.cuda.synchronize()
    for h in handles:
        h.set_stream(0)
        h.reset_launch_count()
        h.set_profiling(True)
    n_prof = 3
    sh.run(n_prof, norms=False)
    torch.cuda.synchronize()
    prof = [h.profile_read() for h in handles]
    launches = sum(h.launch_count() for h in handles) * args.steps // n_prof
    for h in handles:
        h.set_profiling(False)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = r * n * args.steps / (ms_max / 1e3)
    # dominant family kernel on this rank (slab: local families, pencil: cross)
    pk, pk_kind = peaks()
    best = None
    subs = ([g.part(*d) for d in sh.geo.parts(rank)] if not halo
            else [sh.geo.slab_grid(g, rank), sh.geo.pencil_grid(g, rank)])
    for h, (fms, fcnt), sub in zip(handles, prof, subs):
        fe = _family_edges(sub)
        for j in range(len(fms)):
            if fcnt[j] and (best is None or fms[j] > best[0]):
                best = (float(fms[j]), int(fcnt[j]), 4 * (2 * sub.n + fe[j]), j)
    mean_ms = best[0] / best[1]
    achieved = best[2] / (mean_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": pk, "unit": "GB/s",
            "frac": achieved / pk, "traffic": None, "peak_kind": pk_kind,
            "kernel": "family %d prox sweep (rank %d)" % (best[3], rank),
            "bytes_per_launch": best[2], "mean_launch_ms": mean_ms}
    # e2e: build the rank's shards from host arrays, cold start, K steps, read y back
    # the rank's host input arrays (its slab and pencil) exist before the timed
    # region, as a user's instance would
    g2 = g if halo else HostPartsGrid(spec, seed=args.seed, device=local)
    for d in (sh.geo.parts(rank) or ()) if not halo else ():
        g2.part(*d)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    sh2 = ShardedAAR(g2, TorchComm(), [rank], backend, device="cuda")
    sh2.init_cold()
    sh2.run(args.steps, norms=True)
    ys = sh2.local_shadow()
    wall = time.perf_counter() - t0
    wt = torch.tensor([wall], dtype=torch.float64, device="cuda")
    dist.all_reduce(wt, op=dist.ReduceOp.MAX)
    wall = float(wt.item())
    geo = sh.geo
    h2d = 8 * (geo.n_slab + geo.n_pencil) + 8 * (geo.n_slab * r + geo.n_pencil)
    d2h = 8 * (geo.n_slab * len(ys[rank][0]) + geo.n_pencil)
    e2e = {"value": r * n * args.steps / wall, "unit": "updates/s",
           "h2d_bytes_per_step": world * h2d / args.steps,
           "d2h_bytes_per_step": world * d2h / args.steps, "wall_s": wall}
    if rank == 0:
        B_iter = 4 * ((2 * r + 1) * n + sum(int(np.prod([s - abs(o) for s, o in zip(spec.dims, d)]))
                                           for d in DIRECTIONS[spec.connectivity]))
        line = {
            "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32",
            "arithmetic": "fp32 anchor-relative scan, fp64 drift c and segment values",
            "data": "synthetic (BASELINE.json generator, seed %d)" % args.seed,
            "config": {"workload": args.workload, "dims": list(spec.dims),
                       "connectivity": spec.connectivity, "r": r, "n": n, "precision": "f32",
                       "step": "1 AAR iteration", "parallelism": "slab%d" % world,
                       "exchange": "2 x NCCL all-to-all of fp32 per iteration",
                       "launch": mode,
                       "l2": "working set %.0f MB > 126 MB L2, no flush needed"
                             % (B_iter / 1e6)},
            "roofline": roof, "cpu_baseline": None, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_path(args, local):
    """BASELINE cfg5's warm-started lambda path through the public API
    (solve_path: one upload, pairwise weights rescaled on the device, the AAR
    state carried over), from pinned host arrays; wall clock of the whole path.
    The CPU figure is the oracle's per-iteration time on the same instance x
    the path's iterations (extrapolated, labelled so)."""
    import torch
    import paracut_b200 as pc
    from paracut_b200.instances import CONFIGS, LAMBDA_PATH, make_instance
    torch.cuda.set_device(local)
    wl = args.workload if args.workload != "cfg4" else "cfg5"
    spec = CONFIGS[wl]
    precision = args.precision or "f32"
    g = make_instance(spec, seed=args.seed)
    gp = pinned_instance(g)
    del g
    r, n = len(gp.dir_weights), gp.n
    cfg = pc.SolverConfig(max_iters=spec.iters, check_every=spec.iters, precision=precision,
                          device=local)
    walls, out = [], None
    for _ in range(2):  # the first also pays lazy module loading
        out = None
        t0 = time.perf_counter()
        out = pc.solve_path(gp, LAMBDA_PATH, cfg, keep_states=False)
        _ = [int(res.labeling[0]) + int(res.labeling[-1]) for res in out]  # host arrays, read back in solve
        walls.append(time.perf_counter() - t0)
    wall = min(walls)
    iters = sum(res.iterations for res in out)
    line = {"metric": METRIC + " (warm-started lambda path)", "mode": "lambda_path",
            "value": r * n * iters / wall, "unit": "updates/s", "wall_s": wall,
            "wall_s_runs": walls, "iterations": iters, "higher_is_better": True,
            "dtype": "f32" if precision == "f32" else "f64",
            "config": {"workload": wl, "dims": list(spec.dims), "lambdas": list(LAMBDA_PATH),
                       "iters_per_lambda": spec.iters, "precision": precision,
                       "inputs": "pinned host arrays, one upload for the whole path"},
            "per_lambda": [{"lambda": lam, "iterations": res.iterations,
                            "energy": float(res.energy), "gap": float(res.gap)}
                           for lam, res in zip(LAMBDA_PATH, out)]}
    if not args.no_cpu:
        from oracle import oracle as orc
        spi = cpu_port_rate(make_instance(spec, seed=args.seed), 1, orc.max_threads())[1]
        line["cpu_baseline"] = {"value": r * n / spi, "unit": "updates/s",
                                "cores": orc.max_threads(), "kind": "port",
                                "path_wall_s": spi * iters, "extrapolated": True,
                                "sample": "1 AAR iteration on the whole instance after one "
                                          "warm-up iteration, x the path's iterations"}
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    world, rank, local = dist_setup(args)
    if args.path and args.impl == "ours":
        if rank == 0:
            run_path(args, local)
        return
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    if world > 1 or args.sharded:
        run_sharded(args, world, rank, local)
        return

    import torch
    import torch.distributed as dist
    import paracut_b200 as pc
    from paracut_b200 import _native
    from paracut_b200.instances import CONFIGS, make_instance, algorithmic_bytes

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = CONFIGS[args.workload]
    precision = args.precision or ("f64" if spec.dtype == "f64" else "f32")
    b = 4 if precision == "f32" else 8
    g = make_instance(spec, seed=args.seed + rank)
    S = _native.GridSolver(g, precision=precision, device=local)
    r, n = S.r, S.n
    stream = torch.cuda.Stream(device=local)
    S.set_stream(stream.cuda_stream)
    clocks = ClockSampler(local)
    clocks.start()
    S.init_cold()
    # warm-up: W iterations, rounded up to a multiple of the library's graph
    # block (8), with the CUDA graphs of the plain iterations captured on the
    # first block (the library's default waits for 64 eager iterations), so
    # the timed region is the steady state of a long solve
    warm = max(8 * ((args.warmup + 7) // 8), 8)
    S.set_graph_after(0)
    S.run(warm, norms=False)
    S.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    time.sleep(0.3)
    clocks.mark_start()
    S.reset_launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    S.run(args.steps, norms=False)  # (small grids: CUDA-graph replays of 8 iterations)
    ev1.record(stream)
    ev1.synchronize()
    clocks.mark_end()
    ms = ev0.elapsed_time(ev1)
    launches = S.launch_count()
    clk = clocks.stop()
    torch.cuda.synchronize()
    # per-family kernel times: CUDA events around every family launch, over
    # eager iterations right after the timed region (same state, same kernels)
    S.set_profiling(True)
    S.run(max(min(args.steps, 20), 2), norms=False)
    torch.cuda.synchronize()
    fam_ms, fam_cnt = S.profile_read()
    S.set_profiling(False)

    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * r * n * args.steps / (ms_max / 1e3)

    # roofline of the dominant kernel: per-launch algorithmic bytes / mean duration
    pk, pk_kind = peaks()
    fam = int(np.argmax(fam_ms))
    nedge = [int(np.count_nonzero(a)) for a in g.dir_weights]
    fam_edges = _family_edges(g)
    per_launch = b * (2 * n + fam_edges[fam])
    if precision == "f64":  # the exact sweep is one launch over all families
        per_launch = sum(b * (2 * n + e) for e in fam_edges)
    mean_ms = fam_ms[fam] / max(int(fam_cnt[fam]), 1)
    achieved = per_launch / (mean_ms / 1e3) / 1e9
    traffic = _ncu_traffic(args.workload, fam)
    issue = _ncu_issue(args.workload, fam, mean_ms)
    B_iter = algorithmic_bytes(g, r, b)
    roof = {"bound": "hbm", "achieved": achieved, "peak": pk, "unit": "GB/s",
            "frac": achieved / pk, "traffic": traffic,
            "kernel": ("exact prox sweep, all families in one launch" if precision == "f64"
                       else "family %d (%s) prox sweep" % (fam, pc.decompose_grid(g).families[fam])),
            "bytes_per_launch": per_launch, "mean_launch_ms": mean_ms,
            "share_of_step": float(mean_ms * args.steps / ms) if ms > 0 else None,
            "peak_kind": pk_kind,
            "per_family_ms": [float(v / max(int(c), 1)) for v, c in zip(fam_ms, fam_cnt)],
            "iteration_achieved_gbs": B_iter * args.steps / (ms / 1e3) / 1e9,
            "iteration_bytes": B_iter, "iteration_frac": B_iter * args.steps / (ms / 1e3) / 1e9 / pk,
            "issue": issue}

    e2e = None
    if not args.no_e2e:
        S.close()
        del S
        torch.cuda.synchronize()
        dims, wbytes = g.dims, g.w.nbytes + sum(a.nbytes for a in g.dir_weights)
        gp = pinned_instance(g)  # the step's inputs in pinned host memory (contract)
        cfg = pc.SolverConfig(algorithm="aar", max_iters=args.steps,
                              check_every=args.steps + 1, precision=precision,
                              device=local)
        walls = []
        res = None
        for _rep in range(3):  # median of three end-to-end solves
            res = None  # release the previous solve's device state first
            t0 = time.perf_counter()
            res = pc.solve(gp, pc.decompose_grid(gp), cfg)
            # the step's result: solve returns the labeling (n bytes) in host
            # memory, copied inside the call (a host pass over it, e.g.
            # np.count_nonzero, would add 2.4 ms of numpy time at cfg4)
            _ = int(res.labeling[0]) + int(res.labeling[-1])
            walls.append(time.perf_counter() - t0)
        wall = float(np.median(walls))
        wt = torch.tensor([wall], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        wall = float(wt.item())
        nb = (n + 7) // 8
        d2h = n + 2 * nb + 2 * 8 * 4  # labels (uint8), two packed check labelings, scalars
        e2e = {"value": world * r * n * args.steps / wall, "unit": "updates/s",
               "h2d_bytes_per_step": wbytes / args.steps, "d2h_bytes_per_step": d2h / args.steps,
               "wall_s": wall, "wall_s_runs": walls, "certified": bool(res.certified),
               "gap": float(res.gap)}

    ttc = None
    if rank == 0 and world == 1 and not args.no_ttc:
        ttc = time_to_cut(pc, gp if not args.no_e2e else g, precision, local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(g, args.workload, iters_all=args.cpu_iters,
                           ttc_iters=ttc["iterations"] if ttc else None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "warmup_run": warm,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if precision == "f32" else "f64",
            "arithmetic": ("fp32 anchor-relative scan, fp64 drift c and segment values"
                           if precision == "f32" else "fp64, bitwise the reference"),
            "data": "synthetic (BASELINE.json generator, seed %d+rank)" % args.seed,
            "config": {"workload": args.workload, "dims": list(spec.dims),
                       "connectivity": spec.connectivity, "r": r, "n": n,
                       "precision": precision, "step": "1 AAR iteration",
                       "parallelism": "replicas" if world > 1 else "single",
                       "l2": "working set %.0f MB > 126 MB L2, no flush needed"
                             % (B_iter / 1e6)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "time_to_cut": ttc,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def pinned_instance(g):
    """The instance with its unaries and direction weights copied into pinned
    (page-locked) host memory: the e2e step's inputs, per the bench contract."""
    import torch
    from paracut_b200.graph import GridEnergy

    def pin(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()
    return GridEnergy(g.dims, g.connectivity, pin(g.w), [pin(a) for a in g.dir_weights])


def time_to_cut(pc, g, precision, device, reps=3):
    """Second half of the metric: wall time to a certified optimal cut (gap <=
    1e-6, the reference's GAP_SLACK) through the public API from host arrays,
    reference stopping rule (checks every 10 iterations); f32 runs hand over to
    the fast fp64 mode (f64s) once the fp32 gap stalls.  Median of `reps` solves."""
    cfg = pc.SolverConfig(max_iters=20000, check_every=10, precision=precision, device=device,
                          thresholds=(0.0, 1e-6, -1e-6, 1e-3),
                          polish_iters=5000 if precision == "f32" else 0,
                          polish_stall=5 if precision == "f32" else 0,
                          polish_gap=1e-2)
    walls, res = [], None
    for _ in range(reps):
        res = None
        t0 = time.perf_counter()
        res = pc.solve(g, pc.decompose_grid(g), cfg)
        _ = int(res.labeling[0]) + int(res.labeling[-1])  # (host array, read back in solve)
        walls.append(time.perf_counter() - t0)
    ps = res.monitor.get("polish_start")
    return {"value": float(np.median(walls)), "unit": "s", "wall_s_runs": walls,
            "iterations": int(res.iterations), "certified": bool(res.certified),
            "gap": float(res.gap), "energy": float(res.energy),
            "threshold": float(res.threshold),
            "polish_start": int(ps[0]) if ps else None,
            "rule": "gap <= 1e-6 at a check (every 10 iterations), thresholds 0, +-1e-6, 1e-3; "
                    "host arrays in, labels out"}


def _family_edges(g):
    """|E_j| per family (nonzero edges each chain family owns), decompose_grid order."""
    dw = g.dir_weights
    nz = [int(np.count_nonzero(a)) for a in dw]
    if g.connectivity == "2D-4" or g.connectivity == "3D-6":
        return nz
    # 2D-8: zig-zag phase 0 takes d1 on even columns, d2 on odd; phase 1 the rest
    d1, d2 = dw[2], dw[3]
    even = (np.arange(d1.shape[1]) % 2) == 0
    z0 = int(np.count_nonzero(d1[:, even])) + int(np.count_nonzero(d2[:, ~even]))
    z1 = int(np.count_nonzero(d2[:, even])) + int(np.count_nonzero(d1[:, ~even]))
    return [nz[0], nz[1], z0, z1]


def _ncu_issue(workload, fam, mean_ms, sms=148, sm_ghz=1.965):
    """The instruction-issue roofline of the same kernel: its warp instructions
    per launch (committed ncu capture) / its live mean launch time, against 4
    warp instructions per cycle per SM at the max SM clock."""
    path = os.path.join(ROOT, "profiles", "ncu_issue.json")
    try:
        with open(path) as f:
            inst = json.load(f).get(workload, {}).get(str(fam))
    except Exception:
        inst = None
    if not inst or not mean_ms:
        return None
    achieved = inst / (mean_ms / 1e3) / 1e9
    peak = sms * 4 * sm_ghz
    return {"bound": "issue", "warp_instructions": inst, "achieved": achieved, "peak": peak,
            "unit": "G warp-instr/s", "frac": achieved / peak}


def _ncu_traffic(workload, fam):
    """dram bytes per launch of that kernel from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            data = json.load(f)
        return data.get(workload, {}).get(str(fam))
    except Exception:
        return None


if __name__ == "__main__":
    main()
