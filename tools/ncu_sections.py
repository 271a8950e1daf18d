"""Warp instructions per code section of the sweep kernels from an ncu source
page (--page source --csv --print-source cuda,sass), per kernel, normalised
per warp-position (n / 32 positions of 32 chains per launch).

    python tools/ncu_sections.py src.csv N_NODES
"""
import csv
import sys
from collections import defaultdict

# fast_sweep.cuh sections, located by their first line (the file as it is now:
# re-run on a capture of the same source)
MARKS = [
    ("cp/tma helpers", "__device__ __forceinline__ void mbar_init"),
    ("rcp/ring index", "__device__ __forceinline__ double rcp_small"),
    ("lag/global", "__device__ __noinline__ double z_global"),
    ("other fast_sweep", "struct Spec {"),
    ("setup", "__global__ void __launch_bounds__(WARPS * 32)"),
    ("issue", "  auto issue = [&](int T) {"),
    ("prefetch G/X", "  auto prefetch = [&](int T) {"),
    ("to_z", "  auto to_z = [&](int T) {"),
    ("retire", "  auto retire_impl = [&](int T"),
    ("scan trip", "  auto scan = [&](int lo_pos"),
    ("scan vote", "    for (;;) {\n      const int nact"),
    ("VER", "  int ff = 0x7fffffff, fl = -1;"),
    ("main loop", "  if (!VER && warp_live && rhi > 0) {"),
    ("epilogue", "  if constexpr (VER) {\n    __syncwarp();"),
    ("merge", "// Intra-chain split: merge points"),
]


def _sections():
    import os
    src = open(os.path.join(os.path.dirname(__file__), "..", "paracut_b200", "csrc",
                            "fast_sweep.cuh")).read()
    out = []
    for name, mark in MARKS:
        i = src.find(mark)
        if i >= 0:
            out.append((src.count("\n", 0, i) + 1, name))
    return sorted(out)


SECTIONS = _sections()


def section(path, ln):
    if not path.endswith("fast_sweep.cuh"):
        return path.rsplit("/", 1)[-1]
    name = "header"
    for start, nm in SECTIONS:
        if ln >= start:
            name = nm
    return name


def main(path, n):
    rows = list(csv.reader(open(path)))
    file = func = None
    hdr = None
    line = None
    agg = defaultdict(lambda: defaultdict(lambda: [0, 0]))
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            file = r[1]
            continue
        if len(r) >= 2 and r[0] == "Function Name":
            func = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            line = int(r[0])
            continue
        if r[2] in ("...", "-") or line is None:
            continue
        try:
            ex = int(r[hdr["Instructions Executed"]])
            st = int(r[hdr["Warp Stall Sampling (All Samples)"]])
        except (ValueError, KeyError):
            continue
        a = agg[func][section(file, line)]
        a[0] += ex
        a[1] += st
    wp = n / 32.0
    for f, secs in agg.items():
        tot = sum(v[0] for v in secs.values())
        tst = sum(v[1] for v in secs.values()) or 1
        print("%s: %.1f warp-instr / warp-position (launches summed)" % (f[:90], tot / wp))
        for s, (e, st) in sorted(secs.items(), key=lambda kv: -kv[1][0]):
            print("   %-18s %7.1f  %5.1f%% inst  %5.1f%% stall" % (s, e / wp, 100.0 * e / tot, 100.0 * st / tst))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
