"""Warp instructions per code section of the sweep kernels from an ncu source
page (--page source --csv --print-source cuda,sass), per kernel, normalised
per warp-position (n / 32 positions of 32 chains per launch).

    python tools/ncu_sections.py src.csv N_NODES
"""
import csv
import sys
from collections import defaultdict

# fast_sweep.cuh line ranges (inclusive) -> section
SECTIONS = [
    ("cp/tma helpers", 125, 192), ("rcp/ring index", 193, 227),
    ("lag/global", 236, 281), ("setup", 482, 639), ("issue", 640, 700),
    ("prefetch G/X", 701, 729), ("to_z", 730, 738), ("retire", 739, 854),
    ("scan trip", 855, 986), ("scan vote", 987, 999), ("main loop", 1095, 1143),
    ("epilogue", 1144, 1161),
]


def section(path, ln):
    if not path.endswith("fast_sweep.cuh"):
        return path.rsplit("/", 1)[-1]
    for name, a, b in SECTIONS:
        if a <= ln <= b:
            return name
    return "other fast_sweep"


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
