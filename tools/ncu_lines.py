"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = None
    func = None
    agg = {}
    line = None
    for r in rows:
        if len(r) >= 2 and r[0] == "Function Name":
            func = r[1]
        if r and r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            line = (func, int(r[0]), r[1])
            agg.setdefault(line, [0, 0, 0])
            continue
        if r[2] in ("...", "-") or line is None:
            continue
        try:
            stall = int(r[hdr["Warp Stall Sampling (All Samples)"]])
            ex = int(r[hdr["Instructions Executed"]])
            thr = int(r[hdr["Thread Instructions Executed"]])
        except (ValueError, KeyError):
            continue
        a = agg[line]
        a[0] += stall
        a[1] += ex
        a[2] += thr
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_e = sum(v[1] for v in agg.values()) or 1
    print("total samples %d, warp instructions %d" % (tot_s, tot_e))
    for (f, ln, src), (s, e, t) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print("%5d %5.1f%% stall %5.1f%% inst  thr/inst %4.1f  %s" % (
            ln, 100.0 * s / tot_s, 100.0 * e / tot_e, t / max(e, 1), src.strip()[:90]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
