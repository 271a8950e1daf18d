"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_*] --csv).

    python tools/launch_summary.py launches.csv [--skip-setup]
Prints per-kernel launch count, mean duration, share of the listed time, and
DRAM bytes per launch when captured."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = [r for r in csv.reader(open(path)) if r and r[0] != "==PROF=="]
    hdr = None
    data = OrderedDict()
    for r in rows:
        if r[0] == "ID":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        lid = int(r[hdr["ID"]])
        ent = data.setdefault(lid, {"name": r[hdr["Kernel Name"]], "grid": r[hdr["Grid Size"]]})
        ent[r[hdr["Metric Name"]]] = float(r[hdr["Metric Value"]].replace(",", ""))
    return data


def main(path):
    data = load(path)
    agg = OrderedDict()
    for lid, ent in data.items():
        name = ent["name"].split("(")[0].replace("void ", "")
        key = name + " grid" + ent["grid"]
        a = agg.setdefault(key, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += ent.get("gpu__time_duration.sum", 0.0)
        a[2] += ent.get("dram__bytes_read.sum", 0.0)
        a[3] += ent.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values()) or 1.0
    print("%-70s %5s %12s %7s %14s" % ("kernel", "count", "mean_us", "share", "dram_MB/launch"))
    for k, (n, t, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("%-70s %5d %12.1f %6.1f%% %14.1f" % (k[:70], n, t / n / 1e3, 100 * t / tot,
                                                   (rd + wr) / n / 1e6))


if __name__ == "__main__":
    main(sys.argv[1])
