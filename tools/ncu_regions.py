"""Instruction share per source-line range of an ncu cuda,sass source CSV.
usage: python tools/ncu_regions.py src.csv start:end:name ..."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
line = None
agg = {}
for r in rows:
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        line = int(r[0])
        continue
    if r[2] in ("...", "-"):
        continue
    try:
        agg[line] = agg.get(line, 0) + int(r[hdr["Instructions Executed"]])
    except (ValueError, KeyError):
        pass
tot = sum(agg.values())
for spec in sys.argv[2:]:
    a, b, name = spec.split(":")
    v = sum(x for l, x in agg.items() if int(a) <= l < int(b))
    print("%-10s %6.1f%%  %.3g" % (name, 100.0 * v / tot, v))
print("total", tot)
