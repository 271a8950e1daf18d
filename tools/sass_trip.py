"""Instruction count of the lag-free scan loop (the backward-branch loop with
PCB_SCAN_UNROLL MUFU.RCPs and no global loads) of every fast::k_sweep
instantiation in a built library.

    python tools/sass_trip.py [path/to/libparacut_b200.so]
"""
import re
import subprocess
import sys
from collections import Counter

so = sys.argv[1] if len(sys.argv) > 1 else "paracut_b200/_lib/libparacut_b200.so"
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", txt)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if "fast7k_sweep" not in name:
        continue
    lines = [l.strip() for l in f.split("\n") if re.match(r"\s*/\*[0-9a-f]{4,5}\*/", l)]
    addr = lambda l: int(re.match(r"/\*([0-9a-f]+)\*/", l).group(1), 16)
    best = None
    for l in lines:
        m = re.search(r"BRA (0x[0-9a-f]+)", l)
        if not m:
            continue
        tgt, a = int(m.group(1), 16), addr(l)
        if tgt >= a:
            continue
        body = [x for x in lines if tgt <= addr(x) <= a]
        nm = sum("MUFU.RCP" in x for x in body)
        if nm >= 1 and not any("LDG" in x or "CALL" in x for x in body):
            if best is None or len(body) > len(best[2]):
                best = (tgt, a, body, nm)
    if best is None:
        continue
    ops = Counter()
    for x in best[2]:
        op = x.split("*/")[1].strip().split(";")[0]
        if op.startswith("@"):
            op = op.split(None, 1)[1]
        ops[op.split()[0].split(".")[0]] += 1
    alu = sum(ops[o] for o in ("ISETP", "FSETP", "PLOP3", "SEL", "FSEL", "LOP3", "SHF", "VIMNMX", "VIMNMX3", "PRMT", "IADD3", "VIADD"))
    print("%-45s %4d instr, %d trips -> %.1f per trip (ALU-ish %.1f)" % (
        name[:45], len(best[2]), best[3], len(best[2]) / best[3], alu / best[3]))
