"""Print the hot scan loop of a cuobjdump -sass listing (the backward-branch
loop containing MUFU.RCP and no global loads) with an opcode histogram."""
import re
import sys
from collections import Counter

lines = [l.strip() for l in open(sys.argv[1])]
best = None
for l in lines:
    m = re.search(r'BRA (0x[0-9a-f]+)', l)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    a = int(re.match(r'/\*([0-9a-f]+)\*/', l).group(1), 16)
    if tgt < a and a - tgt < 0x900:
        body = [x for x in lines if tgt <= int(re.match(r'/\*([0-9a-f]+)\*/', x).group(1), 16) <= a]
        if any('MUFU.RCP' in x for x in body) and not any('LDG' in x for x in body):
            best = (tgt, a, body)
tgt, a, body = best
ops = Counter()
for x in body:
    op = x.split('*/')[1].strip()
    if op.startswith('@'):
        op = op.split(None, 1)[1]
    ops[op.split()[0].split('.')[0]] += 1
print(hex(tgt), hex(a), len(body), ops.most_common())
if len(sys.argv) > 2:
    for x in body:
        print(x[:110])
