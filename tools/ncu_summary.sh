#!/bin/bash
# usage: tools/ncu_summary.sh REPORT.ncu-rep  -- local analysis of a capture
REP=$1
ncu -i $REP --page source --csv --print-source cuda,sass 2>/dev/null > /tmp/_cs.csv
python tools/ncu_lines.py /tmp/_cs.csv 30
ncu -i $REP --page details --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h={x:i for i,x in enumerate(r[0])}
want=['Duration','Executed Instructions','Avg. Active Threads Per Warp','Achieved Active Warps Per SM','Executed Ipc Active','DRAM Throughput','Issue Slots Busy','Registers Per Thread','Theoretical Active Warps per SM']
for row in r[1:]:
    if row[h['Metric Name']] in want: print(row[h['Metric Name']].ljust(35), row[h['Metric Unit']].ljust(10), row[h['Metric Value']])
"
ncu -i $REP --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin))
h=r[0]
out=[]
for i,name in enumerate(h):
    if name in ('dram__bytes_read.sum','dram__bytes_write.sum'): print(name, r[1][i], r[2][i])
    if 'smsp__average_warps_issue_stalled' in name and 'per_issue_active' in name and 'not_issued' not in name:
        out.append((float(r[2][i]), name.split('stalled_')[1].split('_per')[0]))
print(' '.join('%s=%.2f'%(n,v) for v,n in sorted(out,reverse=True)[:8]))
"
