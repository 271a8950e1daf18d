"""Summarise an ncu --set full capture of family sweeps (details + raw CSV).

    python tools/ncu_fam_summary.py DIR "title"   (DIR holds details.csv, raw.csv)
"""
import csv
import sys

d, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
want = ['Duration', 'Executed Instructions', 'Avg. Active Threads Per Warp',
        'Achieved Active Warps Per SM', 'Theoretical Active Warps per SM', 'Executed Ipc Active',
        'DRAM Throughput', 'Issue Slots Busy', 'Registers Per Thread', 'SM Active Cycles',
        'Elapsed Cycles']
print(title)
det = list(csv.reader(open(d + "/details.csv")))
h = {x: i for i, x in enumerate(det[0])}
cur = None
for r in det[1:]:
    key = (r[h['ID']], r[h['Kernel Name']])
    if key != cur:
        cur = key
        print("\n== launch", r[h['ID']], r[h['Kernel Name']][:60])
    if r[h['Metric Name']] in want:
        print("  %-36s %-12s %s" % (r[h['Metric Name']], r[h['Metric Unit']], r[h['Metric Value']]))
raw = list(csv.reader(open(d + "/raw.csv")))
hdr, units = raw[0], raw[1]
for k, r in enumerate(raw[2:]):
    print("\n== launch %d raw" % k)
    st, pipes = [], []
    for i, name in enumerate(hdr):
        if name in ('dram__bytes_read.sum', 'dram__bytes_write.sum'):
            print("  %s %s %s" % (name, units[i], r[i]))
        if name.startswith('smsp__average_warps_issue_stalled_') and name.endswith('_per_issue_active.ratio'):
            try:
                st.append((float(r[i]), name[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
            except ValueError:
                pass
        if name.startswith('sm__inst_executed_pipe_') and name.endswith('.avg.pct_of_peak_sustained_active'):
            try:
                pipes.append((float(r[i]), name[len('sm__inst_executed_pipe_'):-len('.avg.pct_of_peak_sustained_active')]))
            except ValueError:
                pass
    print("  stalls per issue: " + ' '.join('%s=%.2f' % (n, v) for v, n in sorted(st, reverse=True)[:8]))
    print("  pipe utilisation %: " + ' '.join('%s=%.1f' % (n, v) for v, n in sorted(pipes, reverse=True)[:7]))
