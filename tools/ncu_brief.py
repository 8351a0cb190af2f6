"""Brief ncu report: key throughput metrics, stall reasons and SASS hot spots."""
import csv, subprocess, sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, v = r[0], r[2]
keys = ['Kernel Name', 'Block Size', 'gpu__time_duration.sum', 'smsp__inst_executed.sum',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum']
for i, k in enumerate(h):
    if k in keys or ('smsp__average_warps_issue_stalled' in k and k.endswith('ratio')):
        try:
            if 'stalled' in k and float(v[i]) < 0.05:
                continue
        except ValueError:
            pass
        print(f"{k:90s} {v[i]}")
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    s = list(csv.reader(src.splitlines()))
    hh, rows = s[1], s[2:]
    ie, ws = hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(x[ie]) for x in rows) or 1
    stot = sum(int(x[ws]) for x in rows) or 1
    seg = int(sys.argv[2])
    for st in range(0, len(rows), seg):
        ch = rows[st:st + seg]
        a = sum(int(x[ie]) for x in ch)
        b = sum(int(x[ws]) for x in ch)
        if a / tot > 0.02 or b / stot > 0.02:
            ops = [x[1].split()[1] if x[1].strip().startswith('@') else x[1].split()[0] for x in ch]
            c = Counter(o.split('.')[0] for o in ops)
            print(f"{st:5d} inst {100 * a / tot:5.1f}% stall {100 * b / stot:5.1f}%  ", dict(c.most_common(7)))
