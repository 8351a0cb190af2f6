"""Per-CUDA-line aggregation of an ncu report's SASS metrics (shared-memory
wavefronts, instructions, stall samples).  python tools/ncu_lines2.py rep [topN]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cs = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                    capture_output=True, text=True).stdout
sa = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                    capture_output=True, text=True).stdout
addr2line = {}
cur_file, cur_line = None, None
for row in csv.reader(cs.splitlines()):
    if len(row) == 2 and row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        continue
    if len(row) < 4:
        continue
    if row[0].strip().isdigit():
        cur_line = int(row[0])
        continue
    for x in row[:4]:
        if x.startswith("0x"):
            addr2line[x] = (cur_file, cur_line)
rows = list(csv.reader(sa.splitlines()))
h = rows[1]
ix = {k: h.index(k) for k in ("Address", "Source", "Instructions Executed", "L1 Wavefronts Shared",
                              "L1 Wavefronts Shared Ideal", "Warp Stall Sampling (All Samples)")}
agg = defaultdict(lambda: [0, 0, 0, 0])
tot = [0, 0, 0, 0]
for r in rows[2:]:
    if len(r) < len(h):
        continue
    key = addr2line.get(r[ix["Address"]], ("?", 0))
    vals = [int(r[ix[k]] or 0) for k in ("Instructions Executed", "L1 Wavefronts Shared",
                                         "L1 Wavefronts Shared Ideal", "Warp Stall Sampling (All Samples)")]
    for i, v in enumerate(vals):
        agg[key][i] += v
        tot[i] += v
print(f"total inst {tot[0]}, shared wavefronts {tot[1]} (ideal {tot[2]}), stall samples {tot[3]}")
print("by shared wavefronts:")
for key, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"  {key[0]}:{key[1]:<5d} inst {100 * v[0] / tot[0]:5.1f}%  wavefronts {100 * v[1] / max(tot[1], 1):5.1f}% "
          f"(x{v[1] / max(v[2], 1):.2f} of ideal)  stalls {100 * v[3] / max(tot[3], 1):5.1f}%")
print("by stall samples:")
for key, v in sorted(agg.items(), key=lambda kv: -kv[1][3])[:top]:
    print(f"  {key[0]}:{key[1]:<5d} inst {100 * v[0] / tot[0]:5.1f}%  wavefronts {100 * v[1] / max(tot[1], 1):5.1f}%  "
          f"stalls {100 * v[3] / max(tot[3], 1):5.1f}%")
