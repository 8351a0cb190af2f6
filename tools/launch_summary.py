"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        hdr, start = r, i + 1
        break
iK, iV, iM = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[start:]:
    if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
        continue
    name = r[iK].split("(")[0].replace("void ", "")[:60]
    v = float(r[iV])
    tot += v
    agg[name][0] += 1
    agg[name][1] += v
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
print(f"total {tot / 1e3:.1f} us   (per unit: {tot / 1e3 / div:.1f} us, divisor {div})")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{t / 1e3:10.1f} us {t / 1e3 / div:9.1f} us/unit {c:6d}  {k}")
