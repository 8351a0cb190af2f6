"""Per-source-line totals (instructions executed, stall samples) from an
ncu report: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines = {}
fname = None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        key = (fname, int(r[0]))
    except ValueError:
        continue
    num = lambda k: int(d.get(k, "0")) if d.get(k, "0").isdigit() else 0
    lines[key] = (r[1][:90], num("Instructions Executed"),
                  num("Warp Stall Sampling (All Samples)"))
tot_i = sum(v[1] for v in lines.values()) or 1
tot_s = sum(v[2] for v in lines.values()) or 1
print(f"total instructions {tot_i}, stall samples {tot_s}")
for (f, ln), (src, ni, ns) in sorted(lines.items(), key=lambda kv: -kv[1][2])[:top]:
    print(f"{f}:{ln:4d} inst {100*ni/tot_i:5.1f}% stall {100*ns/tot_s:5.1f}%  {src}")
