"""Summarise ncu --set full reports into profiles/ (JSON + markdown)."""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
}
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "msecond": 1e-3}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main():
    out, md = {}, ["| kernel | time (us) | DRAM read+write (MB) | DRAM GB/s | DRAM % | FP64 pipe % | occupancy % | regs |",
                   "|---|---|---|---|---|---|---|---|"]
    for rep in sys.argv[2:]:
        hdr, units, data = rows(rep)
        idx = {k: hdr.index(k) for k in WANT if k in hdr}
        iK = hdr.index("Kernel Name")
        for r in data:
            name = r[iK].split("(")[0].replace("void ", "")
            rec = {}
            for k, key in WANT.items():
                if k in idx:
                    v = r[idx[k]]
                    try:
                        v = float(v.replace(",", ""))
                    except ValueError:
                        continue
                    rec[key] = v * UNITS.get(units[idx[k]], 1.0)
            if name in out:
                continue
            t = rec.get("duration", float("nan"))
            b = rec.get("dram_read", 0) + rec.get("dram_write", 0)
            rec["dram_bytes"] = b
            rec["dram_gbs"] = b / t / 1e9 if t else None
            rec["report"] = rep
            out[name] = rec
            md.append(f"| `{name[:60]}` | {t * 1e6:.1f} | {b / 1e6:.1f} | {rec['dram_gbs']:.0f} | "
                      f"{rec.get('dram_pct', 0):.1f} | {rec.get('fp64_pipe_pct', 0):.1f} | "
                      f"{rec.get('occupancy_pct', 0):.1f} | {rec.get('regs', 0):.0f} |")
    with open(sys.argv[1] + ".json", "w") as fh:
        json.dump(out, fh, indent=1)
    with open(sys.argv[1] + ".md", "w") as fh:
        fh.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
