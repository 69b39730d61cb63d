"""Summarise an .ncu-rep: per-kernel duration/DRAM/L2 and top source-level
stall sites. Usage: python tools/ncu_summary.py rep.ncu-rep [kernel_regex]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, data = raw[0], raw[1], raw[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread",
        "lts__t_sectors_op_write.sum", "lts__t_sectors_op_read.sum", "lts__t_sectors_op_red.sum"]
for d in data:
    name = d[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]
    if kre and not re.search(kre, name):
        continue
    parts = [name[:40]]
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            parts.append(f"{w.split('.')[0].replace('__', ':')}={d[i]}{units[i]}")
    print(" | ".join(parts))
if kre:
    src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "-k", f"regex:{kre}", "-c", "1"))))
    h = src[1]
    rows = [r for r in src[2:] if len(r) == len(h) and r[0] != "Address"]
    si, so, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
    f = lambda x: float(x) if x not in ("", "-") else 0.0
    tot = sum(f(r[si]) for r in rows)
    print(f"stall samples {tot:.0f}")
    for r in sorted(rows, key=lambda r: -f(r[si]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 15]:
        print(f"{f(r[si]) / max(tot, 1) * 100:5.1f}%  {r[ie]:>9}  {r[so][:100]}")
