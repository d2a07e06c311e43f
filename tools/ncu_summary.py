"""Key metrics per kernel launch from an ncu report (details page).
Usage: python tools/ncu_summary.py report.ncu-rep [kernel-substring]"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "DRAM Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Avg. Active Threads Per Warp", "Waves Per SM"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
seen = {}
for row in rows[1:]:
    d = dict(zip(hdr, row))
    if flt not in d.get("Kernel Name", "") or d.get("Metric Name") not in WANT:
        continue
    key = (d["ID"], d["Kernel Name"][:60])
    seen.setdefault(key, []).append(f"{d['Metric Name']}={d['Metric Value']}{d['Metric Unit'] and ' ' + d['Metric Unit']}")
for (i, k), v in seen.items():
    print(f"[{i}] {k}\n    " + "\n    ".join(v))
