"""Summarise one kernel of an `ncu --set full` report into the JSON bench.py
reads for the roofline's measured fields (profiles/ncu_<config>_force.json):
DRAM bytes per launch, fp64 pipe utilisation, issue activity, instructions.
Usage: python tools/ncu_to_json.py report.ncu-rep kernel-regex config out.json"""
import csv
import io
import json
import re
import subprocess
import sys

rep, pat, cfg, out = sys.argv[1:5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], dict(zip(rows[0], rows[1]))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
         "ms": 1e3, "msecond": 1e3, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}
pick = None
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if re.search(pat, d.get("Kernel Name", "")):
        pick = d
if pick is None:
    raise SystemExit(f"no kernel matching {pat}")


def f(k):
    """value in base units (bytes, microseconds, Hz)"""
    try:
        return float(str(pick.get(k, "")).replace(",", "")) * SCALE.get(units.get(k, ""), 1)
    except ValueError:
        return None


rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
res = {
    "kernel": re.sub(r"\(.*", "", pick["Kernel Name"]).replace("void b2md::", ""),
    "config": cfg,
    "dram_bytes_per_launch": (rd or 0) + (wr or 0),
    "dram_read_bytes": rd,
    "dram_write_bytes": wr,
    "gpu_time_us": f("gpu__time_duration.sum"),
    "fp64_pipe_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "warp_instructions": f("smsp__inst_executed.sum"),
    "sm_clock_hz": f("smsp__cycles_elapsed.avg.per_second"),
    "source": f"{rep} (ncu --set full --clock-control none; caches flushed by ncu between kernels)",
}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
