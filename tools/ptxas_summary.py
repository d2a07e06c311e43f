"""Registers / spills per kernel from an nvcc -Xptxas -v log (demangled names).
Usage: python tools/ptxas_summary.py paper_1507_07548_b200/lib/ptxas.log [filter]"""
import re
import subprocess
import sys

log = open(sys.argv[1]).read().splitlines()
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
rows = []
for ln in log:
    m = re.search(r"Compiling entry function '([^']+)'|Function properties for (\S+)", ln)
    if m:
        cur = m.group(1) or m.group(2)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)))
        rows.append([cur, None, spill])
    m = re.search(r"Used (\d+) registers", ln)
    if m and rows and rows[-1][1] is None:
        rows[-1][1] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True,
                       text=True).stdout.splitlines()
for (mangled, regs, spill), nm in zip(rows, names):
    if flt in nm:
        nm = re.sub(r"\(b2md::[^)]*\)", "", nm)
        print(f"{regs if regs is not None else -1:>4} regs  spill {spill[0]:>4}/{spill[1]:<4} {nm}")
