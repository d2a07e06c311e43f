"""Warp-stall samples and executed instructions of one kernel in an ncu report,
attributed to CUDA source lines through the cubin's line table.
Usage: python tools/ncu_lines.py report.ncu-rep mangled-kernel-name cubin ncu-kernel-regex [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, name, cubin, kre = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(sass) if l.startswith("//---") and name in l)
off2line, cur = {}, None
for l in sass[start + 1:]:
    if l.startswith("//---"):
        break
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ix, ad = hdr.index("Instructions Executed"), hdr.index("Address")
sm = hdr.index("Warp Stall Sampling (All Samples)")
seq, seen = [], set()
for r in rows[2:]:
    try:
        n, a = int(r[ix] or 0), int(r[ad], 16)
    except (ValueError, IndexError):
        continue
    if a in seen:
        break
    seen.add(a)
    seq.append((a, n, int(r[sm] or 0)))
base = seq[0][0]
samp, inst = collections.Counter(), collections.Counter()
for a, n, s in seq:
    ln = off2line.get(a - base, ("?", 0))
    samp[ln] += s
    inst[ln] += n
tot = max(1, sum(samp.values()))
print(f"samples {tot}  instructions {sum(inst.values())}")
files = {}
for (f, l), s in samp.most_common(top):
    if f not in files:
        try:
            files[f] = open(f).read().split("\n")
        except OSError:
            files[f] = []
    text = files[f][l - 1].strip()[:70] if 0 < l <= len(files[f]) else ""
    print(f"{s / tot * 100:5.1f}% {inst[(f, l)]:10d} {f.split('/')[-1]}:{l} {text}")
