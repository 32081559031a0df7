"""Instruction mix (executed warp instructions by opcode) and top stall PCs
from an ncu report's SASS source page.
    python tools/sass_mix.py report.ncu-rep KERNEL_REGEX"""
import csv
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ix = {k: hdr.index(k) for k in ("Source", "Instructions Executed", "Warp Stall Sampling (All Samples)")}
mix, stall = Counter(), Counter()
total = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    op = r[ix["Source"]].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    try:
        n = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    mix[o] += n
    total += n
    stall[o] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
print("total warp instructions", total)
for o, n in mix.most_common(30):
    print(f"{o:10s} {n:12d} {100 * n / total:5.1f}%  stall samples {stall[o]}")
