"""Opcode histogram of a kernel's SASS between two addresses (or whole kernel).
    python tools/sass_stats.py file.sass [lo_hex hi_hex]"""
import re
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 62
ins = []
for ln in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        a = int(m.group(1), 16)
        op = re.sub(r"^@!?U?P\w+\s+", "", m.group(2).strip()).split()[0]
        if lo <= a < hi:
            ins.append(op)
c = Counter(o.split(".")[0] for o in ins)
print(len(ins), "instructions")
for k, v in c.most_common(40):
    print(f"{v:6d} {k}")
