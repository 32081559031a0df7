"""Opcode mix of the largest loops in a cuobjdump -sass listing.
    cuobjdump -sass -fun NAME obj.o > f.sass; python tools/sass_loops.py f.sass [N]"""
import collections
import re
import sys

ops = []
for l in open(sys.argv[1]).read().splitlines():
    m = re.match(r'\s+/\*([0-9a-f]+)\*/\s+(.*?);', l)
    if not m:
        continue
    toks = m.group(2).strip().split()
    if toks[0].startswith('@'):
        toks = toks[1:]
    tgt = re.search(r'BRA.*?(0x[0-9a-f]+)', m.group(2))
    ops.append((int(m.group(1), 16), toks[0], int(tgt.group(1), 16) if tgt else None))
loops = sorted(((a - t, t, a) for a, o, t in ops if t is not None and t < a), reverse=True)
for size, t, a in loops[: int(sys.argv[2]) if len(sys.argv) > 2 else 2]:
    body = [o for x, o, _ in ops if t <= x <= a]
    c = collections.Counter(o.split('.')[0] for o in body)
    print(f"loop {t:#x}..{a:#x}: {len(body)} instructions")
    print("  ", ", ".join(f"{k} {v}" for k, v in c.most_common(24)))
