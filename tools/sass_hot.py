"""Top SASS lines by stall samples: python tools/sass_hot.py report KERNEL_REGEX [N]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
i_src, i_st = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
recs = []
for n, r in enumerate(rows[2:]):
    if len(r) < len(hdr):
        continue
    try:
        recs.append((int(r[i_st]), n, r[i_src].strip()))
    except ValueError:
        pass
tot = sum(s for s, _, _ in recs)
print("total samples", tot)
for s, n, src in sorted(recs, reverse=True)[:N]:
    print(f"{s:7d} {100*s/tot:5.1f}%  #{n:5d}  {src}")
