"""Per-kernel SASS opcode counts of the shipped liblrx.so (cuobjdump -sass):
the Blackwell-native instructions that prove the tensor-core / TMA / packed
paths (UTCHMMA = tcgen05.mma, LDTM = tcgen05.ld, UTMALDG / UTMASTG = TMA
tensor load / store, UBLKCP = bulk copy, SYNCS = mbarrier, FFMA2 / FMUL2 /
FADD2 = packed fp32x2, MUFU.EX2 / RCP / RSQ ...).  Static counts (one per
instruction in the binary, not executed counts).
    python tools/sass_opcodes.py [liblrx.so] > profiles/sass_opcodes.json"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = ("UTCHMMA", "UTCQMMA", "UTCMMA", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMACMDFLUSH", "UBLKCP", "SYNCS",
        "FFMA2", "FMUL2", "FADD2", "MUFU.EX2", "MUFU.RCP", "MUFU.RSQ", "MUFU.SQRT", "MUFU.LG2", "MUFU.SIN",
        "MUFU.COS", "SHFL", "LDS", "STS", "LDG", "STG", "FFMA", "FMUL", "DFMA", "HMMA")


def main(lib):
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    out = {}
    for block in re.split(r"\n\s+Function : ", sass)[1:]:
        name = block.split("\n", 1)[0].strip()
        ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*(?:\.[A-Z0-9_]+)*)", block)
        cnt = collections.Counter()
        for op in ops:
            base = op.split(".")[0]
            key = "MUFU." + op.split(".")[1] if base == "MUFU" and "." in op else base
            if key in KEEP:
                cnt[key] += 1
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip() or name
        out[dem[:200]] = {"total": len(ops), **dict(sorted(cnt.items()))}
    tot = collections.Counter()
    for v in out.values():
        for k, n in v.items():
            tot[k] += n
    return {"library": os.path.relpath(lib, ROOT), "n_kernels": len(out), "totals": dict(sorted(tot.items())),
            "kernels": dict(sorted(out.items()))}


if __name__ == "__main__":
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2602_08810_b200", "liblrx.so")
    json.dump(main(lib), sys.stdout, indent=1)
    print()
