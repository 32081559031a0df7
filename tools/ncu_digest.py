"""Digest an ncu --set full report: headline metrics, stall reasons and the
per-opcode stall breakdown from the SASS source page.
    python tools/ncu_digest.py report.ncu-rep [kernel-regex]"""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_warps",
        "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(path, regex=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    names = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        names.append(name)
        print("==", name[:110])
        for k in KEYS:
            if k in hdr:
                print(f"   {k:60s} {r[hdr.index(k)]} {units[hdr.index(k)]}")
        st = sorted(((num(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for i, h in enumerate(hdr)
                     if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")), reverse=True)
        print("   stalls:", [(n, int(v)) for v, n in st[:9]])
    for name in sorted(set(names)):
        short = name.split("(")[0].split()[-1].split("<")[0]
        if regex and regex not in name:
            continue
        src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                              "regex:" + short], capture_output=True, text=True).stdout
        srows = list(csv.reader(src.splitlines()))
        if len(srows) < 3:
            continue
        h = srows[1]
        seen, byop = set(), collections.defaultdict(collections.Counter)
        cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
        for r in srows[2:]:
            if len(r) != len(h) or r[0] in seen:
                continue
            seen.add(r[0])
            toks = r[1].split()
            if not toks:
                continue
            op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
            for c in cols:
                byop[op][c] += num(r[h.index(c)])
            byop[op]["inst"] += num(r[h.index("Instructions Executed")])
        print("== per-opcode:", short)
        for op, c in sorted(byop.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "inst"))[:14]:
            s = sum(v for k, v in c.items() if k != "inst")
            print(f"   {op:8s} samples {s:7.0f} inst {c['inst'] / 1e6:8.1f}M",
                  {k.replace("stall_", ""): int(v) for k, v in c.most_common(5) if k != "inst"})


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
