"""Summarise an ncu report (or a launch-list CSV) into JSON for profiles/.
    python tools/ncu_summary.py report.ncu-rep > out.json
    python tools/ncu_summary.py --launches launches.csv > out.json"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        rec = {"kernel": row[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                rec[k] = f"{row[i]} {units[i]}".strip()
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(row[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        rec["top_stall_samples"] = [[n, v] for v, n in sorted(stalls, reverse=True)[:6]]
        res.append(rec)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value")}
    d = defaultdict(dict)
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        d[(int(r[0]), r[ix["Kernel Name"]])][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    return [{"id": i, "kernel": k, **m} for (i, k), m in sorted(d.items())]


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        json.dump(launches(sys.argv[2]), sys.stdout, indent=1)
    else:
        json.dump(full(sys.argv[1]), sys.stdout, indent=1)
