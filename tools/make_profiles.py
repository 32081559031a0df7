"""Summarise a round's gpurun_out captures into profiles/ (tracked):
launch lists -> profiles/<tag>_launches_<wl>.json (last step only, with the
step share of every kernel), full captures -> profiles/<tag>_ncu_full_<wl>.json,
and profiles/ncu_traffic.json (DRAM bytes per launch of each workload's
dominant kernel, read by bench.py for roofline.traffic).
    python tools/make_profiles.py TAG"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import full, launches  # noqa: E402

tag = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles")
os.makedirs(out, exist_ok=True)
go = os.path.join(ROOT, "gpurun_out")
# dominant kernel per workload (the bench.py probe), matched on the launch list
DOM = {"rglru": r"bwd_rev2_kernel", "s6": r"s6v3::bwd_kernel", "s6_long": r"s6v3::bwd(_agg)?_kernel",
       "s5": r"gemm_tf32x3_kernel", "lru": r"mimo::bwd_kernel", "s6_layer": r"s6v3::bwd_kernel",
       "rglru_layer": r"gemm_tf32x3_kernel"}
traffic = {}
for wl, pat in DOM.items():
    path = os.path.join(go, f"launches_{wl}_{tag}.csv")
    if not os.path.exists(path):
        continue
    rs = launches(path)
    # prof_step runs 2 identical steps after the setup kernels: the step is the
    # longest K with names[-2K:-K] == names[-K:]; keep the second (warm) copy
    names = [r["kernel"] for r in rs]
    K = next(k for k in range(len(rs) // 2, 0, -1) if names[-2 * k:-k] == names[-k:])
    half = rs[-K:]
    tot = sum(r.get("gpu__time_duration.sum", 0) for r in half)
    for r in half:
        r["step_share"] = r.get("gpu__time_duration.sum", 0) / tot if tot else None
    json.dump({"step_ns": tot, "launches": half}, open(os.path.join(out, f"{tag}_launches_{wl}.json"), "w"), indent=1)
    dom = [r for r in half if re.search(pat, r["kernel"])]
    if dom:
        if wl in ("s5", "rglru_layer"):  # one GEMM launch: the one with the most DRAM traffic
            dom = [max(dom, key=lambda r: r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"])]
        b = sum(r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"] for r in dom)
        traffic[wl] = {"probe": b,
                       "kernels": [r["kernel"][:80] for r in dom], "source": f"profiles/{tag}_launches_{wl}.json"}
    print(wl, f"step {tot / 1e3:.1f} us", f"dominant {[r['kernel'][:40] for r in dom]}")
for wl in ("s6", "s5", "rglru", "s6_long", "s6_layer"):
    rep = os.path.join(go, f"prof_{wl}_{tag}.ncu-rep")
    if os.path.exists(rep):
        json.dump(full(rep), open(os.path.join(out, f"{tag}_ncu_full_{wl}.json"), "w"), indent=1)
        print("full", wl)
json.dump(traffic, open(os.path.join(out, "ncu_traffic.json"), "w"), indent=1)
