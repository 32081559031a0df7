"""Sweep RG-LRU TMA plan overrides (LRX_RGLRU_LW / _STAGES / _SEGS) at the
per-rank batch of the 1/2/4/8-GPU runs; prints fwd / bwd ms per setting.
usage: python tools/rglru_sweep.py B [B ...]   (env sets are listed below)"""
import itertools, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

SETS = [dict(), dict(LRX_RGLRU_LW="128"), dict(LRX_RGLRU_LW="128", LRX_RGLRU_STAGES="16"),
        dict(LRX_RGLRU_LW="32", LRX_RGLRU_STAGES="16"), dict(LRX_RGLRU_LW="64", LRX_RGLRU_STAGES="12")]
if os.environ.get("SWEEP"):  # "PF:SEGS,..." e.g. "4:1,8:1,16:2"
    SETS = [{k: v for k, v in (("LRX_RGLRU_PF", a), ("LRX_RGLRU_SEGS", b)) if v != "a"}
            for a, b in (x.split(":") for x in os.environ["SWEEP"].split(","))]


def tm(f, n=5):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


w = dict(bench.WORKLOADS["rglru"])
for B in [int(x) for x in sys.argv[1:]] or [8, 64]:
    prob = bench.build_problem(w, B, torch.device("cuda", 0))
    for env in SETS:
        for k in ("LRX_RGLRU_LW", "LRX_RGLRU_STAGES", "LRX_RGLRU_SEGS", "LRX_RGLRU_PF"):
            os.environ.pop(k, None)
        os.environ.update(env)
        ctx = prob["fwd"]()
        f = tm(prob["fwd"])
        b = tm(lambda: prob["bwd"](ctx))
        print(f"B={B} {env}: fwd {f:.3f} ms  bwd {b:.3f} ms  total {f + b:.3f}", flush=True)
    del prob
    torch.cuda.empty_cache()
