"""RG-LRU C4 fwd / bwd at a per-rank batch share (B = 64/N), graph-replayed:
the plan sweep behind the multi-GPU per-rank efficiency.  Usage:
python tools/rg_smallb.py 32 16 8   (env overrides LRX_RGLRU_* apply)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench


from rg_smallb_util import tm  # noqa: E402


w = dict(bench.WORKLOADS[os.environ.get("WL", "rglru")])
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("LRX_RGLRU")) or "default"
for B in [int(x) for x in sys.argv[1:]] or [32, 16, 8]:
    prob = bench.build_problem(w, B, torch.device("cuda", 0))
    ctx = prob["fwd"]()
    f = tm(prob["fwd"])
    b = tm(lambda: prob["bwd"](ctx))
    ideal = 20.26 * B / 64
    print(f"B={B:3d} fwd {f:.3f} bwd {b:.3f} total {f + b:.3f} ms (B/64 of C4 = {ideal:.3f}; eff {ideal / (f + b):.3f}) [{tag}]",
          flush=True)
    del prob, ctx
    torch.cuda.empty_cache()
