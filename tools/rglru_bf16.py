"""RG-LRU C4 shape with bf16 I/O (optional dtype): fwd / bwd per kernel family."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

w = dict(bench.WORKLOADS["rglru"], dtype="bf16")
prob = bench.build_problem(w, 64, torch.device("cuda", 0))
for mode in ("auto", "tma", "lookback", "stream"):
    os.environ["LRX_RGLRU_MODE"] = mode
    try:
        ctx = prob["fwd"]()
        for _ in range(2):
            prob["bwd"](prob["fwd"]())
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        ctx = prob["fwd"]()
        ev[1].record()
        prob["bwd"](ctx)
        ev[2].record()
        torch.cuda.synchronize()
        print(f"bf16 {mode}: fwd {ev[0].elapsed_time(ev[1]):.3f} ms  bwd {ev[1].elapsed_time(ev[2]):.3f} ms", flush=True)
    except Exception as e:
        print(mode, "failed:", e)
