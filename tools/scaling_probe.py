"""Per-GPU share of the batch-sharded workloads: time fwd+bwd at B/N for N in
1,2,4,8 on one GPU (what each rank runs in the N-GPU job; no collectives in
the step).  Ideal strong scaling: t(B/N) = t(B)/N."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

def tm(prob, n=5):
    """fwd+bwd replayed from CUDA graphs (as bench.py times it)."""
    for _ in range(2):
        c = prob["fwd"](); prob["bwd"](c)
    torch.cuda.synchronize()
    g_f, g_b = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_f):
        gc = prob["fwd"]()
    with torch.cuda.graph(g_b):
        prob["bwd"](gc)
    for _ in range(2):
        g_f.replay(); g_b.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g_f.replay(); g_b.replay()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n

for wl in sys.argv[1:] or ["rglru", "s6"]:
    w = dict(bench.WORKLOADS[wl])
    base = None
    for N in (1, 2, 4, 8):
        prob = bench.build_problem(w, w["B"] // N, torch.device("cuda", 0))
        ms = tm(prob)
        base = base or ms
        print(f"{wl} N={N} B/N={w['B'] // N}: {ms:.3f} ms per rank-step, scaling efficiency {base / N / ms:.3f}", flush=True)
        del prob
        torch.cuda.empty_cache()
