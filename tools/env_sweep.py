"""Time one workload's fwd / bwd (CUDA-graph replays) at several per-rank
batches under several env settings (kernel plan overrides).
usage: python tools/env_sweep.py WORKLOAD "B1,B2" "K=V;K=V|K=V|-"   ('-' = no overrides)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench


def graph_ms(f, n=10):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


wl, bs, sets = sys.argv[1], [int(x) for x in sys.argv[2].split(",")], sys.argv[3].split("|")
w = dict(bench.WORKLOADS[wl])
keys = set()
for st in sets:
    keys |= {kv.split("=")[0] for kv in st.split(";") if "=" in kv}
for B in bs:
    prob = bench.build_problem(w, B, torch.device("cuda", 0))
    for st in sets:
        for k in keys:
            os.environ.pop(k, None)
        env = dict(kv.split("=", 1) for kv in st.split(";") if "=" in kv)
        os.environ.update(env)
        ctx = prob["fwd"]()
        f = graph_ms(prob["fwd"])
        b = graph_ms(lambda: prob["bwd"](ctx))
        print(f"{wl} B={B} {st}: fwd {f:.3f} ms  bwd {b:.3f} ms  total {f + b:.3f}", flush=True)
    del prob
    torch.cuda.empty_cache()
