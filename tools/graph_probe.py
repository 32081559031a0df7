"""Can a workload's fwd+bwd step be captured in one CUDA graph?  Times eager vs replay."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
wl = sys.argv[1] if len(sys.argv) > 1 else "lru"
w = dict(bench.WORKLOADS[wl])
prob = bench.build_problem(w, w["B"], torch.device("cuda", 0))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        ctx = prob["fwd"](); prob["bwd"](ctx)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g):
        ctx = prob["fwd"]()
        out = prob["bwd"](ctx)
except Exception as e:
    print("capture failed:", type(e).__name__, str(e)[:300]); sys.exit(0)
def tm(fn, n=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
def eager():
    c = prob["fwd"](); prob["bwd"](c)
print(wl, "eager %.3f ms" % tm(eager), "graph %.3f ms" % tm(g.replay))
