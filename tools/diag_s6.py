"""Diagnose host-side overheads of the s6 bench step (CPU enqueue time, allocator)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
w = dict(bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "s6"])
prob = bench.build_problem(w, w["B"], torch.device("cuda", 0))
for _ in range(3):
    prob["bwd"](prob["fwd"]())
torch.cuda.synchronize()
st = torch.cuda.memory_stats()
a0 = st.get("num_device_alloc", 0); f0 = st.get("num_device_free", 0)
s = torch.cuda.current_stream()
for k in range(5):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(s); c0 = time.perf_counter()
    ctx = prob["fwd"](); c1 = time.perf_counter()
    e1.record(s)
    prob["bwd"](ctx); c2 = time.perf_counter()
    e2.record(s)
    torch.cuda.synchronize()
    print(f"step {k}: gpu fwd {e0.elapsed_time(e1):.3f} bwd {e1.elapsed_time(e2):.3f} ms | cpu fwd {1e3*(c1-c0):.3f} bwd {1e3*(c2-c1):.3f} ms")
st = torch.cuda.memory_stats()
print("device allocs", st.get("num_device_alloc", 0) - a0, "frees", st.get("num_device_free", 0) - f0)
# bench-like: no sync between steps
st = torch.cuda.memory_stats(); a0 = st.get("num_device_alloc", 0)
evs = []
ctx = None
c0 = time.perf_counter()
for k in range(6):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(s); t0 = time.perf_counter()
    ctx = prob["fwd"](); t1 = time.perf_counter()
    e[1].record(s)
    prob["bwd"](ctx); t2 = time.perf_counter()
    e[2].record(s)
    evs.append((e, 1e3 * (t1 - t0), 1e3 * (t2 - t1)))
torch.cuda.synchronize()
for e, cf, cb in evs:
    print(f"nosync: gpu fwd {e[0].elapsed_time(e[1]):.3f} bwd {e[1].elapsed_time(e[2]):.3f} | cpu fwd {cf:.3f} bwd {cb:.3f}")
st = torch.cuda.memory_stats()
print("device allocs (nosync)", st.get("num_device_alloc", 0) - a0, "reserved GB", torch.cuda.memory_reserved() / 1e9)
