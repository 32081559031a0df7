"""Per-token decode latency: eager Layer.step vs StepGraph replay.
    python tools/decode_bench.py [d_model] [batch]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_08810_b200 as lrx

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
T = 200
for kind, n, dt in (("s5", 128, "f32"), ("lru", 64, "f32"), ("s6", 16, "bf16"), ("rglru", None, "f32"),
                    ("s4d", 16, "f32")):
    layer = lrx.make_layer(kind, m, n, dtype=dt, seed=0)
    u = torch.randn(B, T, m, device="cuda").to(layer.io_dtype)
    st = layer.init_state(B)
    for k in range(10):
        layer.step(st, u[:, k])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(T):
        y, st = layer.step(st, u[:, k])
    torch.cuda.synchronize()
    te = (time.perf_counter() - t0) / T * 1e6
    g = layer.step_graph(layer.init_state(B))
    for k in range(10):
        g.step(u[:, k])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(T):
        g.step(u[:, k])
    torch.cuda.synchronize()
    tg = (time.perf_counter() - t0) / T * 1e6
    print(f"{kind:6s} d_model={m} batch={B}: eager {te:7.1f} us/token   graph {tg:7.1f} us/token", flush=True)
