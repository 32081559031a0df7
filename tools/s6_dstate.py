"""S6 scan throughput across d_state (v3 kernels take N = 16; other N the v2 path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_08810_b200 as lrx
from paper_2602_08810_b200 import ops

B, L, D = 4, 4096, 1024
for N in (16, 32, 64):
    layer = lrx.make_layer("s6", D, N, dtype="bf16", seed=0)
    u = torch.randn(B, L, D, device="cuda").to(torch.bfloat16)
    gy = torch.randn(B, L, D, device="cuda").to(torch.bfloat16)
    pre = torch.randn(B, L, D, device="cuda") * 0.5 - 2
    Bk = torch.randn(B, L, N, device="cuda"); Ck = torch.randn(B, L, N, device="cuda")
    p = (layer.b_delta, layer.a_log)
    def step():
        y, ck = ops.s6_scan_fwd(u, pre, *p, Bk, Ck, layer.D)
        ops.s6_scan_bwd(u, pre, *p, Bk, Ck, layer.D, ck, gy)
    step(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        step()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"s6 B={B} L={L} D={D} N={N}: {ms:.3f} ms fwd+bwd, {B * L * D * N / ms / 1e6:.0f} Gelem/s", flush=True)
