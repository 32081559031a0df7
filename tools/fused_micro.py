"""Time the fused MIMO projection + scan kernels alone at C2 / C1 shapes
(LRX_MIMO_FUSED_ORDER=row: row-major unit claims)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_08810_b200 import ops

def tm(fn, n=10):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3

for (B, L, m, P) in [(32, 4096, 256, 128), (8, 1024, 128, 64)]:
    dev = "cuda"
    u2 = torch.randn(B * L, m, device=dev)
    wt = torch.randn(2 * P, m, device=dev) / m ** 0.5
    A, Al = ops.mimo_fused_weights(wt, ops.tf32_lo(wt))
    abar = torch.polar(torch.full((P,), 0.9, device=dev), torch.rand(P, device=dev)).to(torch.complex64)
    scale = torch.ones(P, dtype=torch.complex64, device=dev)
    x, _ = ops.mimo_fused_fwd(A, Al, u2, abar, scale, B, L, want_bu=False)
    f = tm(lambda: ops.mimo_fused_fwd(A, Al, u2, abar, scale, B, L, want_bu=False))
    b = tm(lambda: ops.mimo_fused_bwd(A, Al, u2, 2.0, abar, scale, x))
    g = tm(lambda: ops.gemm_f32(u2, wt, ops.tf32_lo(wt)))
    print(f"B{B} L{L} m{m} P{P}: fused fwd {f:.1f} us, bwd {b:.1f} us; plain GEMM u W^T {g:.1f} us", flush=True)
