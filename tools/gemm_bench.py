"""Time lrx_gemm_f32 (tcgen05 3xTF32) against torch fp32 matmul on the S5 shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_08810_b200 import ops


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for M, N, K in [(131072, 256, 256), (8192, 128, 128), (131072, 128, 256)]:
    A = torch.randn(M, K, device="cuda")
    Bt = torch.randn(N, K, device="cuda")
    lo = ops.tf32_lo(Bt)
    W = Bt.T.contiguous()
    out = torch.empty(M, N, device="cuda")
    ms_l = t(lambda: ops.gemm_f32(A, Bt, lo, out=out))
    ms_t = t(lambda: torch.matmul(A, W, out=out))
    fl = 2 * M * N * K
    byt = 4 * (M * K + M * N)
    print(f"M={M} N={N} K={K}: tcgen05 3xTF32 {ms_l*1e3:8.1f} us ({fl/ms_l/1e9:6.1f} TFLOP/s, {byt/ms_l/1e6:6.0f} GB/s) | "
          f"torch fp32 {ms_t*1e3:8.1f} us ({fl/ms_t/1e9:6.1f} TFLOP/s)")
