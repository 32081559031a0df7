"""Large projection GEMMs (RG-LRU gate shapes): tcgen05 3xTF32 vs cuBLAS fp32 / 1xTF32."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_08810_b200 import ops


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for M, N, K in ((131072, 2560, 2560), (131072, 256, 256), (65536, 1536, 1536)):
    A = torch.randn(M, K, device="cuda"); W = torch.randn(N, K, device="cuda"); lo = ops.tf32_lo(W)
    fl = 2 * M * N * K
    ms = t(lambda: ops.gemm_f32(A, W, lo))
    torch.backends.cuda.matmul.allow_tf32 = False
    ms32 = t(lambda: A @ W.T)
    torch.backends.cuda.matmul.allow_tf32 = True
    mstf = t(lambda: A @ W.T)
    torch.backends.cuda.matmul.allow_tf32 = False
    G = torch.randn(M, N, device="cuda")
    mtn = t(lambda: ops.gemm_f32_tn(G, A))
    print(f"M={M} N={N} K={K}: tcgen05 3xTF32 {ms:.3f} ms ({fl / ms / 1e9:.0f} TF/s useful, {3 * fl / ms / 1e9:.0f} issued)"
          f" | cuBLAS fp32 {ms32:.3f} ms ({fl / ms32 / 1e9:.0f}) | cuBLAS 1xTF32 {mstf:.3f} ms ({fl / mstf / 1e9:.0f})"
          f" | tn (G^T A) {mtn:.3f} ms ({fl / mtn / 1e9:.0f})", flush=True)
    del A, W, lo, G
    torch.cuda.empty_cache()
