import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_2602_08810_b200 import ops
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
M, N, K = 131072, 1536, 96
A = torch.randn(M, K, device="cuda"); W = torch.randn(N, K, device="cuda") / 10; lo = ops.tf32_lo(W)
bias = torch.randn(N, device="cuda"); out = torch.empty(M, N, device="cuda")
print("act0 %.1f us" % t(lambda: ops.gemm_f32(A, W, lo, out=out)))
print("bias %.1f us" % t(lambda: ops.gemm_f32(A, W, lo, bias=bias, out=out)))
print("softplus %.1f us" % t(lambda: ops.gemm_f32(A, W, lo, bias=bias, act=ops.ACT_SOFTPLUS, out=out)))
print("bf16 out plain: %.1f us" % t(lambda: ops.gemm_bf16(A.bfloat16(), W.bfloat16(), out_dtype=torch.bfloat16)))
