"""S5-shaped GEMM calls (with and without the fused skip epilogue)."""
import os, sys
root = sys.argv[1] if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
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
    return a.elapsed_time(b) / reps * 1e3


M, N, K = 131072, 256, 256
A = torch.randn(M, K, device="cuda"); Bt = torch.randn(N, K, device="cuda"); lo = ops.tf32_lo(Bt)
Cin = torch.randn(M, N, device="cuda"); cs = torch.randn(N, device="cuda"); out = torch.empty(M, N, device="cuda")
print(root, "plain %.1f us" % t(lambda: ops.gemm_f32(A, Bt, lo, out=out)),
      "| skip %.1f us" % t(lambda: ops.gemm_f32(A, Bt, lo, Cin=Cin, colscale=cs, out=out)),
      "| tn %.1f us" % (t(lambda: ops.gemm_f32_tn(A, Cin)) if hasattr(ops, "gemm_f32_tn") else 0))
