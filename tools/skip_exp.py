import os, sys
sys.path.insert(0, "/root/repo") if os.path.exists("/root/repo") else None
import torch
from paper_2602_08810_b200 import ops
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
M, N, K = 131072, 256, 256
A = torch.randn(M, K, device="cuda"); Bt = torch.randn(N, K, device="cuda"); lo = ops.tf32_lo(Bt)
Cin = torch.randn(M, N, device="cuda"); cs = torch.randn(N, device="cuda"); out = torch.empty(M, N, device="cuda")
def two_pass():
    ops.gemm_f32(A, Bt, lo, out=out)
    out.addcmul_(Cin, cs)
print("fused skip %.1f us" % t(lambda: ops.gemm_f32(A, Bt, lo, Cin=Cin, colscale=cs, out=out)),
      "| plain + addcmul %.1f us" % t(two_pass), "| addcmul alone %.1f" % t(lambda: out.addcmul_(Cin, cs)))
x = torch.randn(M, 256, device="cuda"); y2 = torch.randn(M, 256, device="cuda")
print("gD reduce_rows dot %.1f us" % t(lambda: ops.reduce_rows(x, M, 256, other=y2)))
