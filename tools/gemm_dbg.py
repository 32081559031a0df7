import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_08810_b200 import ops, _lib
torch.manual_seed(0)
for K, M, N in [(32, 128, 64), (64, 128, 128), (4096, 256, 256)]:
    A = torch.randn(K, M, device="cuda"); B = torch.randn(K, N, device="cuda")
    ks = _lib.i64(); _lib.lib().lrx_gemm_f32_tn_splits(M, N, K, _lib.ref(ks))
    part = torch.full((ks.value, M * N), 7.0, device="cuda")
    _lib.check(_lib.lib().lrx_gemm_f32_tn(_lib.ptr(A), _lib.ptr(B), _lib.ptr(part), M, N, K, 1.0, _lib.stream()))
    torch.cuda.synchronize()
    ref = A.double().T @ B.double()
    C = part.view(ks.value, M, N).sum(0)
    print(K, M, N, "splits", ks.value, "part stats", part.abs().max().item(), (part == 7.0).float().mean().item(),
          "rel", ((C.double() - ref).abs().max() / ref.abs().max()).item())
    # is it the transpose?
    print("   rel vs B^T A", ((C.double().T - ref.T).abs().max() / ref.abs().max()).item() if M == N else "")
