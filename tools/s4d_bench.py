"""S4D layer fwd+bwd: fused kernel vs the generic-operator path (LRX_S4D_GENERIC=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_08810_b200 as lrx

B, L, H, N = 8, 4096, 256, 64
layer = lrx.make_layer("s4d", H, N, dtype="f32", seed=0)
u = torch.randn(B, L, H, device="cuda")
gy = torch.randn(B, L, H, device="cuda")


def step():
    y, tape = layer.forward(u, tape=True)
    lrx.layer_backward(layer, tape, gy)


for mode in ("fused", "generic"):
    os.environ["LRX_S4D_GENERIC"] = "1" if mode == "generic" else "0"
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"s4d B={B} L={L} H={H} N={N} {mode}: {ms:.3f} ms fwd+bwd ({B * L * H * N / ms / 1e6:.1f} Gelem/s)")
