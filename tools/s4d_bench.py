"""S4D layer fwd+bwd: fused kernel vs the generic-operator path (LRX_S4D_GENERIC=1),
constant and per-step (asynchronous) steps, over a few shapes.
    python tools/s4d_bench.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_08810_b200 as lrx  # noqa: E402

SHAPES = [(8, 4096, 256, 64), (1, 65536, 64, 64), (2, 16384, 32, 16)]


def bench(B, L, H, N, asyn, mode):
    os.environ["LRX_S4D_GENERIC"] = "1" if mode == "generic" else "0"
    layer = lrx.make_layer("s4d", H, N, "zoh", asynchronous=asyn, dtype="f32", seed=0)
    u = torch.randn(B, L, H, device="cuda")
    gy = torch.randn(B, L, H, device="cuda")
    deltas = torch.rand(B, L, device="cuda") * 2 + 0.1 if asyn else None

    def step():
        y, tape = layer.forward(u, deltas=deltas, tape=True)
        lrx.layer_backward(layer, tape, gy)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print(f"s4d B={B} L={L} H={H} N={N} {'async' if asyn else 'const'} {mode}: {ms:.3f} ms fwd+bwd "
          f"({B * L * H * N / ms / 1e6:.1f} Gelem/s)", flush=True)


for shp in SHAPES:
    for asyn in (False, True):
        for mode in ("fused", "generic"):
            try:
                bench(*shp, asyn, mode)
            except torch.OutOfMemoryError:
                print(f"s4d {shp} {asyn} {mode}: OOM")
                torch.cuda.empty_cache()
