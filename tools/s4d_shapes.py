"""S4D fused kernel vs the generic operator path across shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_08810_b200 as lrx

for B, L, H, N in ((8, 4096, 256, 64), (1, 65536, 64, 64), (1, 16384, 256, 16), (2, 8192, 128, 32)):
    layer = lrx.make_layer("s4d", H, N, dtype="f32", seed=0)
    u = torch.randn(B, L, H, device="cuda"); gy = torch.randn(B, L, H, device="cuda")
    res = []
    for mode in ("0", "1", "auto"):
        os.environ.pop("LRX_S4D_GENERIC", None)
        if mode != "auto":
            os.environ["LRX_S4D_GENERIC"] = mode
        def step():
            y, tape = layer.forward(u, tape=True)
            lrx.layer_backward(layer, tape, gy)
        step(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            step()
        b.record(); torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / 3)
    print(f"B={B} L={L} H={H} N={N}: fused {res[0]:.2f} ms  generic {res[1]:.2f} ms  auto {res[2]:.2f} ms", flush=True)
