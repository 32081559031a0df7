"""Time the RG-LRU step paths alone (CUDA events, 200 back-to-back tokens)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_08810_b200 as lrx
from paper_2602_08810_b200 import _lib

for B, W in ((1, 1024), (8, 2560), (16, 2560), (1, 4096)):
    layer = lrx.make_layer("rglru", W, dtype="f32", seed=0)
    st = layer.init_state(B)
    u = torch.randn(B, W, device="cuda")
    y = torch.empty(B, W, device="cuda")
    lib = _lib.lib()
    def fused():
        lib.lrx_rglru_step_fused(0, _lib.ptr(st.x), _lib.ptr(u), _lib.ptr(layer.W_r), _lib.ptr(layer.W_i),
                                 _lib.ptr(layer.lambda_param), _lib.ptr(layer.b_r), _lib.ptr(layer.b_i), _lib.ptr(y),
                                 B, W, _lib.stream())
    def gemv():
        qr = u @ layer.W_r.T
        qi = u @ layer.W_i.T
        lib.lrx_rglru_step(0, _lib.ptr(st.x), _lib.ptr(u), _lib.ptr(qr), _lib.ptr(qi), _lib.ptr(layer.lambda_param),
                           _lib.ptr(layer.b_r), _lib.ptr(layer.b_i), _lib.ptr(y), B, W, _lib.stream())
    for name, f in (("fused", fused), ("cublas+step", gemv)):
        for _ in range(20):
            f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(200):
            f()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 200 * 1e3
        print(f"B={B} W={W} {name}: {us:.1f} us/token  ({2 * W * W * 4 / us / 1e3:.0f} GB/s weights)", flush=True)
