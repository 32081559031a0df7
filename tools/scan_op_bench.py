"""Generic scan operator (lrx_scan_fwd / lrx_scan_bwd, _scan_kernels.py:17-153)
throughput: time-major [L, N] f32 / c64, per-step a, on device."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_08810_b200.scan import run_fwd
from paper_2602_08810_b200.autograd import pullback


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


for L, N, dt in ((4096, 1 << 18, torch.float32), (65536, 1 << 14, torch.float32), (4096, 1 << 17, torch.complex64),
                 (1 << 20, 1024, torch.float32)):
    a = (torch.rand(L, N, device="cuda") * 0.5 + 0.5).to(dt)
    b = torch.randn(L, N, device="cuda").to(dt)
    ms = t(lambda: run_fwd(a, True, b, None))
    x = run_fwd(a, True, b, None)
    gx = torch.randn_like(b)
    mb = t(lambda: pullback(a, True, x, None, gx))
    es = a.element_size()
    print(f"L={L} N={N} {dt}: fwd {ms:.3f} ms ({3 * L * N * es / ms / 1e6:.0f} GB/s)  bwd {mb:.3f} ms "
          f"({5 * L * N * es / mb / 1e6:.0f} GB/s: a, x, gx in; g, ga out)", flush=True)
    del a, b, x, gx
    torch.cuda.empty_cache()
