"""Micro-timing of the S6 operator kernels on a bench workload (CUDA events,
median of reps).  python tools/s6_micro.py [workload] [batch]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2602_08810_b200 import ops

wl = sys.argv[1] if len(sys.argv) > 1 else "s6"
w = dict(bench.WORKLOADS[wl])
B = int(sys.argv[2]) if len(sys.argv) > 2 else w["B"]
prob = bench.build_problem(w, B, torch.device("cuda", 0))
layer = prob["layer"]
args = (prob["u"], prob["pre"], layer.b_delta, layer.a_log, prob["Bk"], prob["Ck"], layer.D)


def timeit(fn, reps=7):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


y, ck = ops.s6_scan_fwd(*args)
print(f"{wl} B={B} geo={ops.s6_geometry(prob['u'].dtype, B, w['L'], w['H'], w['N'])}")
print(f"fwd (ckpt)    {timeit(lambda: ops.s6_scan_fwd(*args)):.3f} ms")
print(f"fwd (no ckpt) {timeit(lambda: ops.s6_scan_fwd(*args, ckpt=False)):.3f} ms")
print(f"bwd           {timeit(lambda: ops.s6_scan_bwd(*args, ck, prob['gy'])):.3f} ms")

# delta-input mode (the layer's GEMM-epilogue softplus): scan only, and the GEMM itself
if wl == "s6":
    import torch.nn.functional as F
    delta = F.softplus(prob["pre"] + layer.b_delta).contiguous()
    ad = (prob["u"], delta, layer.b_delta, layer.a_log, prob["Bk"], prob["Ck"], layer.D)
    yd, ckd = ops.s6_scan_fwd(*ad, flags=ops.S6_DELTA_IN)
    print(f"fwd delta-in  {timeit(lambda: ops.s6_scan_fwd(*ad, flags=ops.S6_DELTA_IN)):.3f} ms")
    print(f"bwd delta-in  {timeit(lambda: ops.s6_scan_bwd(*ad, ckd, prob['gy'], flags=ops.S6_DELTA_IN)):.3f} ms")
    T_ = prob["u"].shape[0] * prob["u"].shape[1]
    p1 = torch.randn((T_, layer.d_rank), device="cuda")
    wdp = layer.W_delta_proj.T.contiguous()
    print(f"gemm p1 W_dp        {timeit(lambda: ops.gemm_f32(p1, wdp)):.3f} ms")
    print(f"gemm p1 W_dp + sp   {timeit(lambda: ops.gemm_f32(p1, wdp, bias=layer.b_delta, act=ops.ACT_SOFTPLUS)):.3f} ms")
