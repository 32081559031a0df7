"""Benchmark: scan Gelem/s (B*L*H*N) fwd+bwd on B200, with the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl lrx|reference]

One JSON line on rank 0 (driver contract).  A step is one forward + backward
pass of the scan operator over one batch of synthetic inputs that are already
resident in HBM (the `value`); `e2e` is the same metric through the public
Python API with pinned HOST buffers and the H2D/D2H copies inside the timed
region.  Workloads are BASELINE.json's configs:

  lru     configs[0]  LRU   B=8  L=1024   H=128  N=64  (complex)    f32
  s5      configs[1]  S5    B=32 L=4096   H=256  P=128 (complex)    f32, ZOH
  s6      configs[2]  S6    B=16 L=8192   D=1536 N=16               bf16 I/O, fp32 accum
  rglru   configs[3]  RG-LRU B=64 L=16384 W=2560                    f32   (default)
  s6_long configs[4]  S6    B=1  L=2^20   D=2048 N=16               bf16 I/O, sequence-parallel

The default is the RG-LRU config: BASELINE.json's metric is the scan's HBM
throughput at 1/2/4/8 GPUs, and configs[3] is the config it names for the
8-GPU batch sharding ("Benchmark").  Multi-GPU: one process
per GPU (torchrun); the batch is split across ranks with no data-path
collective (total work fixed: strong scaling); time = max over ranks.

The operator boundary is the one a framework binds (paper_2602_08810_b200.ops):
for S6 / RG-LRU the dense projections producing (pre, B_k, C_k) / (qr, qi) are
outside the scan; for S5 / LRU the B and C
projections are part of the recurrence x = abar x + B u, y = Re(C x) + D u and
are inside the step.

`--impl reference` times the reference's own CPU algorithm (the oracle
restatement in oracle/port.py: numpy + the C restatement of the numba loops,
chunk-parallel over all host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

# The step allocates its outputs like any torch op (y, checkpoints, gradients:
# up to 1.6 GB each).  With large blocks unsplittable the caching allocator
# reuses them exactly step after step instead of splitting a freed block for
# a smaller request and calling cudaMalloc (host-blocking, ~3 ms per GB)
# inside the timed region.
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "max_split_size_mb:256")


ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "lru": dict(kind="lru", B=8, L=1024, H=128, N=64, dtype="f32", cfg=0),
    "s5": dict(kind="s5", B=32, L=4096, H=256, N=128, dtype="f32", cfg=1),
    "s6": dict(kind="s6", B=16, L=8192, H=1536, N=16, dtype="bf16", cfg=2),
    "rglru": dict(kind="rglru", B=64, L=16384, H=2560, N=1, dtype="f32", cfg=3),
    "s6_long": dict(kind="s6", B=1, L=2 ** 20, H=2048, N=16, dtype="bf16", cfg=4, seqpar=True),
    # drop-in layer level (make_layer forward(tape) + layer_backward): the input
    # projections on the tcgen05 GEMMs (bf16 kind::f16 / fp32 3xTF32) + the scan
    "s6_layer": dict(kind="s6", B=16, L=8192, H=1536, N=16, dtype="bf16", cfg=2, layer=True),
    "rglru_layer": dict(kind="rglru", B=64, L=16384, H=2560, N=1, dtype="f32", cfg=3, layer=True),
}
DEFAULT_WORKLOAD = "rglru"
L2_BYTES = 126 * 1024 * 1024
METRIC = "scan Gelem/s (B·L·H·N) fwd+bwd, HBM GB/s vs peak, at 1/2/4/8 B200"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _tensor_peak():
    """TF32 dense tensor peak = half the measured bf16 GEMM rate (Blackwell runs
    kind::tf32 at 1/2 the kind::f16 rate)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]) / 2, "measured bf16 / 2 (tf32)"
    except Exception:
        return 1590.0 / 2, "fallback bf16 / 2 (tf32)"


def _traffic(workload, kernel):
    """Per-launch DRAM bytes from the committed ncu capture (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload, {}).get(kernel)
    except Exception:
        return None


def _state_dims(w):
    """(lanes description, elements per step) for a workload dict."""
    return w["B"] * w["L"] * w["H"] * w["N"]


# ---------------------------------------------------------------------------
# clocks sampler (driver timing rules)

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.idx = device_index
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        rows = [r for r in self.rows if len(r) == 6 and r[0].replace(".", "").isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(float(r[0]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# GPU arm

def _lib_ws(nbytes, device):
    import torch
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def build_problem(w, B, device, L=None, group=None):
    """Synthetic inputs (reference init + N(0,1) activations, on device) and a
    step function fwd+bwd at the operator boundary.  `L` overrides the
    sequence length (this rank's slice in sequence-parallel mode)."""
    import torch

    import paper_2602_08810_b200 as lrx
    from paper_2602_08810_b200 import ops

    kind, H, N = w["kind"], w["H"], w["N"]
    L = L or w["L"]
    layer = lrx.make_layer(kind, H, None if kind == "rglru" else (N if kind != "s5" else 2 * N), dtype=w["dtype"],
                           seed=0, device=device)
    g = torch.Generator(device=device).manual_seed(1234 + (torch.distributed.get_rank()
                                                           if torch.distributed.is_initialized() else 0))
    io = layer.io_dtype
    u = torch.randn((B, L, H), generator=g, device=device, dtype=torch.float32).to(io)
    gy = torch.randn((B, L, H), generator=g, device=device, dtype=torch.float32).to(io)
    prob = {"layer": layer, "u": u, "gy": gy, "B": B}
    if w.get("layer"):
        return _layer_problem(w, prob, layer, B, L, device)
    if kind == "rglru":
        with torch.no_grad():
            u2 = u.reshape(B * L, H)
            prob["qr"] = (u2 @ layer.W_r.T.to(io)).reshape(B, L, H)
            prob["qi"] = (u2 @ layer.W_i.T.to(io)).reshape(B, L, H)
        args = (layer.lambda_param, layer.b_r, layer.b_i)

        def fwd():
            return ops.rglru_scan_fwd(prob["u"], prob["qr"], prob["qi"], *args)

        def bwd(ctx):
            return ops.rglru_scan_bwd(prob["u"], prob["qr"], prob["qi"], *args, ctx[1], prob["gy"], y=ctx[0])

        bpe = torch.tensor([], dtype=io).element_size()
        # algorithmic bytes: fwd reads u, qr, qi, writes y; bwd reads
        # u, qr, qi, gy and writes gu, gqr, gqi (the states are not counted)
        prob["bytes"] = {"fwd": 4 * B * L * H * bpe, "bwd": 7 * B * L * H * bpe}
        prob["probe"] = dict(name="lrx_rglru_bwd (+3 column sums)", bound="hbm", amount=prob["bytes"]["bwd"],
                             fn=bwd)
        if bpe == 4:  # the kernel streams 7 arrays + the 1/8-size anchor states: its measured mix ceiling
            prob["probe"]["stream"] = dict(dram_bytes=(7 + 1 / 8) * B * L * H * bpe, ceiling_gbs=6097.0,
                                           source="tools/ubench/streams.cu: 4 reads + 3 writes (bwd7), float4, "
                                                  "C4-sized arrays, same pool of B200s")
    elif kind == "s6":
        with torch.no_grad():
            from paper_2602_08810_b200.layers import _mm
            u2 = u.reshape(B * L, H)
            prob["pre"] = (_mm(u2, layer.W_delta) @ layer.W_delta_proj).reshape(B, L, H)
            prob["Bk"] = _mm(u2, layer.W_B.T).reshape(B, L, N)
            prob["Ck"] = _mm(u2, layer.W_C.T).reshape(B, L, N)
        pa = (layer.b_delta, layer.a_log)
        if w.get("seqpar"):
            from paper_2602_08810_b200.distributed import LongS6
            ls = LongS6(group=group)
            args = (prob["u"], prob["pre"], *pa, prob["Bk"], prob["Ck"], layer.D)

            def fwd():
                return ls.forward(*args)

            def bwd(ctx):
                return ls.backward(ctx[1], *args, prob["gy"])
        else:
            def fwd():
                return ops.s6_scan_fwd(prob["u"], prob["pre"], *pa, prob["Bk"], prob["Ck"], layer.D)

            def bwd(ctx):
                return ops.s6_scan_bwd(prob["u"], prob["pre"], *pa, prob["Bk"], prob["Ck"], layer.D, ctx[1],
                                       prob["gy"])

        bu, bp = u.element_size(), prob["pre"].element_size()
        per = B * L * H
        prob["bytes"] = {"fwd": per * (2 * bu + bp) + 2 * B * L * N * bp,
                         "bwd": per * (3 * bu + 2 * bp) + 4 * B * L * N * bp}
        # dominant kernel: the backward scan alone (C-ABI call, outputs preallocated)
        geo = ops.s6_geometry(u.dtype, B, L, H, N)
        f = dict(dtype=torch.float32, device=device)
        pb = {"gu": torch.empty_like(u), "gpre": torch.empty((B, L, H), **f),
              "gB": torch.empty((geo["n_dblk"], B * L * N), **f), "gC": torch.empty((geo["n_dblk"], B * L * N), **f),
              "ga": torch.empty((geo["part_rows"], H * N), **f), "gD": torch.empty((geo["part_rows"], H), **f),
              "gb": torch.empty((geo["part_rows"], H), **f), "ws": _lib_ws(geo["ws_bytes"], device)}

        def probe(ctx):
            from paper_2602_08810_b200 import _lib as L_
            ck = ctx[1]["ckpt"] if isinstance(ctx[1], dict) else ctx[1]
            L_.check(L_.lib().lrx_s6_bwd(
                L_.code_of(u.dtype), L_.ptr(prob["u"]), L_.ptr(prob["pre"]), L_.ptr(pa[0]), L_.ptr(pa[1]),
                L_.ptr(prob["Bk"]), L_.ptr(prob["Ck"]), L_.ptr(layer.D), L_.ptr(ck), L_.ptr(prob["gy"]), None,
                L_.ptr(pb["gu"]), L_.ptr(pb["gpre"]), L_.ptr(pb["gB"]), L_.ptr(pb["gC"]), L_.ptr(pb["ga"]),
                L_.ptr(pb["gD"]), L_.ptr(pb["gb"]), None, B, L, H, N, L_.ptr(pb["ws"]), pb["ws"].numel(), 0,
                L_.stream()))

        # MUFU-bound in fact (2 ex2 per (t, d, n) + softplus per (t, d)): reported beside the HBM roofline
        prob["probe"] = dict(name="lrx_s6_bwd" + (" (segment aggregates + main)" if geo["n_seg"] > 1 else ""),
                             bound="hbm", amount=prob["bytes"]["bwd"], fn=probe,
                             # main pass: 2 ex2 per (t,d,n) + softplus/sigmoid per (t,d); aggregate
                             # pass (segments > 1): 1 ex2 per (t,d,n) + softplus on (S-1)/S of the steps
                             mufu_ops=B * L * H * ((2 * N + 3) + (N + 2) * (geo["n_seg"] - 1) / geo["n_seg"]))
    else:  # s5 / lru: projections are part of the recurrence
        def fwd():
            return layer._forward(prob["u"], None, True)

        def bwd(ctx):
            saved = dict(ctx[1])
            saved["host"] = False
            return layer._backward(saved, prob["gy"])

        c = 8  # complex64 bytes
        per = B * L * H * 4
        st = B * L * N * c
        prob["bytes"] = {"fwd": 2 * per, "bwd": 3 * per}  # fused minimum: u,y / u,gy,gu
        prob["bytes_scan"] = {"fwd": 2 * st, "bwd": 4 * st}
        T_, P2 = B * L, 2 * layer._P  # real width of the interleaved complex state (s5: d_state = 2N, P = N)
        if layer._tc(H, T_) and layer._tc(P2, T_):
            # dominant kernel: the skip-fused output projection y = OUT Re(C x) + D u on tcgen05 (3xTF32);
            # achieved = issued TF32 tensor FLOP/s (3 MMAs per fp32 product)
            xs = torch.randn((T_, P2), device=device)
            wct = layer._wc().T.contiguous()
            wcl = ops.tf32_lo(wct)
            u2 = prob["u"].reshape(T_, H)
            yo = torch.empty((T_, H), device=device)
            prob["probe"] = dict(name="lrx_gemm_f32 (tcgen05 3xTF32, y = OUT Re(Cx) + D u)", bound="tensor",
                                 amount=3 * 2 * T_ * P2 * H,
                                 fn=lambda ctx: ops.gemm_f32(xs, wct, wcl, Cin=u2, colscale=layer.D,
                                                             alpha=layer.OUT_SCALE, out=yo))
        else:
            prob["probe"] = dict(name=f"lrx_{kind}_bwd (projections + scan)", bound="hbm", amount=3 * per,
                                 fn=lambda ctx: bwd(ctx))
    prob["fwd"], prob["bwd"] = fwd, bwd
    return prob


def _layer_problem(w, prob, layer, B, L, device):
    """Layer-level step: forward(tape) + layer_backward of the drop-in layer,
    projections included (layers.py:1020-1118 / 1208-1291).  Roofline probe:
    the dominant kernel -- the S6 backward scan, or the RG-LRU gate projection
    GEMM (tcgen05 3xTF32, issued TF32 FLOP)."""
    import torch

    from paper_2602_08810_b200 import ops
    kind, H, N = w["kind"], w["H"], w["N"]
    T_ = B * L

    def fwd():
        return layer._forward(prob["u"], None, True)

    def bwd(ctx):
        saved = dict(ctx[1])
        saved["host"] = False
        return layer._backward(saved, prob["gy"])

    bpe = prob["u"].element_size()
    if kind == "rglru":
        # scan streams + the four gate GEMMs' operand / output passes
        prob["bytes"] = {"fwd": 4 * T_ * H * bpe + 2 * 2 * T_ * H * 4, "bwd": 7 * T_ * H * bpe + 6 * T_ * H * 4}
        u2 = prob["u"].reshape(T_, H)
        wr = layer.W_r.contiguous()
        wl = ops.tf32_lo(wr)
        out = torch.empty((T_, H), device=device)
        prob["probe"] = dict(name="lrx_gemm_f32 (tcgen05 3xTF32 gate projection u W_r^T)", bound="tensor",
                             amount=3 * 2 * T_ * H * H, fn=lambda ctx: ops.gemm_f32(u2, wr, wl, out=out))
    else:
        saved = fwd()[1]
        pa = (layer.b_delta, layer.a_log)
        pre, Bk, Ck = saved["pre"], saved["Bk"], saved["Ck"]
        prob["bytes"] = {"fwd": T_ * H * (2 * bpe + 4) + 2 * T_ * N * 4, "bwd": T_ * H * (3 * bpe + 2 * 4) + 4 * T_ * N * 4}
        geo = ops.s6_geometry(prob["u"].dtype, B, L, H, N)
        prob["probe"] = dict(name="lrx_s6_bwd (inside the layer step)", bound="hbm", amount=prob["bytes"]["bwd"],
                             fn=lambda ctx: ops.s6_scan_bwd(prob["u"], pre, *pa, Bk, Ck, layer.D, ctx[1]["ckpt"],
                                                            prob["gy"]),
                             mufu_ops=B * L * H * ((2 * N + 3) + (N + 2) * (geo["n_seg"] - 1) / geo["n_seg"]))
    prob["fwd"], prob["bwd"] = fwd, bwd
    return prob


def run_gpu(args, w, rank, world, device):
    import torch
    import torch.distributed as dist

    from paper_2602_08810_b200 import _lib

    B_total = w["B"]
    L_rank = None
    if w.get("seqpar"):  # the time axis is split across ranks (C5)
        if w["L"] % world:
            raise SystemExit(f"L={w['L']} does not split into {world} slices")
        B, L_rank = B_total, w["L"] // world
    else:
        if B_total % world:
            raise SystemExit(f"batch {B_total} does not split over {world} GPUs")
        B = B_total // world
    prob = build_problem(w, B, device, L=L_rank, group=dist.group.WORLD if world > 1 else None)
    fwd, bwd = prob["fwd"], prob["bwd"]
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    ctx = None
    for _ in range(args.warmup):  # same liveness pattern as the timed loop (allocator steady state)
        ctx = fwd()
        bwd(ctx)
    torch.cuda.synchronize()

    # CUDA graphs: the step's kernels are captured once (after the warm-up) and
    # replayed, so the timed steps are not bounded by host launch overhead
    # (LRU C1 is ~70 launches of a few us each).  Every kernel of fwd + bwd
    # still runs every step on the same inputs; collectives (sequence-parallel
    # carries over NCCL) stay eager.
    graphed = False
    launches_per_step = None
    if args.graphs and not (world > 1 and w.get("seqpar")):
        try:
            n_c = _lib.launch_count()
            g_f, g_b = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_f):
                gctx = fwd()
            with torch.cuda.graph(g_b):
                gout = bwd(gctx)
            launches_per_step = _lib.launch_count() - n_c
            for _ in range(2):
                g_f.replay()
                g_b.replay()
            torch.cuda.synchronize()
            fwd, bwd = (lambda: g_f.replay()), (lambda c: g_b.replay())
            graphed = True
        except Exception as exc:  # capture unsupported for this path: stay eager
            print(f"[bench] CUDA graph capture failed ({type(exc).__name__}: {exc}); eager steps", file=sys.stderr)
            torch.cuda.synchronize()

    # Working sets below ~2x the 126 MB L2 (C1: ~30 MB) would be timed
    # L2-resident: flush the L2 before every step (a 256 MB write, outside
    # the per-step events) and time the steps by their own events.
    flush = prob["u"].numel() * prob["u"].element_size() * 8 < 2 * L2_BYTES
    flush_buf = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=device) if flush else None
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    n0 = _lib.launch_count()
    with Clocks(device.index) as clocks:
        barrier()
        torch.cuda.synchronize()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for k in range(args.steps):
            if flush:
                flush_buf.zero_()
            ev[k][0].record(stream)
            ctx = fwd()
            ev[k][1].record(stream)
            bwd(ctx)
            ev[k][2].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = _lib.launch_count() - n0
    if graphed:  # replays do not pass through the host launch counter
        launches = launches_per_step * args.steps
    if os.environ.get("LRX_BENCH_VERBOSE"):
        for k, e in enumerate(ev):
            print(f"step {k}: fwd {e[0].elapsed_time(e[1]):.3f} ms, bwd {e[1].elapsed_time(e[2]):.3f} ms",
                  file=sys.stderr)
        print("allocator:", {k: v for k, v in torch.cuda.memory_stats().items()
                             if k in ("num_device_alloc", "num_device_free", "num_alloc_retries")}, file=sys.stderr)
    ms_fwd = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    ms_bwd = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    ms = ms_fwd + ms_bwd if flush else t_start.elapsed_time(t_end) / args.steps
    t = torch.tensor([ms, ms_fwd, ms_bwd], device=device, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, ms_fwd, ms_bwd = (float(v) for v in t.tolist())

    # dominant kernel alone, CUDA events on the launching stream, after the timed region
    pr = prob["probe"]
    ctx = prob["fwd"]()  # eager (the probe launches the kernel itself)
    for _ in range(2):
        pr["fn"](ctx)
    torch.cuda.synchronize()
    ka, kb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ka.record(stream)
    nrep = max(3, args.steps)
    for _ in range(nrep):
        pr["fn"](ctx)
    kb.record(stream)
    torch.cuda.synchronize()
    probe_ms = ka.elapsed_time(kb) / nrep
    del ctx
    pt = torch.tensor([probe_ms], device=device, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(pt, op=dist.ReduceOp.MAX)
    probe_ms = float(pt.item())

    # e2e through the public API with pinned host buffers (a batch slice)
    e2e = run_e2e(args, w, prob, device)
    if world > 1:
        te = torch.tensor([e2e["ms"]], device=device, dtype=torch.float64)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e["ms"] = float(te.item())
    l2 = ("working set < 2x L2: L2 flushed (256 MB write) before every step, steps timed by their own events"
          if flush else "inputs > L2 (126 MB): no flush needed")
    return {"ms": ms, "ms_fwd": ms_fwd, "ms_bwd": ms_bwd, "launches": launches, "graphed": graphed, "l2": l2,
            "clocks": clocks.summary(),
            "bytes": prob["bytes"], "B_rank": B, "e2e": e2e, "probe": {k: v for k, v in pr.items() if k != "fn"},
            "probe_ms": probe_ms}


def run_e2e(args, w, prob, device):
    """Same step through the public API with HOST (pinned) buffers: H2D of the
    step's inputs, the operator fwd+bwd, D2H of every output, all timed.  The
    batch slice is processed in sub-batches on their own CUDA streams so the PCIe
    copies of one sub-batch overlap the kernels of the next (the host buffers
    are allocated and pinned once, outside the timed region)."""
    import torch

    from paper_2602_08810_b200 import layer_backward, ops

    kind, H, N = w["kind"], w["H"], w["N"]
    L = prob["u"].shape[1]
    names = ({"rglru": ("u", "qr", "qi", "gy"), "s6": ("u", "pre", "Bk", "Ck", "gy")}.get(kind, ("u", "gy"))
             if not w.get("layer") else ("u", "gy"))
    # the whole per-rank batch by default: inputs + outputs pinned (~2x the
    # input bytes), within ~45% of the host memory shared by the local ranks
    row = sum(prob[n][:1].numel() * prob[n].element_size() for n in names)
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:  # pragma: no cover - psutil is in the image
        avail = 64 << 30
    local = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    budget = 0.45 * avail / local
    Bs = prob["B"] if args.e2e_batch <= 0 else min(prob["B"], args.e2e_batch)
    while Bs > 1 and 2 * row * Bs > budget:
        Bs //= 2
    if w.get("seqpar") and 2 * row * Bs > budget:  # a time slice of this rank's sequence (host memory)
        frac = 1
        while frac < 64 and 2 * row * Bs / frac > budget:
            frac *= 2
        L = L // frac
        for n in ("u", "pre", "Bk", "Ck", "gy"):
            prob = dict(prob)
            prob[n] = prob[n][:, :L].contiguous()
    host = {n: prob[n][:Bs].cpu().pin_memory() for n in names}
    layer = prob["layer"]
    h2d = sum(t.numel() * t.element_size() for t in host.values())
    # sub-batches pipeline the PCIe copies: H2D of sub-batch i+1 and D2H of i
    # run on the two copy engines while i computes; the step approaches
    # max(H2D, D2H) + one sub-batch's share
    # one-row sub-batches: the finest overlap of the two copy engines with the
    # kernels (measured C4 full batch: 1-row 85 GB/s of PCIe traffic, 2-row 67, 8-row 48; tools/e2e_sweep.sh)
    n_sub = 1
    if kind in ("rglru", "s6") and not w.get("seqpar"):
        n_sub = next((k for k in (8, 4, 2) if Bs % k == 0), 1)
        while Bs // n_sub > int(os.environ.get("LRX_E2E_ROWS", "1")) and n_sub < Bs:
            n_sub *= 2
    sb = Bs // n_sub
    # sub-batches round-robin over a few streams: consecutive sub-batches still overlap, and each
    # stream's caching-allocator pool is reused by its next sub-batch instead of growing per stream
    # (tools/e2e_streams.sh: 4 streams vs one per sub-batch: rglru_layer 1.6 -> 5.4 Gelem/s, s6_layer 163 -> 174)
    n_streams = min(n_sub, int(os.environ.get("LRX_E2E_STREAMS", "4")))
    streams = [torch.cuda.Stream(device) for _ in range(n_streams)]

    def compute(d):
        if w.get("layer"):
            y, tape = layer.forward(d["u"], tape=True)
            g = layer_backward(layer, tape, d["gy"])
            return [y, g.u] + list(g.params.values())
        if kind == "rglru":
            y, ck = ops.rglru_scan_fwd(d["u"], d["qr"], d["qi"], layer.lambda_param, layer.b_r, layer.b_i)
            r = ops.rglru_scan_bwd(d["u"], d["qr"], d["qi"], layer.lambda_param, layer.b_r, layer.b_i, ck, d["gy"],
                                   y=y)
            return [y, r["gu_local"], r["gqr"], r["gqi"], r["gla"], r["gb_r"], r["gb_i"]]
        if kind == "s6" and w.get("seqpar"):
            from paper_2602_08810_b200.distributed import LongS6
            ls = LongS6()
            a = (d["u"], d["pre"], layer.b_delta, layer.a_log, d["Bk"], d["Ck"], layer.D)
            y, ctx = ls.forward(*a)
            return [y] + list(ls.backward(ctx, *a, d["gy"]).values())
        if kind == "s6":
            y, ck = ops.s6_scan_fwd(d["u"], d["pre"], layer.b_delta, layer.a_log, d["Bk"], d["Ck"], layer.D)
            r = ops.s6_scan_bwd(d["u"], d["pre"], layer.b_delta, layer.a_log, d["Bk"], d["Ck"], layer.D, ck,
                                d["gy"])
            return [y] + list(r.values())
        y, tape = layer.forward(d["u"], tape=True)
        g = layer_backward(layer, tape, d["gy"])
        return [y, g.u] + list(g.params.values())

    outs_host = [None] * n_sub

    def step():
        d2h = 0
        for i in range(n_sub):
            with torch.cuda.stream(streams[i % n_streams]):
                d = {n: t[i * sb:(i + 1) * sb].to(device, non_blocking=True) for n, t in host.items()}
                outs = compute(d)
                if outs_host[i] is None:
                    outs_host[i] = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in outs]
                for hbuf, o in zip(outs_host[i], outs):
                    hbuf.copy_(o, non_blocking=True)
                d2h += sum(o.numel() * o.element_size() for o in outs)
        return d2h

    step()  # allocates and pins the host outputs once
    torch.cuda.synchronize()
    reps = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(reps):
        d2h = step()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / reps
    return {"ms": ms, "batch": Bs, "L": L, "h2d": h2d, "d2h": d2h, "elems": Bs * L * H * N, "sub_batches": n_sub, "streams": n_streams}


# ---------------------------------------------------------------------------
# CPU reference arm (oracle restatement of the reference algorithm)

# Sample shapes of the CPU arms: identical B / H / N,
# C1 and C2 at full length, C3 / C4 at L/64, C5 at L/1024 (its L/64 sample
# alone would take ~30 s per step).  Time scales linearly in L for a scan.
CPU_TIMED_L = {"lru": 1024, "s5": 4096, "s6": 8192 // 64, "rglru": 16384 // 64, "s6_long": 2 ** 20 // 1024,
               "s6_layer": 8192 // 64, "rglru_layer": 16384 // 64}


def cpu_problem(w, workload, cores, seed=0):
    """One fwd+bwd of the reference algorithm (the oracle restatement: numpy +
    the C restatement of the numba loops, time-chunk parallel over `cores`
    workers as the reference's mode="parallel") on the sample shape.
    Returns (run, elems, desc)."""
    from oracle import port

    kind, B, H, N = w["kind"], w["B"], w["H"], w["N"]
    L = CPU_TIMED_L[workload]
    dt = np.float32
    p = port.init_params(kind, H, None if kind == "rglru" else (N if kind != "s5" else 2 * N), dtype="f32",
                         seed=seed)
    rng = port.Rng(seed + 1)
    u = rng.normal((B, L, H)).astype(dt)
    gy = rng.normal((B, L, H)).astype(dt)
    if w.get("layer"):
        lay = port.Layer(kind, p)

        def run():
            y, sv = lay.forward(u, "parallel", cores)
            lay.backward(sv, gy)
    elif kind == "rglru":
        qr, qi = u @ p["W_r"].T, u @ p["W_i"].T

        def run():
            port.rglru_scan(u, qr, qi, p["lambda_param"], p["b_r"], p["b_i"], gy, "parallel", cores)
    elif kind == "s6":
        pre = (u @ p["W_delta"]) @ p["W_delta_proj"]
        Bk, Ck = u @ p["W_B"].T, u @ p["W_C"].T

        def run():
            port.s6_scan(u, pre, p["b_delta"], p["a_log"], Bk, Ck, p["D"], gy, "parallel", cores)
    else:
        lay = port.Layer(kind, p)

        def run():
            y, sv = lay.forward(u, "parallel", cores)
            lay.backward(sv, gy)
    where = "the layer boundary (projections included)" if w.get("layer") else "the same operator boundary"
    desc = (f"{kind} B={B} L={L} (of {w['L']}) H={H} N={N} f32, fwd+bwd at {where}, "
            f"reference algorithm (oracle port), mode='parallel' workers={cores}")
    return run, B * L * H * N, desc


def _blas_threads(n):
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=n)
    except Exception:  # pragma: no cover - threadpoolctl is in the image
        import contextlib
        return contextlib.nullcontext()


def cpu_sample(w, workload, budget_s=12.0, cores=None, seed=0):
    """Rate of the reference algorithm on the host's cores: (Gelem/s, desc, cores, ms per sample)."""
    cores = cores or os.cpu_count() or 1
    with _blas_threads(cores):
        run, elems, desc = cpu_problem(w, workload, cores, seed)
        run()  # warm (pools, page-in)
        n, t0 = 0, time.perf_counter()
        while True:
            run()
            n += 1
            if time.perf_counter() - t0 > budget_s or n >= 20:
                break
    dt_s = (time.perf_counter() - t0) / n
    return elems / dt_s / 1e9, f"{desc}, mean of {n} runs", cores, dt_s * 1e3


def reference_arm(args, w, config):
    """--impl reference: the reference's CPU algorithm on all host cores, one
    sample step per timed step (measured, not extrapolated), then one 1-core
    step for the single-thread row."""
    cores = os.cpu_count() or 1
    with _blas_threads(cores):
        run, elems, desc = cpu_problem(w, args.workload, cores)
        for _ in range(args.warmup):
            run()
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            run()
            times.append(time.perf_counter() - t0)
    ms = float(np.mean(times)) * 1e3
    v = elems / (ms * 1e-3) / 1e9
    with _blas_threads(1):
        run1, _, desc1 = cpu_problem(w, args.workload, 1)
        t0 = time.perf_counter()
        run1()
        ms1 = (time.perf_counter() - t0) * 1e3
    L_t = CPU_TIMED_L[args.workload]
    cfg = dict(config, timed_L=L_t,
               timing=(f"measured at L={L_t} with the config's B/H/N (value = rate of the timed sample; "
                       f"a full-L step takes ms_per_step x {w['L'] // L_t}, linear in L)"
                       if L_t != w["L"] else "measured at the full config"))
    return {"metric": METRIC, "value": v, "unit": "Gelem/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference", "config": cfg,
            "cpu_baseline": {"value": v, "unit": "Gelem/s", "cores": cores, "kind": "port",
                             "sample": f"{desc}, mean of {args.steps} steps",
                             "one_core": {"value": elems / (ms1 * 1e-3) / 1e9, "unit": "Gelem/s", "cores": 1,
                                          "ms": ms1, "sample": f"{desc1}, OpenBLAS 1 thread, one step"}},
            "e2e": {"value": v, "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="lrx", choices=["lrx", "reference"])
    ap.add_argument("--e2e-batch", type=int, default=0, help="e2e batch rows per rank (0 = the whole per-rank batch)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graphs", dest="graphs", action="store_false",
                    help="launch every kernel from the host instead of replaying the captured step")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    elems = _state_dims(w)
    config = {"workload": f"{args.workload}: configs[{w['cfg']}] {w['kind']} B={w['B']} L={w['L']} H={w['H']} "
                          f"N={w['N']}", "global_batch": w["B"], "seq_len": w["L"], "width": w["H"],
              "d_state": w["N"],
              "parallelism": (f"sequence-parallel x{world} (+ in-kernel time segments)" if w.get("seqpar")
                              else f"batch-sharded x{world}" if world > 1 else "single GPU"),
              "l2": "inputs > L2 (126 MB): no flush needed"}

    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(reference_arm(args, w, config)), flush=True)
        return

    import torch
    import torch.distributed as dist
    # LRX_BENCH_ONE_GPU=1 (test hook): every rank on cuda:0 over gloo, to
    # exercise the multi-rank plumbing on a single-GPU box (timings meaningless)
    one_gpu = os.environ.get("LRX_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    if world > 1:
        # NCCL's init log states the communicator's rank count and transport
        # (NVLink / NVLS) on stderr, so the scaling run can be checked
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local if world > 1 else torch.cuda.current_device())
    torch.cuda.set_device(device)
    r = run_gpu(args, w, rank, world, device)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    config["l2"] = r["l2"]
    value = elems / (r["ms"] * 1e-3) / 1e9
    pr, pms = r["probe"], r["probe_ms"]
    if pr["bound"] == "tensor":
        tpk, tsrc = _tensor_peak()
        achieved = pr["amount"] / (pms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tpk, "unit": "TFLOP/s", "frac": achieved / tpk,
                "traffic": _traffic(args.workload, "probe"), "kernel": pr["name"], "peak_source": tsrc,
                "per_launch_ms": pms, "algorithmic_flops_per_launch": pr["amount"]}
    else:
        peak, peak_kind = _peaks()
        achieved = pr["amount"] / (pms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": _traffic(args.workload, "probe"), "kernel": pr["name"], "peak_source": peak_kind,
                "per_launch_ms": pms, "algorithmic_bytes_per_launch": pr["amount"],
                "step_share": pms / r["ms"]}
        if "stream" in pr:  # achieved DRAM rate against the measured ceiling of the kernel's stream mix
            sc = pr["stream"]
            dr = sc["dram_bytes"] / (pms * 1e-3) / 1e9
            roof["stream_ceiling"] = {"dram_GBps": dr, "ceiling_GBps": sc["ceiling_gbs"],
                                      "frac": dr / sc["ceiling_gbs"], "source": sc["source"]}
        if "mufu_ops" in pr:  # the binding unit of the S6 scan: MUFU ex2 (16/clk/SM, ubench-measured 4.62 T/s)
            mu = pr["mufu_ops"] / (pms * 1e-3) / 1e12
            roof["compute"] = {"bound": "mufu", "achieved": mu, "peak": 4.62, "unit": "Tops/s", "frac": mu / 4.62,
                               "peak_source": "tools/ubench/mufu.cu on this pool's B200 (ex2.approx.f32)"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, desc, cores, _ = cpu_sample(w, args.workload)
        cpu = {"value": v, "unit": "Gelem/s", "cores": cores, "kind": "port", "sample": desc}
    e = r["e2e"]
    e2e = {"value": e["elems"] * world / (e["ms"] * 1e-3) / 1e9, "unit": "Gelem/s",
           "h2d_bytes_per_step": e["h2d"], "d2h_bytes_per_step": e["d2h"],
           "sample": f"B={e['batch']} of {r['B_rank']} per rank (L={e['L']}) through paper_2602_08810_b200.ops / "
                     f"layer API, pinned host buffers, {e['sub_batches']} sub-batches overlapped on {e['streams']} streams; host wall clock "
                     f"incl. H2D + kernels + D2H", "ms_per_step": e["ms"]}
    line = {"metric": METRIC, "value": value, "unit": "Gelem/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": {"f32": "f32", "bf16": "bf16 io / f32 accum"}[w["dtype"]],
            "data": "synthetic (reference init, N(0,1) activations, projections from the layer's weights)",
            "config": config, "cuda_graphs": r["graphed"], "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": r["launches"],
            "clocks": r["clocks"],
            "kernels": {"fwd_ms": r["ms_fwd"], "bwd_ms": r["ms_bwd"],
                        "fwd_GBps": r["bytes"]["fwd"] / (r["ms_fwd"] * 1e-3) / 1e9,
                        "bwd_GBps": r["bytes"]["bwd"] / (r["ms_bwd"] * 1e-3) / 1e9}}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
