"""Scan-level operators: thin torch wrappers over the fused C-ABI kernels.

These are the operator boundary between a layer's dense projections (GEMMs)
and its recurrence — the unit the benchmark measures ("scan Gelem/s") and the
unit a framework integration binds.  All tensors live on the
current CUDA device; outputs are allocated here, workspaces are transient.

  rglru_scan_fwd / rglru_scan_bwd   layers.py:1208-1291 (gates + scan + pullback)
  s6_scan_fwd / s6_scan_bwd         layers.py:1038-1118 (delta softplus, ZOH/Euler
                                    discretisation, scan, C readout, D skip)
  mimo_scan_fwd / mimo_scan_bwd     layers.py:666-704 (v = scale * Bu, scan,
                                    d abar / d scale reductions)
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import _lib

__all__ = ["rglru_scan_fwd", "rglru_scan_bwd", "s6_geometry", "s6_scan_fwd", "s6_scan_bwd", "s6_fwd_carry",
           "s6_bwd_carry", "mimo_scan_fwd", "mimo_scan_bwd", "reduce_rows", "gemm_f32", "gemm_f32_tn", "tf32_lo",
           "gemm_bf16", "ACT_NONE", "ACT_SOFTPLUS", "ACT_SIGMOID",
           "s4d_scan_fwd", "s4d_scan_bwd", "S4D_FUSED_N"]


def reduce_rows(part, rows, cols, other=None):
    """Fixed-order device reduction out[j] = sum_r part[r, j] (* other[r, j]:
    a column-wise dot product when `other` is given)."""
    out = torch.empty(cols, dtype=part.dtype, device=part.device)
    lib, code = _lib.lib(), _lib.code_of(part.dtype)
    if other is None and rows <= 4096:  # short columns: one launch, no workspace
        _lib.check(lib.lrx_reduce_rows(code, _lib.ptr(part), _lib.ptr(out), rows, cols, _lib.stream()))
        return out
    ws = _lib.workspace(lib.lrx_reduce_rows_ws_bytes(code, rows, cols), part.device)
    _lib.check(lib.lrx_reduce_rows_ws(code, _lib.ptr(part), _lib.ptr(other), _lib.ptr(out), rows, cols,
                                      _lib.ptr(ws), ws.numel(), _lib.stream()))
    return out


# ---------------------------------------------------------------------------
# RG-LRU

def rglru_scan_fwd(u, qr, qi, lambda_param, b_r, b_i):
    """y = x of the gated recurrence; u/qr/qi [B, L, W] (f32/f64/bf16).
    Returns (y, ckpt): ckpt [n_chunks + 1, B*W] holds the state entering every
    time chunk and, in its last row, the final state."""
    B, L, W = u.shape
    lib = _lib.lib()
    code = _lib.code_of(u.dtype)
    ck, nc = _lib.i64(), _lib.i64()
    _lib.check(lib.lrx_rglru_chunking(code, L, _lib.ref(ck), _lib.ref(nc)))
    y = torch.empty_like(u)
    ckpt = torch.empty((nc.value + 1, B * W), dtype=lambda_param.dtype, device=u.device)
    ws = _lib.workspace(lib.lrx_rglru_workspace_bytes(code, B, L, W), u.device)
    _lib.check(lib.lrx_rglru_fwd(code, _lib.ptr(u), _lib.ptr(qr), _lib.ptr(qi), _lib.ptr(lambda_param),
                                 _lib.ptr(b_r), _lib.ptr(b_i), _lib.ptr(y), _lib.ptr(ckpt), B, L, W, _lib.ptr(ws),
                                 ws.numel(), _lib.stream()))
    return y, ckpt


def rglru_scan_bwd(u, qr, qi, lambda_param, b_r, b_i, ckpt, gy, y=None):
    """Pullback of rglru_scan_fwd.  The default kernel reconstructs the states
    from ckpt while it walks backwards; y (the forward output = the state) is
    used only by the y-streaming variant (LRX_RGLRU_MODE=tma).  Returns dict
    with gu_local (the s*i*g term; the gate-GEMM terms are the caller's), gqr,
    gqi ([B, L, W]) and the batch/time sums gla (sum 8 r gloga), gb_r, gb_i."""
    B, L, W = u.shape
    lib = _lib.lib()
    code = _lib.code_of(u.dtype)
    gu, gqr, gqi = torch.empty_like(u), torch.empty_like(u), torch.empty_like(u)
    f = dict(dtype=lambda_param.dtype, device=u.device)
    gla, gbr, gbi = (torch.empty(W, **f) for _ in range(3))
    ws = _lib.workspace(lib.lrx_rglru_workspace_bytes(code, B, L, W), u.device)
    _lib.check(lib.lrx_rglru_bwd(code, _lib.ptr(u), _lib.ptr(qr), _lib.ptr(qi), _lib.ptr(lambda_param),
                                 _lib.ptr(b_r), _lib.ptr(b_i), _lib.ptr(ckpt), _lib.ptr(y), _lib.ptr(gy),
                                 _lib.ptr(gu), _lib.ptr(gqr), _lib.ptr(gqi), _lib.ptr(gla), _lib.ptr(gbr),
                                 _lib.ptr(gbi), B, L, W, _lib.ptr(ws), ws.numel(), _lib.stream()))
    return {"gu_local": gu, "gqr": gqr, "gqi": gqi, "gla": gla, "gb_r": gbr, "gb_i": gbi}


# ---------------------------------------------------------------------------
# S6

S6_REUSE_AGG = 1
S6_DELTA_IN = 2
SCHEME_CODE = {"zoh": 0, "bilinear": 1, "dirac": 2}


def s6_geometry(io_dtype, B, L, D, N):
    """dict(ckpt_len, n_ckpt, n_dblk, n_seg, part_rows, ws_bytes) for these extents."""
    g = (ctypes.c_int64 * 6)()
    _lib.check(_lib.lib().lrx_s6_geometry(_lib.code_of(io_dtype), B, L, D, N, g))
    return dict(zip(("ckpt_len", "n_ckpt", "n_dblk", "n_seg", "part_rows", "ws_bytes"), (int(v) for v in g)))


def _s6_ws(geo, device, ws):
    if ws is not None:
        return ws
    return _lib.workspace(geo["ws_bytes"], device)


class GroupedCkpt:
    """Checkpoints of a d_state > 16 scan run as 16-state groups (one v3
    checkpoint tensor per group); [:, -1] is the final state [B, D, N]."""

    def __init__(self, parts):
        self.parts = parts

    def __getitem__(self, idx):
        if idx != (slice(None), -1):
            raise IndexError("GroupedCkpt supports [:, -1] (the final state) only")
        return torch.cat([c[:, -1] for c in self.parts], dim=-1)


def _grouped(u, D, N, x0=None, ws=None, flags=0):
    """d_state a multiple of 16 above 16: the v3 kernels run per 16-state group
    (the recurrence is diagonal; the readout and the gradients of u / pre are
    sums over the groups, accumulated in fp32)."""
    if N <= 16 or N % 16 or ws is not None or flags & S6_REUSE_AGG or u.dtype not in (torch.float32, torch.bfloat16):
        return False
    geo = s6_geometry(torch.float32, u.shape[0], u.shape[1], D, 16)
    return geo["n_dblk"] > 0 and D % 4 == 0 and os.environ.get("LRX_S6_NOGROUP") != "1"


def _group_args(a_log, Bk, Ck, Dskip, g):
    sl = slice(16 * g, 16 * g + 16)
    return (a_log[:, sl].contiguous(), Bk[..., sl].contiguous(), Ck[..., sl].contiguous(),
            Dskip if g == 0 else torch.zeros_like(Dskip))


def s6_scan_fwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, x0=None, ws=None, flags=0, ckpt=True):
    """Selective scan; u [B, L, D] (f32/f64/bf16), pre [B, L, D] and Bk/Ck
    [B, L, N] in compute precision.  x0 [B, D, N] optionally seeds the state.
    Returns (y, ckpt); ckpt[:, -1] is the final state [B, D, N] (None with
    ckpt=False: inference, no checkpoint writes).  `ws`/`flags`: workspace
    holding per-segment maps from s6_fwd_carry (flags=S6_REUSE_AGG).
    d_state = 32, 48, 64, ...: 16-state groups on the v3 kernels."""
    B, L, D = u.shape
    N = Bk.shape[-1]
    if _grouped(u, D, N, x0, ws, flags):
        u32 = u.float()
        y, parts = None, []
        for g in range(N // 16):
            ag, Bg, Cg, Dg = _group_args(a_log, Bk, Ck, Dskip, g)
            x0g = x0[..., 16 * g:16 * g + 16].contiguous() if x0 is not None else None
            yg, ckg = s6_scan_fwd(u32, pre, b_delta, ag, Bg, Cg, Dg, x0=x0g, ckpt=ckpt, flags=flags)
            y = yg if y is None else y.add_(yg)
            parts.append(ckg)
        return y.to(u.dtype), (GroupedCkpt(parts) if ckpt else None)
    return _s6_scan_fwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, x0, ws, flags, ckpt)


def _s6_scan_fwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, x0=None, ws=None, flags=0, ckpt=True):
    """Selective scan; u [B, L, D] (f32/f64/bf16), pre [B, L, D] and Bk/Ck
    [B, L, N] in compute precision.  x0 [B, D, N] optionally seeds the state.
    Returns (y, ckpt); ckpt[:, -1] is the final state [B, D, N] (None with
    ckpt=False: inference, no checkpoint writes).  `ws`/`flags`: workspace
    holding per-segment maps from s6_fwd_carry (flags=S6_REUSE_AGG)."""
    B, L, D = u.shape
    N = Bk.shape[-1]
    geo = s6_geometry(u.dtype, B, L, D, N)
    y = torch.empty_like(u)
    ck = torch.empty((B, geo["n_ckpt"], D, N), dtype=a_log.dtype, device=u.device) if ckpt else None
    ws = _s6_ws(geo, u.device, ws)
    _lib.check(_lib.lib().lrx_s6_fwd(_lib.code_of(u.dtype), _lib.ptr(u), _lib.ptr(pre), _lib.ptr(b_delta),
                                     _lib.ptr(a_log), _lib.ptr(Bk), _lib.ptr(Ck), _lib.ptr(Dskip), _lib.ptr(x0),
                                     _lib.ptr(y), _lib.ptr(ck), B, L, D, N, _lib.ptr(ws), ws.numel(), flags,
                                     _lib.stream()))
    return y, ck


def s6_scan_bwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, ckpt, gy, h_in=None, want_h_out=False, ws=None, flags=0):
    if isinstance(ckpt, GroupedCkpt):
        if ws is not None or flags & S6_REUSE_AGG:
            raise ValueError("reused segment maps (ws / flags) need d_state == 16; LongS6 groups itself")
        u32, gy32 = u.float(), gy.float()
        out, cat = None, ("gBk", "gCk", "ga_log") + (("h_out",) if want_h_out else ())
        for g, ckg in enumerate(ckpt.parts):
            ag, Bg, Cg, Dg = _group_args(a_log, Bk, Ck, Dskip, g)
            hg = h_in[..., 16 * g:16 * g + 16].contiguous() if h_in is not None else None
            r = _s6_scan_bwd(u32, pre, b_delta, ag, Bg, Cg, Dg, ckg, gy32, h_in=hg, want_h_out=want_h_out,
                             flags=flags)
            if out is None:
                out = {k: ([v] if k in cat else v) for k, v in r.items()}
            else:  # fixed group order; the carries split by group (diagonal recurrence)
                out["gu_local"].add_(r["gu_local"])
                out["gpre"].add_(r["gpre"])
                out["gb_delta"].add_(r["gb_delta"])
                for k in cat:
                    out[k].append(r[k])
        out["gu_local"] = out["gu_local"].to(u.dtype)
        for k in cat:
            out[k] = torch.cat(out[k], dim=-1)
        return out
    return _s6_scan_bwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, ckpt, gy, h_in, want_h_out, ws, flags)


def _s6_scan_bwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, ckpt, gy, h_in=None, want_h_out=False, ws=None, flags=0):
    """Pullback of s6_scan_fwd.  Returns dict: gu_local (D gy + delta sum_n g B),
    gpre (d/d pre) [B, L, D]; gBk, gCk [B, L, N]; ga_log [D, N]; gD, gb_delta [D];
    with want_h_out also h_out [B, D, N] = d loss / d x0.  h_in [B, D, N] is
    the cotangent carry entering from the right (sequence-parallel mode)."""
    B, L, D = u.shape
    N = Bk.shape[-1]
    geo = s6_geometry(u.dtype, B, L, D, N)
    ndb, prow = geo["n_dblk"], geo["part_rows"]
    f = dict(dtype=a_log.dtype, device=u.device)
    gu, gpre = torch.empty_like(u), torch.empty(u.shape, **f)
    gBp, gCp = torch.empty((ndb, B * L * N), **f), torch.empty((ndb, B * L * N), **f)
    gap, gDp, gbp = torch.empty((prow, D * N), **f), torch.empty((prow, D), **f), torch.empty((prow, D), **f)
    h_out = torch.empty((B, D, N), **f) if want_h_out else None
    ws = _s6_ws(geo, u.device, ws)
    _lib.check(_lib.lib().lrx_s6_bwd(
        _lib.code_of(u.dtype), _lib.ptr(u), _lib.ptr(pre), _lib.ptr(b_delta), _lib.ptr(a_log), _lib.ptr(Bk),
        _lib.ptr(Ck), _lib.ptr(Dskip), _lib.ptr(ckpt), _lib.ptr(gy), _lib.ptr(h_in), _lib.ptr(gu), _lib.ptr(gpre),
        _lib.ptr(gBp), _lib.ptr(gCp), _lib.ptr(gap), _lib.ptr(gDp), _lib.ptr(gbp), _lib.ptr(h_out), B, L, D, N,
        _lib.ptr(ws), ws.numel(), flags, _lib.stream()))
    out = {"gu_local": gu, "gpre": gpre,
           "gBk": reduce_rows(gBp, ndb, B * L * N).reshape(B, L, N),
           "gCk": reduce_rows(gCp, ndb, B * L * N).reshape(B, L, N),
           "ga_log": reduce_rows(gap, prow, D * N).reshape(D, N),
           "gD": reduce_rows(gDp, prow, D), "gb_delta": reduce_rows(gbp, prow, D)}
    if want_h_out:
        out["h_out"] = h_out
    return out


def s6_fwd_carry(u, pre, b_delta, a_log, Bk, ws=None):
    """The slice's forward map for the sequence-parallel exchange:
    x_end = exp(a * sd) * x_in + x_agg.  Returns (x_agg [B, D, N], sd [B, D], ws);
    pass ws with flags=S6_REUSE_AGG to the following s6_scan_fwd."""
    B, L, D = u.shape
    N = Bk.shape[-1]
    geo = s6_geometry(u.dtype, B, L, D, N)
    f = dict(dtype=a_log.dtype, device=u.device)
    x_agg, sd = torch.empty((B, D, N), **f), torch.empty((B, D), **f)
    ws = _s6_ws(geo, u.device, ws)
    _lib.check(_lib.lib().lrx_s6_fwd_carry(_lib.code_of(u.dtype), _lib.ptr(u), _lib.ptr(pre), _lib.ptr(b_delta),
                                           _lib.ptr(a_log), _lib.ptr(Bk), _lib.ptr(x_agg), _lib.ptr(sd), B, L, D,
                                           N, _lib.ptr(ws), ws.numel(), _lib.stream()))
    return x_agg, sd, ws


def s6_bwd_carry(gy, pre, b_delta, a_log, Ck, ws=None):
    """The slice's cotangent map (right to left): h_left = exp(a * sd) * h_right + h_agg.
    Returns (h_agg [B, D, N], sd [B, D], ws) for s6_scan_bwd(flags=S6_REUSE_AGG)."""
    B, L, D = gy.shape
    N = Ck.shape[-1]
    geo = s6_geometry(gy.dtype, B, L, D, N)
    f = dict(dtype=a_log.dtype, device=gy.device)
    h_agg, sd = torch.empty((B, D, N), **f), torch.empty((B, D), **f)
    ws = _s6_ws(geo, gy.device, ws)
    _lib.check(_lib.lib().lrx_s6_bwd_carry(_lib.code_of(gy.dtype), _lib.ptr(gy), _lib.ptr(pre), _lib.ptr(b_delta),
                                           _lib.ptr(a_log), _lib.ptr(Ck), _lib.ptr(h_agg), _lib.ptr(sd), B, L, D,
                                           N, _lib.ptr(ws), ws.numel(), _lib.stream()))
    return h_agg, sd, ws


# ---------------------------------------------------------------------------
# fp32 GEMM on tcgen05 (3xTF32)

def tf32_lo(t):
    """t - tf32(t): the low part of the 3xTF32 split (TF32 = the top 19 bits)."""
    return t - (t.view(torch.int32) & -8192).view(torch.float32)


def gemm_f32(A, Bt, Bt_lo=None, Cin=None, colscale=None, alpha=1.0, beta=0.0, out=None, bias=None, act=0):
    """C = act(alpha A Bt^T + bias) + (colscale or beta) * Cin on the tensor
    cores (3xTF32, fp32-accurate).  A [M, K], Bt [N, K] fp32 contiguous
    (K % 4 == 0); act: ACT_NONE / ACT_SOFTPLUS / ACT_SIGMOID."""
    M, K = A.shape
    N = Bt.shape[0]
    if Bt.shape[1] != K or (Bt_lo is not None and Bt_lo.shape != Bt.shape):
        raise ValueError(f"gemm_f32: A {tuple(A.shape)} and Bt {tuple(Bt.shape)} disagree on K")
    for name, t in (("Cin", Cin), ("out", out)):
        if t is not None and tuple(t.shape) != (M, N):
            raise ValueError(f"gemm_f32: {name} {tuple(t.shape)} is not [M, N] = [{M}, {N}]")
    if Bt_lo is None:
        Bt_lo = tf32_lo(Bt)
    C = out if out is not None else torch.empty((M, N), dtype=torch.float32, device=A.device)
    _lib.check(_lib.lib().lrx_gemm_f32(_lib.ptr(A), _lib.ptr(Bt), _lib.ptr(Bt_lo), _lib.ptr(C), _lib.ptr(Cin),
                                       _lib.ptr(colscale), _lib.ptr(bias), act, M, N, K, alpha, beta, _lib.stream()))
    return C


def gemm_f32_tn(A, B, alpha=1.0):
    """C = alpha A^T B for A [K, M], B [K, N] fp32 row-major (K long): split-K
    tcgen05 3xTF32 partials, summed in a fixed order."""
    K, M = A.shape
    N = B.shape[1]
    if B.shape[0] != K:
        raise ValueError(f"gemm_f32_tn: A {tuple(A.shape)} and B {tuple(B.shape)} disagree on K")
    ks = _lib.i64()
    _lib.check(_lib.lib().lrx_gemm_f32_tn_splits(M, N, K, _lib.ref(ks)))
    part = torch.empty((ks.value, M * N), dtype=torch.float32, device=A.device)
    _lib.check(_lib.lib().lrx_gemm_f32_tn(_lib.ptr(A), _lib.ptr(B), _lib.ptr(part), M, N, K, alpha, _lib.stream()))
    return reduce_rows(part, ks.value, M * N).reshape(M, N)


def cast(t, dtype):
    """bf16 <-> fp32 copy of an activation plane on the lrx streaming kernel
    (any other pair: torch)."""
    pair = (t.dtype, dtype)
    if pair not in ((torch.bfloat16, torch.float32), (torch.float32, torch.bfloat16)) or not t.is_cuda:
        return t.to(dtype)
    t = t.contiguous()
    out = torch.empty(t.shape, dtype=dtype, device=t.device)
    _lib.check(_lib.lib().lrx_cast(_lib.code_of(t.dtype), _lib.code_of(dtype), _lib.ptr(t), _lib.ptr(out), t.numel(),
                                   _lib.stream()))
    return out


# ---------------------------------------------------------------------------
# bf16 GEMM on tcgen05 (kind::f16, fp32 accumulation) with a fused epilogue

ACT_NONE, ACT_SOFTPLUS, ACT_SIGMOID = 0, 1, 2


def gemm_bf16(A, Bt, bias=None, act=ACT_NONE, Cin=None, alpha=1.0, beta=0.0, out=None, out_dtype=torch.float32):
    """C = act(alpha A Bt^T + bias) + beta Cin on the tensor cores, fp32 (or
    bf16, without Cin) out.  A [M, K], Bt [N, K] bf16 contiguous (K % 8 == 0,
    N % 4 == 0)."""
    M, K = A.shape
    N = Bt.shape[0]
    if Bt.shape[1] != K:
        raise ValueError(f"gemm_bf16: A {tuple(A.shape)} and Bt {tuple(Bt.shape)} disagree on K")
    for name, t in (("Cin", Cin), ("out", out)):
        if t is not None and tuple(t.shape) != (M, N):
            raise ValueError(f"gemm_bf16: {name} {tuple(t.shape)} is not [M, N] = [{M}, {N}]")
    C = out if out is not None else torch.empty((M, N), dtype=out_dtype, device=A.device)
    _lib.check(_lib.lib().lrx_gemm_bf16(_lib.ptr(A), _lib.ptr(Bt), _lib.ptr(C), _lib.ptr(Cin), _lib.ptr(bias), M, N,
                                        K, alpha, beta, act, int(C.dtype == torch.bfloat16), _lib.stream()))
    return C


# ---------------------------------------------------------------------------
# MIMO (S5 / LRU)

def mimo_scan_fwd(abar, scale, bu):
    """x_k = abar x_{k-1} + scale bu_k over complex bu [B, L, P]."""
    B, L, P = bu.shape
    lib = _lib.lib()
    code = _lib.code_of(bu.dtype)
    x = torch.empty_like(bu)
    ws = _lib.workspace(lib.lrx_mimo_workspace_bytes(code, B, L, P), bu.device)
    _lib.check(lib.lrx_mimo_fwd(code, _lib.ptr(abar.contiguous()), _lib.ptr(scale.contiguous()), _lib.ptr(bu),
                                _lib.ptr(x), B, L, P, _lib.ptr(ws), ws.numel(), _lib.stream()))
    return x


def mimo_scan_bwd(abar, scale, bu, x, gx, reduce=True):
    """Returns (gbu [B,L,P], gabar [P], gscale [P]) (complex); bu None: no
    gscale (None; lrx_mimo_coef_grads derives it from the weight-gradient GEMM)."""
    B, L, P = x.shape
    lib = _lib.lib()
    code = _lib.code_of(x.dtype)
    ck, nc = _lib.i64(), _lib.i64()
    _lib.check(lib.lrx_mimo_chunking(code, B, L, P, _lib.ref(ck), _lib.ref(nc)))
    nc = nc.value
    gbu = torch.empty_like(x)
    gap = torch.empty(nc * B * P, dtype=x.dtype, device=x.device)
    gsp = torch.empty_like(gap)
    ws = _lib.workspace(lib.lrx_mimo_bwd_workspace_bytes(code, B, L, P), x.device)
    _lib.check(lib.lrx_mimo_bwd(code, _lib.ptr(abar.contiguous()), _lib.ptr(scale.contiguous()), _lib.ptr(bu),
                                _lib.ptr(x), _lib.ptr(gx), _lib.ptr(gbu), _lib.ptr(gap), _lib.ptr(gsp), B, L, P,
                                _lib.ptr(ws), ws.numel(), _lib.stream()))
    if not reduce:  # per-chunk partial rows [nc * B, P] (lrx_mimo_coef_grads sums them)
        return gbu, gap.view(nc * B, P), (gsp.view(nc * B, P) if bu is not None else None)
    return gbu, reduce_rows(gap, nc * B, P), (reduce_rows(gsp, nc * B, P) if bu is not None else None)


# ---------------------------------------------------------------------------
# Fused projection + scan (S5 / LRU, constant steps, fp32): csrc/lrx_mimo_fused.cu

MIMO_FUSED_MAX_L = 8192


def mimo_fused_supported(B, L, m, P, dtype):
    """The fused kernels' domain (lrx_mimo_fused_*: LRX_ERR_UNSUPPORTED outside)."""
    return dtype == torch.float32 and P <= 128 and m % 16 == 0 and L <= MIMO_FUSED_MAX_L and B * L < 2 ** 31


def mimo_fused_weights(wt, wt_lo):
    """[2P, m] interleaved (re, im) projection rows and their TF32 low plane ->
    the fused kernels' [256, m] layout [Re rows (128, zero padded) ; Im rows]."""
    P2, m = wt.shape
    P = P2 // 2
    A = torch.zeros((2, 256, m), dtype=wt.dtype, device=wt.device)
    for i, w in enumerate((wt, wt_lo)):
        A[i, :P] = w[0::2]
        A[i, 128:128 + P] = w[1::2]
    return A[0], A[1]


def _fused_ws(B, L, P, device):
    n = _lib.i64()
    _lib.check(_lib.lib().lrx_mimo_fused_workspace_bytes(B, L, P, _lib.ref(n)))
    return _lib.workspace(n.value, device)


def mimo_fused_fwd(A, A_lo, u2, abar, scale, B, L, want_bu=True):
    """x [B, L, P] complex (and bu = u A^T, for the backward) from u2 [B*L, m]
    in one kernel: the projection lands in TMEM and is scanned there."""
    m = u2.shape[1]
    P = abar.shape[0]
    x = torch.empty((B, L, P), dtype=torch.complex64, device=u2.device)
    bu = torch.empty_like(x) if want_bu else None
    ws = _fused_ws(B, L, P, u2.device)
    _lib.check(_lib.lib().lrx_mimo_fused_fwd(
        _lib.ptr(A), _lib.ptr(A_lo), _lib.ptr(u2), _lib.ptr(abar.contiguous()), _lib.ptr(scale.contiguous()),
        _lib.ptr(x), _lib.ptr(bu), B, L, m, P, _lib.ptr(ws), ws.numel(), _lib.stream()))
    return x, bu


def mimo_fused_bwd(A, A_lo, gy2, alpha, abar, scale, x, reduce=True):
    """(gbu [B, L, P], gabar [P]) from gy2 [B*L, m]: gx = alpha gy A^T lands in
    TMEM and the reverse scan reads it there.  d scale = sum_k conj(bu_k) g_k
    is left to the caller (lrx_mimo_coef_grads derives it from the weight-gradient GEMM)."""
    B, L, P = x.shape
    m = gy2.shape[1]
    n = _lib.i64()
    _lib.check(_lib.lib().lrx_mimo_fused_units(B, L, _lib.ref(n)))
    units = n.value
    gbu = torch.empty_like(x)
    gap = torch.empty(units * P, dtype=x.dtype, device=x.device)
    ws = _fused_ws(B, L, P, x.device)
    _lib.check(_lib.lib().lrx_mimo_fused_bwd(
        _lib.ptr(A), _lib.ptr(A_lo), _lib.ptr(gy2), float(alpha), _lib.ptr(abar.contiguous()),
        _lib.ptr(scale.contiguous()), _lib.ptr(x), _lib.ptr(gbu), _lib.ptr(gap), B, L, m, P, _lib.ptr(ws), ws.numel(),
        _lib.stream()))
    return gbu, (reduce_rows(gap, units, P) if reduce else gap.view(units, P))


def mimo_scan_fwd_ps(lam, delta, deltas, scheme, bu):
    """Per-step (asynchronous) MIMO scan: x_k = abar_k x_{k-1} + scale_k bu_k with
    the discretisation of lam [P] at deltas[b, k] * delta[p] done in the kernel."""
    B, L, P = bu.shape
    x = torch.empty_like(bu)
    lib = _lib.lib()
    code = _lib.code_of(bu.dtype)
    ws = _lib.workspace(lib.lrx_mimo_ps_workspace_bytes(code, B, L, P), bu.device)
    _lib.check(lib.lrx_mimo_fwd_ps(code, _lib.ptr(lam), _lib.ptr(delta), _lib.ptr(deltas), SCHEME_CODE[scheme],
                                   _lib.ptr(bu), _lib.ptr(x), B, L, P, _lib.ptr(ws), ws.numel(), _lib.stream()))
    return x


def mimo_scan_bwd_ps(lam, delta, deltas, scheme, bu, x, gx):
    """Pullback of mimo_scan_fwd_ps: (gbu [B, L, P], glam [P] complex, glog_delta [P])."""
    B, L, P = x.shape
    lib = _lib.lib()
    code = _lib.code_of(x.dtype)
    ck, nc = _lib.i64(), _lib.i64()
    _lib.check(lib.lrx_mimo_chunking(code, B, L, P, _lib.ref(ck), _lib.ref(nc)))
    R = nc.value * B
    gbu = torch.empty_like(x)
    glp = torch.empty((R, P), dtype=x.dtype, device=x.device)
    gdp = torch.empty((R, P), dtype=delta.dtype, device=x.device)
    ws = _lib.workspace(lib.lrx_mimo_ps_workspace_bytes(code, B, L, P), x.device)
    _lib.check(lib.lrx_mimo_bwd_ps(code, _lib.ptr(lam), _lib.ptr(delta), _lib.ptr(deltas), SCHEME_CODE[scheme],
                                   _lib.ptr(bu), _lib.ptr(x), _lib.ptr(gx), _lib.ptr(gbu), _lib.ptr(glp), _lib.ptr(gdp),
                                   B, L, P, _lib.ptr(ws), ws.numel(), _lib.stream()))
    return gbu, reduce_rows(glp, R, P), reduce_rows(gdp, R, P) * delta


# ---------------------------------------------------------------------------
# S4D (fused per-channel complex LTI scan)

S4D_FUSED_N = (8, 16, 32, 64)


def s4d_geometry(dtype, B, L, H, N):
    """(n_seg, ws_bytes): time segments of the fused S4D kernels (partial rows = n_seg * B)."""
    g = (ctypes.c_int64 * 2)()
    _lib.check(_lib.lib().lrx_s4d_geometry(_lib.code_of(dtype), B, L, H, N, g))
    return int(g[0]), int(g[1])


def s4d_scan_fwd(u, c, d, abar=None, w=None, lam=None, b=None, delta=None, deltas=None, scheme="zoh"):
    """y = Re(sum_n c x) + d u over u [B, L, H] (real, f32/f64) with
    x_n = abar_n x_n + w_n u.  Constant step: abar, w (= scale b) [H, N]
    complex.  Per step (asynchronous): lam, b [H, N] complex, delta [H]
    (= exp(log_delta)), deltas [B, L], scheme -- the kernel discretises every
    step.  Returns (y, ckpt, xlast)."""
    B, L, H = u.shape
    N = c.shape[-1]
    ck, nc = _lib.i64(), _lib.i64()
    _lib.check(_lib.lib().lrx_s4d_chunking(L, _lib.ref(ck), _lib.ref(nc)))
    _, wsb = s4d_geometry(u.dtype, B, L, H, N)
    y = torch.empty_like(u)
    ckpt = torch.empty((B, nc.value, H, N), dtype=c.dtype, device=u.device)
    xl = torch.empty((B, H, N), dtype=c.dtype, device=u.device)
    ws = _lib.workspace(wsb, u.device)
    _lib.check(_lib.lib().lrx_s4d_fwd(_lib.code_of(u.dtype), _lib.ptr(u), _lib.ptr(abar), _lib.ptr(w), _lib.ptr(lam),
                                      _lib.ptr(b), _lib.ptr(delta), _lib.ptr(deltas), SCHEME_CODE[scheme],
                                      _lib.ptr(c), _lib.ptr(d), _lib.ptr(y), _lib.ptr(ckpt), _lib.ptr(xl), B, L, H, N,
                                      _lib.ptr(ws), ws.numel(), _lib.stream()))
    return y, ckpt, xl


def s4d_scan_bwd(u, gy, c, d, ckpt, abar=None, w=None, lam=None, b=None, delta=None, deltas=None, scheme="zoh"):
    """Pullback of s4d_scan_fwd: dict gu [B, L, H]; gc [H, N] complex; gd [H];
    constant step: gabar, gw (= sum u g) [H, N] complex; per step: glam, gb
    [H, N] complex and gdl [H] (= d loss / d log_delta).  Batch / segment sums
    in a fixed order (lrx_reduce_rows)."""
    B, L, H = u.shape
    N = c.shape[-1]
    n_seg, wsb = s4d_geometry(u.dtype, B, L, H, N)
    R = n_seg * B
    gu = torch.empty_like(u)
    f = dict(dtype=c.dtype, device=u.device)
    p1, p2, gcp = (torch.empty((R, H * N), **f) for _ in range(3))
    p3 = torch.empty((R, H * N), dtype=u.dtype, device=u.device) if deltas is not None else None
    gdp = torch.empty((R, H), dtype=u.dtype, device=u.device)
    ws = _lib.workspace(wsb, u.device)
    _lib.check(_lib.lib().lrx_s4d_bwd(_lib.code_of(u.dtype), _lib.ptr(u), _lib.ptr(gy), _lib.ptr(abar), _lib.ptr(w),
                                      _lib.ptr(lam), _lib.ptr(b), _lib.ptr(delta), _lib.ptr(deltas),
                                      SCHEME_CODE[scheme], _lib.ptr(c), _lib.ptr(d), _lib.ptr(ckpt), _lib.ptr(gu),
                                      _lib.ptr(p1), _lib.ptr(p2), _lib.ptr(p3), _lib.ptr(gcp), _lib.ptr(gdp), B, L, H,
                                      N, _lib.ptr(ws), ws.numel(), _lib.stream()))
    out = {"gu": gu, "gc": reduce_rows(gcp, R, H * N).reshape(H, N), "gd": reduce_rows(gdp, R, H)}
    s1, s2 = reduce_rows(p1, R, H * N).reshape(H, N), reduce_rows(p2, R, H * N).reshape(H, N)
    if deltas is None:
        out.update(gabar=s1, gw=s2)
    else:
        out.update(glam=s1, gb=s2, gdl=reduce_rows(p3, R, H * N).reshape(H, N).sum(-1) * delta)
    return out
