"""The generic scan operator (mirrors pkg/src/linrec/scan.py:127-201).

x_k = a_k * x_{k-1} + b_k over time-major arrays b [L, *lanes] with a either
[*lanes] (constant) or [L, *lanes] (per-step).  Both entry points run the same
sm_100a operator (lrx_scan_fwd): by default a streaming walk -- one thread per
lane over its time segment, 8-step register tiles, and (when the lanes alone
cannot fill the GPU) time segments reduced by an aggregate pass and folded in
a fixed order; the single-pass anchored decoupled look-back remains behind
LRX_SCAN_STREAM=0.  `workers` is accepted for API compatibility and ignored --
the chunking is the GPU's, so unlike the reference (scan.py:160-162)
`scan_parallel` is bitwise identical to `scan_sequential` for every `workers`
value.

Inputs may be numpy arrays (copied to the current CUDA device; numpy is
returned) or CUDA tensors (results stay on the device).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .numerics import ShapeError

__all__ = ["MIN_CHUNK_LEN", "combine", "identity_element", "plan_chunks", "scan_sequential", "scan_parallel",
           "prepare", "StepState", "init_step_state", "step"]

MIN_CHUNK_LEN = 256  # scan.py:44 (host planning helper kept for API parity)

_OK_DTYPES = (torch.float32, torch.float64, torch.complex64, torch.complex128)


def combine(first, second):
    """(a1,b1) then (a2,b2) -> (a2 a1, a2 b1 + b2)  (scan.py:62-75)."""
    a1, b1 = first
    a2, b2 = second
    ts = [x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x)) for x in (a1, b1, a2, b2)]
    if not (ts[0].shape == ts[1].shape == ts[2].shape == ts[3].shape):
        raise ShapeError(f"combine operands must share a shape, got {tuple(ts[0].shape)}/{tuple(ts[1].shape)} "
                         f"and {tuple(ts[2].shape)}/{tuple(ts[3].shape)}")
    out = (ts[2] * ts[0], ts[2] * ts[1] + ts[3])
    if not isinstance(a1, torch.Tensor):
        return tuple(o.numpy() for o in out)
    return out


def identity_element(shape=(), dtype=np.float64):
    return np.ones(shape, dtype), np.zeros(shape, dtype)


def plan_chunks(length: int, workers: int):
    """Chunk plan of the reference's CPU thread pool (scan.py:139-149)."""
    if length < 1:
        raise ValueError(f"length must be >= 1, got {length}")
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    size = max(MIN_CHUNK_LEN, -(-length // workers))
    return [(s, min(s + size, length)) for s in range(0, length, size)]


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def _as_dev(x):
    if isinstance(x, torch.Tensor):
        return x.to(_dev()) if not x.is_cuda else x, False
    return torch.as_tensor(np.asarray(x)).to(_dev()), True


def prepare(a, b, x0):
    """Normalise to device [L, N] tensors of one dtype (scan.py:87-124)."""
    _lib.lib()
    a, host_a = _as_dev(a)
    b, host_b = _as_dev(b)
    host = host_a or host_b
    if b.ndim < 1 or b.shape[0] < 1:
        raise ShapeError(f"b must be [length, *lanes] with length >= 1, got shape {tuple(b.shape)}")
    lanes = tuple(b.shape[1:])
    if a.ndim == b.ndim:
        if a.shape != b.shape:
            raise ShapeError(f"per-step a must match b exactly: {tuple(a.shape)} vs {tuple(b.shape)}")
        per_step = True
    elif a.ndim == b.ndim - 1:
        if tuple(a.shape) != lanes:
            raise ShapeError(f"constant a must match b's lane shape {lanes}, got {tuple(a.shape)}")
        per_step = False
    else:
        raise ShapeError(f"a must be [*lanes] or [length, *lanes]; got {tuple(a.shape)} for b {tuple(b.shape)}")
    parts = [a, b]
    if x0 is not None:
        x0, _ = _as_dev(x0)
        parts.append(x0)
    dt = parts[0].dtype
    for p in parts[1:]:
        dt = torch.promote_types(dt, p.dtype)
    if dt not in _OK_DTYPES:
        dt = torch.promote_types(dt, torch.float64)
    L = b.shape[0]
    N = int(np.prod(lanes, dtype=np.int64)) if lanes else 1
    b2 = b.to(dt).contiguous().reshape(L, N)
    a2 = a.to(dt).contiguous().reshape((L, N) if per_step else (N,))
    if x0 is not None:
        if tuple(x0.shape) != lanes:
            raise ShapeError(f"x0 must have the lane shape {lanes}, got {tuple(x0.shape)}")
        x0 = x0.to(dt).contiguous().reshape(N)
    return a2, per_step, b2, x0, dt, lanes, host


def run_fwd(a2, per_step, b2, x02):
    L, N = b2.shape
    code = _lib.code_of(b2.dtype)
    L_ = _lib.lib()
    out = torch.empty_like(b2)
    ws = _lib.workspace(L_.lrx_scan_workspace_bytes(code, L, N), b2.device)
    _lib.check(L_.lrx_scan_fwd(code, int(per_step), _lib.ptr(a2), _lib.ptr(b2), _lib.ptr(x02), _lib.ptr(out),
                               L, N, _lib.ptr(ws), ws.numel(), _lib.stream()))
    return out


def _finish(out, L, lanes, host):
    out = out.reshape(L, *lanes)
    return out.cpu().numpy() if host else out


def scan_sequential(a, b, x0=None):
    """All states of the recurrence (scan.py:127-136)."""
    a2, per_step, b2, x02, dt, lanes, host = prepare(a, b, x0)
    return _finish(run_fwd(a2, per_step, b2, x02), b2.shape[0], lanes, host)


def scan_parallel(a, b, x0=None, workers: int = 1):
    """Same contract as scan_sequential (scan.py:152-201); see module notes."""
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    return scan_sequential(a, b, x0)


# ---------------------------------------------------------------------------
# single-step mode (scan.py:209-250)

class StepState:
    """Mutable carry for step(): the current state x (device tensor, updated in
    place) and the step count k (scan.py:209-216)."""

    def __init__(self, x, k=0):
        self.x = x
        self.k = k


def init_step_state(lanes, dtype=np.complex128, x0=None) -> StepState:
    """Fresh state of lane shape `lanes` (from x0 if given, else zeros) on the
    current CUDA device (scan.py:219-229)."""
    lanes = (lanes,) if np.isscalar(lanes) else tuple(lanes)
    td = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
          np.dtype(np.complex64): torch.complex64, np.dtype(np.complex128): torch.complex128}.get(np.dtype(dtype))
    if td is None:
        raise ValueError(f"unsupported state dtype {dtype}")
    x = torch.zeros(lanes, dtype=td, device=_dev())
    if x0 is not None:
        x0t = _as_dev(x0)[0]
        if tuple(x0t.shape) != lanes:
            raise ShapeError(f"x0 shape {tuple(x0t.shape)} != state shape {lanes}")
        x.copy_(x0t.to(td))
    return StepState(x=x, k=0)


def _period(t, shape):
    """Period of `t` when broadcast to `shape` in flat order, or None when it is
    not a plain trailing-dims broadcast (then it is materialised)."""
    if t.numel() == 1:
        return 1
    ts = tuple(t.shape)
    while ts and ts[0] == 1:  # leading singleton dims do not change the flat pattern
        ts = ts[1:]
    if ts == tuple(shape[len(shape) - len(ts):]):
        return t.numel()
    return None


def step(state: StepState, a_k, b_k):
    """Advance one step in place, x <- a_k x + b_k, on the device; returns
    (x, state).  a_k / b_k must broadcast to the state's shape without
    enlarging it (scan.py:232-250)."""
    x = state.x
    a = _as_dev(a_k)[0].to(x.dtype)
    b = _as_dev(b_k)[0].to(x.dtype)
    try:
        if torch.broadcast_shapes(x.shape, a.shape, b.shape) != x.shape:
            raise ShapeError(f"step operands {tuple(a.shape)}/{tuple(b.shape)} would enlarge state "
                             f"{tuple(x.shape)}")
    except RuntimeError as exc:
        raise ShapeError(str(exc)) from None
    shape = tuple(x.shape)
    ops = []
    for t in (a, b):
        p = _period(t, shape)
        if p is None:  # non-trailing broadcast (rare): materialise once
            t, p = torch.broadcast_to(t, shape).contiguous(), x.numel()
        ops.append((t.contiguous(), p))
    (a2, pa), (b2, pb) = ops
    _lib.check(_lib.lib().lrx_scan_step(_lib.code_of(x.dtype), _lib.ptr(x), _lib.ptr(a2), _lib.ptr(b2), x.numel(),
                                        pa, pb, _lib.stream()))
    state.k += 1
    return x, state
