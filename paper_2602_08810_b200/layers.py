"""The layer zoo, device-backed (mirrors pkg/src/linrec/layers.py).

Same constructors, parameter names/shapes/initialisation (bit-identical for
the same seed), forward signature and GradBundle layout as the reference, so
`make_layer` / `Layer.forward` / `layer_backward` are a drop-in.  Execution:

  * s6     lrx_s6_fwd / lrx_s6_bwd       fused selective scan (discretisation,
                                          softplus, readout, D skip) around the
                                          layer's projection GEMMs (cuBLAS)
  * rglru  lrx_rglru_fwd / lrx_rglru_bwd fused gated scan around the gate GEMMs
  * s5/lru lrx_mimo_fwd / lrx_mimo_bwd   complex scan fused with the input
                                          scaling and coefficient reductions,
                                          between the dense B/C projections
                                          (real GEMMs on interleaved complex)
  * s4d and the event-stream (per-step delta) paths of s4d/s5 run on the
    generic operator lrx_scan_fwd / lrx_scan_bwd.

`mode` ("sequential" / "parallel") and `workers` are accepted and validated;
both modes run the same chunk-parallel kernels and agree bitwise.  Inputs may
be numpy arrays (results come back as numpy) or CUDA tensors.  dtype "f32" /
"f64" as in the reference; "bf16" (s6, rglru) = bf16 activations, fp32
parameters and fp32 accumulation.
"""
from __future__ import annotations

import os
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import ops
from .autograd import Tape, layer_backward, pullback, scheme_partials
from .discretize import scheme_factors
from .numerics import Rng, ShapeError, real_dtype, sigmoid
from .scan import run_fwd

__all__ = ["LAYER_KINDS", "SCHEMES_BY_KIND", "UnknownLayer", "LayerConfig", "LayerStepState", "LinearRecurrence",
           "S4D", "S5", "LRU", "S6", "RGLRU", "make_layer", "init_layer", "lti_forward", "ltv_forward",
           "layer_step"]

LAYER_KINDS = ("s4d", "s5", "lru", "s6", "rglru")
# tokens from which the MIMO projections run on the tcgen05 GEMMs (below: cuBLAS)
_TC_MIN_TOKENS = int(os.environ.get("LRX_TC_MIN_TOKENS", "4096"))

SCHEMES_BY_KIND = {"s4d": ("zoh", "bilinear", "dirac"), "s5": ("zoh", "bilinear", "dirac"),
                   "lru": (), "s6": (), "rglru": ()}
STREAM_BLOCK = 512  # layers.py:77 (kept for API parity; the device path is not block-streamed)


class UnknownLayer(ValueError):
    """Requested layer kind is not in the registry."""


@dataclass
class LayerConfig:
    d_model: int
    d_state: int | None = None
    discretization: str | None = None
    asynchronous: bool = False
    dtype: str = "f64"
    extras: dict = field(default_factory=dict)


class LayerStepState:
    """Step-mode carry (layers.py:96-107): the device-resident state x, the
    step count k and the coefficient cache snapshotted from the layer's
    parameters when the state was created (init_state / forward with
    return_state=True).  step() updates x in place and allocates nothing but
    its output."""

    def __init__(self, kind: str, batch: int):
        self.kind = kind
        self.batch = batch
        self.k = 0
        self.x = None
        self.coef = {}


class StepGraph:
    """Graph-captured decode (the reference's generation
    loop calls Layer.step per token, model.py:512-573): the whole per-token
    step of one layer -- input projections, the fused lrx step kernel, the
    readout -- is captured once into a CUDA graph over static input / output
    buffers and replayed per token, so a token costs one graph launch instead
    of 3-6 kernel launches from the host.  The state is updated in place,
    exactly as by Layer.step (same kernels, same results).

        g = layer.step_graph(state)          # or StepGraph(layer, state)
        y_k = g.step(u_k)                    # [batch, d_model] CUDA tensor
        ys = g.run(u_seq)                    # [batch, T, d_model]

    `y_k` is the graph's static output buffer: clone it to keep it past the
    next step.  Per-step deltas (asynchronous dirac layers) are not captured."""

    def __init__(self, layer, state, warmup: int = 2):
        if layer.device.type != "cuda":
            raise RuntimeError("StepGraph needs a CUDA layer")
        self.layer, self.state = layer, state
        self.u = torch.zeros((state.batch, layer.d_model), dtype=layer.io_dtype, device=layer.device)
        x0 = state.x.clone()
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):  # library handles / workspaces before capture
            for _ in range(warmup):
                layer._step(state, self.u, None)
        cur.wait_stream(side)
        state.x.copy_(x0)  # warm-up steps leave no trace
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.y = layer._step(state, self.u, None)

    def step(self, u_k):
        """One token: u_k [batch, d_model] (device or host array) -> y_k."""
        u_k = u_k if isinstance(u_k, torch.Tensor) else torch.as_tensor(np.asarray(u_k))
        if tuple(u_k.shape) != tuple(self.u.shape):
            raise ShapeError(f"u_k shape {tuple(u_k.shape)} does not match {tuple(self.u.shape)}")
        self.u.copy_(u_k, non_blocking=True)
        self.graph.replay()
        self.state.k += 1
        return self.y

    def run(self, u_seq):
        """Feed u_seq [batch, T, d_model] token by token; returns y [batch, T, d_model]."""
        u_seq = u_seq if isinstance(u_seq, torch.Tensor) else torch.as_tensor(np.asarray(u_seq))
        u_seq = u_seq.to(self.layer.device)
        out = torch.empty(u_seq.shape, dtype=self.y.dtype, device=self.layer.device)
        for t in range(u_seq.shape[1]):
            out[:, t].copy_(self.step(u_seq[:, t]))
        return out


def _device(device=None):
    if device is not None:
        return torch.device(device)
    return torch.device("cuda", torch.cuda.current_device())


_SMS = {}


def _sm_count(device):
    """Multiprocessor count of `device` (cached; MIG slices and other parts
    differ from the B200's 148)."""
    idx = torch.device(device).index
    idx = torch.cuda.current_device() if idx is None else idx
    if idx not in _SMS:
        _SMS[idx] = torch.cuda.get_device_properties(idx).multi_processor_count
    return _SMS[idx]


def _pair(rng, shape, std, dt):
    g = rng.split(2)
    return np.asarray(g[0].normal(shape) * std, dt), np.asarray(g[1].normal(shape) * std, dt)


def _log_delta_init(rng, shape, dt):
    return np.asarray(rng.uniform(np.log(1e-3), np.log(1e-1), shape), dt)


def _tc_ok(a, *dims):
    """The tcgen05 3xTF32 GEMMs take fp32 operands with 16-byte rows and enough
    tokens to fill the GPU (see _MIMOBase._tc); the reduction width of the
    NT GEMM (dims[0]) is capped at 8192 (TMEM accumulation, lrx_gemm.cu)."""
    return (a.dtype == torch.float32 and a.is_cuda and a.shape[0] >= _TC_MIN_TOKENS
            and all(d % 4 == 0 and d >= 16 for d in dims) and dims[0] <= 8192)


def _proj(a2, w, lib=None):
    """a2 [T, K] @ w^T for a weight w [N, K]: tcgen05 3xTF32 (fp32-accurate)
    for fp32 activations at >= 4k tokens, else the library GEMM (`lib`,
    default _mm)."""
    if _tc_ok(a2, a2.shape[1], w.shape[0]) and w.dtype == torch.float32:
        return ops.gemm_f32(a2.contiguous(), w.contiguous())
    return (lib or _mm)(a2, w.T)


def _proj_acc(acc, a2, w):
    """acc + a2 @ w^T (acc [T, N] fp32, consumed): the add rides the GEMM epilogue."""
    if _tc_ok(a2, a2.shape[1], w.shape[0]) and w.dtype == torch.float32 and acc.dtype == torch.float32:
        return ops.gemm_f32(a2.contiguous(), w.contiguous(), Cin=acc.contiguous(), beta=1.0)
    return acc + a2 @ w.T


def _wgrad(g2, a2):
    """g2^T @ a2 (token-summed weight gradient): the split-K tcgen05 TN GEMM
    with its fixed-order partial sum, else the library GEMM."""
    if (_tc_ok(g2, g2.shape[1], a2.shape[1]) and a2.dtype == torch.float32 and min(g2.shape[1], a2.shape[1]) >= 32
            and g2.shape[1] * a2.shape[1] * max(1, g2.shape[0] // 4096) <= (1 << 31)):  # split-K partials <= 8 GB
        return ops.gemm_f32_tn(g2.contiguous(), a2.contiguous())
    return g2.T @ a2


def _mm_io(a, b):
    """a @ b in the activation dtype (RG-LRU bf16 gate pre-activations stay
    bf16: the scan streams them at 2 bytes): the bf16 tcgen05 GEMM with a
    bf16 epilogue."""
    if a.dtype == torch.bfloat16 and a.is_cuda:
        K, N = b.shape
        if K % 8 == 0 and N % 8 == 0 and K <= 16384:
            return ops.gemm_bf16(a.contiguous(), b.T.to(torch.bfloat16).contiguous(), out_dtype=torch.bfloat16)
    return torch.matmul(a, b)


def _mm(a, b):
    """Projection GEMM a @ b.  bf16 activations multiply bf16-cast weights on
    the tcgen05 tensor cores (ops.gemm_bf16: fp32 accumulation AND fp32
    output, so the scan sees unrounded projections; layers.py:1020-1027
    computes them at full precision); shapes the kernel does not take go to
    the library GEMM."""
    if a.dtype == torch.bfloat16:
        K, N = b.shape
        if a.is_cuda and K % 8 == 0 and N % 4 == 0 and K <= 16384:
            return ops.gemm_bf16(a.contiguous(), b.T.to(torch.bfloat16).contiguous())
        return torch.mm(a, b.to(torch.bfloat16), out_dtype=torch.float32)
    return a @ b


class LinearRecurrence:
    """Validation, mode dispatch and host/device plumbing shared by all kinds."""

    kind = ""
    lti = True
    continuous = True
    bf16_ok = False

    def __init__(self, d_model, d_state, discretization, asynchronous, dtype, device=None):
        if d_model < 1 or d_state < 1:
            raise ValueError(f"extents must be positive, got d_model={d_model}, d_state={d_state}")
        self.d_model = int(d_model)
        self.d_state = int(d_state)
        self.asynchronous = bool(asynchronous)
        if dtype == "bf16" and not self.bf16_ok:
            raise ValueError(f"{self.kind} supports dtype 'f32' or 'f64'; 'bf16' I/O is s6/rglru only")
        if dtype not in ("f32", "f64", "bf16"):
            real_dtype(dtype)  # raises the reference's ValueError for unknown specs
            dtype = "f32" if real_dtype(dtype) == np.dtype(np.float32) else "f64"
        self.dtype = dtype
        self.rdt = real_dtype(dtype)                         # numpy parameter dtype
        self.tdt = torch.float64 if dtype == "f64" else torch.float32
        self.tcdt = torch.complex128 if dtype == "f64" else torch.complex64
        self.io_dtype = torch.bfloat16 if dtype == "bf16" else self.tdt
        self.cdt = np.dtype(np.complex128) if dtype == "f64" else np.dtype(np.complex64)
        self.device = _device(device)
        # fail loudly now if the kernels cannot run; device="cpu" builds the
        # parameters only (inspection / checkpoint tooling) and cannot forward
        _lib.load(require_gpu=self.device.type == "cuda")
        if self.continuous:
            if discretization is None:
                discretization = "dirac" if self.asynchronous else "zoh"
            if discretization not in SCHEMES_BY_KIND[self.kind]:
                raise ValueError(f"{self.kind} supports discretizations {SCHEMES_BY_KIND[self.kind]}, "
                                 f"got {discretization!r}")
        elif discretization is not None:
            warnings.warn(f"{self.kind} is parameterized directly in discrete time; "
                          f"discretization={discretization!r} is ignored")
            discretization = None
        self.discretization = discretization

    # -- parameters --------------------------------------------------------
    def _p(self, arr):
        return torch.from_numpy(np.array(arr, copy=True, order="C")).to(self.device, self.tdt)

    def parameters(self):
        raise NotImplementedError

    # -- public API ----------------------------------------------------------
    def forward(self, u, mode="sequential", *, workers=1, deltas=None, tape=False, return_state=False):
        """Batched forward over u [batch, length, d_model] (layers.py:218-249)."""
        if self.device.type != "cuda":
            raise RuntimeError(f"{self.kind} layer lives on {self.device}; the scan runs on CUDA only "
                               "(no CPU fallback)")
        u, host = self._check_u(u)
        if mode not in ("sequential", "parallel"):
            raise ValueError(f"mode must be 'sequential' or 'parallel', got {mode!r}")
        if workers < 1:
            raise ValueError(f"workers must be >= 1, got {workers}")
        B, L, _ = u.shape
        deltas = self._check_deltas(deltas, B, L)
        y, saved, xf = self._forward(u, deltas, tape or return_state)
        out_y = y.cpu().numpy() if host else y
        if not (tape or return_state):
            return out_y
        out = [out_y]
        if tape:
            saved["host"] = host
            out.append(Tape(self.kind, **saved))
        if return_state:
            st = self.init_state(B)
            st.x = xf.contiguous().clone()  # step() updates it in place; the tape keeps its own copy
            st.k = L
            out.append(st)
        return tuple(out)

    def backward(self, tape, grad_y):
        return layer_backward(self, tape, grad_y)

    def init_state(self, batch: int = 1) -> LayerStepState:
        """A zeroed step-mode state for `batch` sequences (layers.py:271-273)."""
        if batch < 1:
            raise ValueError(f"batch must be >= 1, got {batch}")
        st = LayerStepState(self.kind, batch)
        st.x = self._zero_state(batch)
        st.coef = self._step_coef()
        return st

    def step(self, state, u_k, delta_k=None):
        """One recurrence update on the device state (layers.py:251-269):
        u_k [batch, d_model] (or [d_model] for a batch-1 state); returns
        (y_k, state).  numpy in -> numpy out, CUDA tensor in -> CUDA tensor out."""
        if self.device.type != "cuda":
            raise RuntimeError(f"{self.kind} layer lives on {self.device}; step runs on CUDA only")
        host = not isinstance(u_k, torch.Tensor)
        shape = tuple(np.shape(u_k)) if host else tuple(u_k.shape)
        squeeze = len(shape) == 1
        if squeeze:
            shape = (1,) + shape
        if shape != (state.batch, self.d_model):
            raise ShapeError(f"u_k shape {tuple(np.shape(u_k))} does not match state batch {state.batch} x "
                             f"d_model {self.d_model}")
        if delta_k is not None and not (self.continuous and self.lti):
            raise ValueError(f"{self.kind} does not accept per-step deltas")
        if host:
            uk = torch.as_tensor(np.ascontiguousarray(np.asarray(u_k, dtype=self.rdt)).reshape(shape))
        else:
            uk = u_k.reshape(shape)
        uk = uk.to(self.device, self.io_dtype).contiguous()
        y = self._step(state, uk, delta_k)
        state.k += 1
        out = y.cpu().numpy() if host else y
        return (out[0] if squeeze else out), state

    def step_graph(self, state) -> "StepGraph":
        """A CUDA-graph-captured per-token step bound to `state` (StepGraph)."""
        return StepGraph(self, state)

    def _zero_state(self, batch):
        raise NotImplementedError

    def _step_coef(self):
        return {}

    # -- plumbing --------------------------------------------------------------
    def _check_u(self, u):
        host = not isinstance(u, torch.Tensor)
        shape = tuple(np.shape(u)) if host else tuple(u.shape)
        if len(shape) != 3 or shape[2] != self.d_model:
            raise ShapeError(f"u must be [batch, length, d_model={self.d_model}], got shape {shape}")
        if shape[1] < 1:
            raise ShapeError("length must be >= 1")
        if host:
            ut = torch.as_tensor(np.ascontiguousarray(np.asarray(u, dtype=self.rdt)))
            ut = ut.to(self.device, non_blocking=False)
        else:
            ut = u.to(self.device)
        return ut.to(self.io_dtype).contiguous(), host

    def _check_deltas(self, deltas, B, L):
        if deltas is None:
            return None
        if not (self.lti and self.continuous):
            raise ValueError(f"per-step deltas apply to continuous-time LTI layers only, not {self.kind}")
        d = deltas if isinstance(deltas, torch.Tensor) else torch.as_tensor(np.asarray(deltas, dtype=self.rdt))
        d = d.to(self.device, self.tdt)
        if d.ndim == 1:
            d = d[None, :].expand(B, L) if d.shape[0] == L else d
        if tuple(d.shape) != (B, L):
            raise ShapeError(f"deltas must be [length] or [batch, length], got {tuple(np.shape(deltas))}")
        if bool(torch.any(d < 0)):
            raise ValueError("deltas must be non-negative")
        return d.contiguous()

    def _gy(self, gy, shape):
        g = gy if isinstance(gy, torch.Tensor) else torch.as_tensor(np.asarray(gy))
        g = g.to(self.device, self.io_dtype).contiguous()
        if tuple(g.shape) != tuple(shape):
            raise ShapeError(f"grad_y shape {tuple(g.shape)} does not match output {tuple(shape)}")
        return g

    @staticmethod
    def _out(grads, gu, host):
        if not host:
            return grads, gu
        return ({k: v.detach().cpu().numpy() for k, v in grads.items()}, gu.detach().cpu().numpy())

    def _w(self, t):
        """Weight in the activation dtype for the projection GEMMs."""
        return t.to(self.io_dtype) if self.io_dtype != t.dtype else t


# ---------------------------------------------------------------------------
# generic-operator helpers (s4d, async s4d/s5)

def _tm(x):
    """[B, L, ...] -> contiguous time-major [L, B*...]."""
    L = x.shape[1]
    return x.transpose(0, 1).contiguous().reshape(L, -1)


class S4D(LinearRecurrence):
    """Per-channel SISO complex diagonal SSM (layers.py:352-613)."""

    kind = "s4d"
    lti = True
    continuous = True

    def __init__(self, d_model, d_state=None, discretization=None, *, asynchronous=False, dtype="f64", rng=None,
                 seed=0, device=None):
        super().__init__(d_model, 64 if d_state is None else d_state, discretization, asynchronous, dtype, device)
        rng = rng if rng is not None else Rng(seed)
        r_b, r_c, r_d = rng.split(3)
        m, n, dt = self.d_model, self.d_state, self.rdt
        self.lambda_re_log = self._p(np.full((m, n), np.log(0.5), dt))
        self.lambda_im = self._p(np.broadcast_to(np.pi * np.arange(n, dtype=dt), (m, n)))
        br, bi = _pair(r_b, (m, n), 1.0, dt)
        cr, ci = _pair(r_c, (m, n), 1.0 / np.sqrt(n), dt)
        self.b_re, self.b_im, self.c_re, self.c_im = map(self._p, (br, bi, cr, ci))
        self.d = self._p(np.ones(m, dt))
        self.log_delta = self._p(_log_delta_init(r_d, m, dt))

    def parameters(self):
        return {"lambda_re_log": self.lambda_re_log, "lambda_im": self.lambda_im, "b.re": self.b_re,
                "b.im": self.b_im, "c.re": self.c_re, "c.im": self.c_im, "d": self.d, "log_delta": self.log_delta}

    def _lam(self):
        return torch.complex(-torch.exp(self.lambda_re_log), self.lambda_im)

    def _coeffs(self, deltas):
        """Coefficients in f64 (parameter-sized; see S5._abar_scale)."""
        lam = torch.complex(-torch.exp(self.lambda_re_log.double()), self.lambda_im.double())
        delta = torch.exp(self.log_delta.double())
        b = torch.complex(self.b_re.double(), self.b_im.double())
        if deltas is None:
            abar, scale = scheme_factors(self.discretization, lam, delta[:, None])
        else:
            deff = deltas.double()[:, :, None] * delta                       # [B,L,m]
            abar, scale = scheme_factors(self.discretization, lam, deff[..., None])
        return lam, delta, b, abar, scale

    def _fused(self, deltas, shape):
        """Fused S4D kernel (csrc/lrx_s4d.cu) for d_state in {8, 16, 32, 64}:
        constant steps and per-step deltas (discretised in the kernel), time
        segments for long sequences over few channels; other widths take the
        generic operator path."""
        return self.d_state in ops.S4D_FUSED_N and os.environ.get("LRX_S4D_GENERIC") != "1"

    def _fused_args(self, deltas):
        c = torch.complex(self.c_re, self.c_im).contiguous()
        if deltas is None:  # coefficients in f64 on the device, one launch (lrx_s4d_coef)
            m, n = self.d_model, self.d_state
            abar = torch.empty((m, n), dtype=self.tcdt, device=self.device)
            w = torch.empty_like(abar)
            _lib.check(_lib.lib().lrx_s4d_coef(
                _lib.code_of(self.tdt), ops.SCHEME_CODE[self.discretization], _lib.ptr(self.lambda_re_log),
                _lib.ptr(self.lambda_im), _lib.ptr(self.b_re), _lib.ptr(self.b_im), _lib.ptr(self.log_delta), m, n,
                _lib.ptr(abar), _lib.ptr(w), _lib.stream()))
            return c, dict(abar=abar, w=w)
        # per-step discretisation in the kernel; bilinear cannot be singular
        # here: Re(lambda) = -exp(.) < 0 and deltas >= 0 keep |1 - delta lambda / 2| >= 1
        return c, dict(lam=self._lam().to(self.tcdt).contiguous(), b=torch.complex(self.b_re, self.b_im).contiguous(),
                       delta=torch.exp(self.log_delta).contiguous(), deltas=deltas.to(self.tdt).contiguous(),
                       scheme=self.discretization)

    def _forward(self, u, deltas, keep):
        if self._fused(deltas, u.shape):
            c, kw = self._fused_args(deltas)
            y, ckpt, xlast = ops.s4d_scan_fwd(u, c, self.d.contiguous(), **kw)
            saved = {"u": u, "ckpt": ckpt, "deltas": deltas, "fused": True} if keep else {}
            return y, saved, xlast
        B, L, m = u.shape
        n = self.d_state
        lam, delta, b, abar, scale = self._coeffs(deltas)
        w = (scale * b).to(self.tcdt) * u[..., None]                          # [B,L,m,n]
        abar = abar.to(self.tcdt)
        if deltas is None:
            a2, per = abar.reshape(-1).repeat(B), False
        else:
            a2, per = _tm(abar), True
        x2 = run_fwd(a2.contiguous(), per, _tm(w), None)                     # [L, B*m*n]
        xt = x2.reshape(L, B, m, n)
        c = torch.complex(self.c_re, self.c_im)
        y = torch.einsum("lbhn,hn->blh", xt, c).real + self.d * u
        saved = {"u": u, "x2": x2, "deltas": deltas} if keep else {}
        return y.contiguous(), saved, xt[-1]

    # -- step mode (layers.py:550-613) ----------------------------------------
    def _zero_state(self, batch):
        return torch.zeros((batch, self.d_model, self.d_state), dtype=self.tcdt, device=self.device)

    def _step_coef(self):
        lam, delta, b, abar, scale = self._coeffs(None)
        return {"lam": lam, "delta": delta, "b": b, "abar": abar.to(self.tcdt).contiguous(),
                "w": (scale * b).to(self.tcdt).contiguous(),
                "c": torch.complex(self.c_re, self.c_im).contiguous(), "d": self.d.contiguous()}

    def _step(self, st, uk, delta_k):
        cf = st.coef
        abar, w = cf["abar"], cf["w"]
        if delta_k is not None:
            if self.discretization != "dirac":
                raise NotImplementedError("per-step deltas in step mode require the dirac scheme")
            a_k, s_k = scheme_factors("dirac", cf["lam"], cf["delta"][:, None] * float(delta_k))
            abar, w = a_k.to(self.tcdt).contiguous(), (s_k * cf["b"]).to(self.tcdt).contiguous()
        y = torch.empty((st.batch, self.d_model), dtype=self.tdt, device=self.device)
        _lib.check(_lib.lib().lrx_s4d_step(_lib.code_of(self.tcdt), _lib.ptr(st.x), _lib.ptr(abar), _lib.ptr(w),
                                           _lib.ptr(cf["c"]), _lib.ptr(cf["d"]), _lib.ptr(uk), _lib.ptr(y),
                                           st.batch, self.d_model, self.d_state, _lib.stream()))
        return y

    def _backward_fused(self, s, gy):
        u, ckpt, host, deltas = s["u"], s["ckpt"], s["host"], s["deltas"]
        gy = self._gy(gy, u.shape)
        c, kw = self._fused_args(deltas)
        r = ops.s4d_scan_bwd(u, gy, c, self.d.contiguous(), ckpt, **kw)
        gc = r["gc"]
        if deltas is None:  # scheme partials in f64 on the device, one launch (lrx_s4d_coef_grads)
            m, n = self.d_model, self.d_state
            g = torch.empty((4, m, n), dtype=self.tdt, device=self.device)
            gld = torch.empty(m, dtype=self.tdt, device=self.device)
            _lib.check(_lib.lib().lrx_s4d_coef_grads(
                _lib.code_of(self.tdt), ops.SCHEME_CODE[self.discretization], _lib.ptr(self.lambda_re_log),
                _lib.ptr(self.lambda_im), _lib.ptr(self.b_re), _lib.ptr(self.b_im), _lib.ptr(self.log_delta),
                _lib.ptr(r["gabar"].contiguous()), _lib.ptr(r["gw"].contiguous()), m, n, _lib.ptr(g[0]),
                _lib.ptr(g[1]), _lib.ptr(g[2]), _lib.ptr(g[3]), _lib.ptr(gld), _lib.stream()))
            grads = {"lambda_re_log": g[0], "lambda_im": g[1], "b.re": g[2], "b.im": g[3], "log_delta": gld}
        else:  # the kernel accumulated the per-step scheme partials (autograd.py:186-211)
            glam, gb = r["glam"], r["gb"]
            grads = {"lambda_re_log": -torch.exp(self.lambda_re_log.to(glam.real.dtype)) * glam.real,
                     "lambda_im": glam.imag, "b.re": gb.real, "b.im": gb.imag, "log_delta": r["gdl"]}
        grads.update({"c.re": gc.real, "c.im": gc.imag, "d": r["gd"]})
        grads = {k: v.to(self.tdt).contiguous() for k, v in grads.items()}
        return self._out({k: grads[k] for k in self.parameters()}, r["gu"], host)

    def _backward(self, s, gy):
        if s.get("fused"):
            return self._backward_fused(s, gy)
        u, x2, deltas, host = s["u"], s["x2"], s["deltas"], s["host"]
        B, L, m = u.shape
        n = self.d_state
        gy = self._gy(gy, u.shape)
        lam, delta, b, abar, scale = self._coeffs(deltas)
        cd = self.tcdt
        c = torch.complex(self.c_re, self.c_im)
        xt = x2.reshape(L, B, m, n)
        gd = (gy * u).sum((0, 1))
        gu = gy * self.d
        gyt = gy.transpose(0, 1)
        gc = torch.einsum("lbh,lbhn->hn", gyt.to(cd), xt.conj())
        gxt = gyt[..., None] * c.conj()
        per = deltas is not None
        a2 = _tm(abar.to(cd)) if per else abar.to(cd).reshape(-1).repeat(B)
        g2, ga, _ = pullback(a2.contiguous(), per, x2, None, gxt.reshape(L, -1).contiguous())
        gw = g2.reshape(L, B, m, n)
        c128 = torch.complex128
        if not per:
            gabar = ga.reshape(B, m, n).sum(0).to(c128)
            gpsi = torch.einsum("lbhn,blh->hn", gw, u.to(cd)).to(c128)
            gu = gu + torch.einsum("lbhn,hn->blh", gw, (scale * b).conj().to(cd)).real
            gscale = b.conj() * gpsi
            gb = scale.conj() * gpsi
            dal, dad, dsl, dsd = scheme_partials(self.discretization, lam, delta[:, None], abar, scale)
            glam = dal.conj() * gabar + dsl.conj() * gscale
            gdel = ((dad.conj() * gabar).real + (dsd.conj() * gscale).real).sum(-1)
            glog_delta = gdel * delta
        else:
            ga_k = ga.reshape(L, B, m, n).transpose(0, 1).to(c128)
            gw_b = gw.transpose(0, 1)
            gpsi_k = (gw_b * u[..., None]).to(c128)
            gu = gu + torch.einsum("blhn,blhn->blh", gw_b, (scale * b).conj().to(cd)).real
            gscale_k = b.conj() * gpsi_k
            gb = (scale.conj() * gpsi_k).sum((0, 1))
            deff = deltas.double()[:, :, None] * delta
            dal, dad, dsl, dsd = scheme_partials(self.discretization, lam, deff[..., None], abar, scale)
            glam = (dal.conj() * ga_k + dsl.conj() * gscale_k).sum((0, 1))
            gdeff = ((dad.conj() * ga_k).real + (dsd.conj() * gscale_k).real).sum(-1)
            glog_delta = torch.einsum("blh,bl->h", gdeff, deltas.double()) * delta
        t = self.tdt
        grads = {"lambda_re_log": (-torch.exp(self.lambda_re_log.double()) * glam.real).to(t),
                 "lambda_im": glam.imag.to(t).contiguous(),
                 "b.re": gb.real.to(t).contiguous(), "b.im": gb.imag.to(t).contiguous(),
                 "c.re": gc.real.contiguous(), "c.im": gc.imag.contiguous(), "d": gd,
                 "log_delta": glog_delta.to(t)}
        return self._out(grads, gu, host)


# ---------------------------------------------------------------------------
# MIMO: S5 / LRU


class _MIMOBase(LinearRecurrence):
    """x [B, L, P] complex between bu = B u and y = OUT Re(C x) + D u
    (layers.py:616-704).  Complex projections run as real GEMMs on the
    interleaved (re, im) layout."""

    OUT_SCALE = 1.0

    @property
    def _P(self):
        raise NotImplementedError

    def _wb(self):
        """[m, 2P] real: u @ Wb = interleaved B u."""
        return torch.stack((self.B_re.T, self.B_im.T), dim=-1).reshape(self.d_model, 2 * self._P).contiguous()

    def _wc(self):
        """[2P, m] real: x2 @ Wc = Re(C x)."""
        return torch.stack((self.C_re.T, -self.C_im.T), dim=1).reshape(2 * self._P, self.d_model).contiguous()

    def _abar_scale(self, deltas):
        """(abar, scale) in the compute dtype plus f64 context for the grads."""
        raise NotImplementedError

    # -- fused coefficient work (csrc/lrx_coef.cu) ------------------------------
    _KIND_CODE = None
    _SCHEME_CODE = {"zoh": 0, "bilinear": 1, "dirac": 2}

    def _coef_params(self):
        raise NotImplementedError

    def _fused(self, deltas):
        """One-launch coefficient/layout work for constant steps (bilinear S5
        keeps the torch path: its singular-set check is a host decision)."""
        return deltas is None and (self.kind == "lru" or self.discretization in ("zoh", "dirac"))

    def _coef_pack(self, fused=(False, False)):
        """abar, scale, the f64 context and the real GEMM layouts of B / C
        (with 3xTF32 low planes for fp32) from one lrx_mimo_coef launch;
        fused = (forward, backward): B / the gx projection also in the fused
        projection + scan layout (wbf / wgf [256, m])."""
        P, m, dev = self._P, self.d_model, self.device
        lo = self.tdt == torch.float32
        abar = torch.empty(P, dtype=self.tcdt, device=dev)
        scale = torch.empty(P, dtype=self.tcdt, device=dev)
        extra = torch.empty((P, 8), dtype=torch.float64, device=dev)
        w = torch.empty((4, 2 if lo else 1, 2 * P * m), dtype=self.tdt, device=dev)
        wbf, wgf = (torch.empty((2 if lo else 1, 256 * m), dtype=self.tdt, device=dev) if f else None for f in fused)
        p0, p1, p2 = self._coef_params()
        _lib.check(_lib.lib().lrx_mimo_coef(
            self._KIND_CODE, self._SCHEME_CODE.get(self.discretization, 0), _lib.code_of(self.tdt), _lib.ptr(p0),
            _lib.ptr(p1), _lib.ptr(p2), _lib.ptr(self.B_re), _lib.ptr(self.B_im), _lib.ptr(self.C_re),
            _lib.ptr(self.C_im), P, m, _lib.ptr(abar), _lib.ptr(scale), _lib.ptr(extra), _lib.ptr(w[0]),
            _lib.ptr(w[1]), _lib.ptr(w[2]), _lib.ptr(w[3]), _lib.ptr(wbf), _lib.ptr(wgf), int(lo), _lib.stream()))
        shp = {"wbt": (2 * P, m), "wb": (m, 2 * P), "wct": (m, 2 * P), "wgt": (2 * P, m)}
        pk = {"abar": abar, "scale": scale, "extra": extra}
        for i, k in enumerate(shp):
            pk[k] = w[i, 0].view(shp[k])
            pk[k + "_lo"] = w[i, 1].view(shp[k]) if lo else None
        for k, t in (("wbf", wbf), ("wgf", wgf)):
            if t is not None:
                pk[k], pk[k + "_lo"] = t[0].view(256, m), (t[1].view(256, m) if lo else None)
        return pk

    def _coef_grads_fused(self, pk, ga, gsc, R, R2):
        P, m, dev, dt = self._P, self.d_model, self.device, self.tdt
        g = torch.empty((3, P), dtype=dt, device=dev)
        gb = torch.empty((2, P, m), dtype=dt, device=dev)
        gc = torch.empty((2, m, P), dtype=dt, device=dev)
        p0, p1, p2 = self._coef_params()
        _lib.check(_lib.lib().lrx_mimo_coef_grads(
            self._KIND_CODE, self._SCHEME_CODE.get(self.discretization, 0), _lib.code_of(dt), _lib.ptr(p0),
            _lib.ptr(p1), _lib.ptr(p2), _lib.ptr(pk["extra"]), _lib.ptr(ga.contiguous()), ga.numel() // P,
            _lib.ptr(gsc.contiguous() if gsc is not None else None), gsc.numel() // P if gsc is not None else 1,
            _lib.ptr(R.contiguous()),
            _lib.ptr(R2.contiguous()), _lib.ptr(self.B_re), _lib.ptr(self.B_im), float(self.OUT_SCALE), _lib.ptr(g[0]),
            _lib.ptr(g[1]), _lib.ptr(g[2]), _lib.ptr(gb[0]), _lib.ptr(gb[1]), _lib.ptr(gc[0]), _lib.ptr(gc[1]),
            P, m, _lib.stream()))
        keys = self._coef_keys
        return {keys[0]: g[0], keys[1]: g[1], keys[2]: g[2], "B.re": gb[0], "B.im": gb[1], "C.re": gc[0],
                "C.im": gc[1]}

    def _tc(self, K, T):
        """fp32 projections run on the tcgen05 3xTF32 GEMMs (ops.gemm_f32 /
        gemm_f32_tn) when the row width keeps TMA rows 16-byte aligned and
        there are enough tokens T (>= 4096, measured: C1 LRU 8k tokens 0.18 ->
        0.15 ms per step on them; at 1k tokens cuBLAS wins); f64 layers, odd
        widths and tiny batches use the library (cuBLAS) GEMM."""
        return self.tdt == torch.float32 and K % 4 == 0 and K <= 8192 and T >= _TC_MIN_TOKENS

    def _forward(self, u, deltas, keep):
        if self._fused(deltas):
            return self._forward_fused(u, keep)
        B, L, m = u.shape
        P = self._P
        u2 = u.reshape(B * L, m)
        if self._tc(m, B * L):
            bu = torch.view_as_complex(ops.gemm_f32(u2.contiguous(), self._wb().T.contiguous()).reshape(B, L, P, 2))
        else:
            bu = torch.view_as_complex((u2 @ self._wb()).reshape(B, L, P, 2))   # [B,L,P]
        if deltas is None:
            abar, scale, extra = self._abar_scale(deltas)
            x = ops.mimo_scan_fwd(abar, scale, bu)
        else:  # per-step discretisation inside the scan kernel (no [B, L, P] coefficient planes)
            x = ops.mimo_scan_fwd_ps(*self._ps_args(deltas), bu)
        if self._tc(2 * P, B * L):  # y = OUT Re(C x) + D u, the D u skip fused into the GEMM epilogue
            y = ops.gemm_f32(torch.view_as_real(x).reshape(B * L, 2 * P), self._wc().T.contiguous(),
                             Cin=u2.contiguous(), colscale=self.D.contiguous(),
                             alpha=self.OUT_SCALE).reshape(B, L, m)
        else:
            y = torch.addmm((self.D * u).reshape(B * L, m), torch.view_as_real(x).reshape(B * L, 2 * P), self._wc(),
                            alpha=self.OUT_SCALE).reshape(B, L, m)
        saved = {"u": u, "x": x, "bu": bu, "deltas": deltas} if keep else {}
        return y, saved, x[:, -1]

    def _gemm_scan(self, B, L):
        """Which directions run the projection and the scan as one tcgen05
        kernel (csrc/lrx_mimo_fused.cu: bu / gx scanned out of TMEM), as
        (forward, backward).  Domain: fp32 on the tensor-core route, P <= 128,
        L <= 8192.  Measured (tools/gpu_fused_ab2.sh): both win with enough
        128-step units to fill the GPU (C2, 1024 units: step 801 -> 739 us);
        with few units (C1: 64) the serial per-unit scan loses to the
        separate launches (133 -> 175 us).  LRX_MIMO_FUSED / LRX_MIMO_FUSED_BWD
        = 0 / 1 force a direction off / on."""
        ok = self._tc(self.d_model, B * L) and ops.mimo_fused_supported(B, L, self.d_model, self._P, self.tdt)
        units = B * -(-L // 128)
        auto = units >= 4 * _sm_count(self.device)

        def on(var):
            env = os.environ.get(var)
            return ok and (env == "1" or (env is None and auto))
        return on("LRX_MIMO_FUSED"), on("LRX_MIMO_FUSED_BWD")

    def _forward_fused(self, u, keep):
        B, L, m = u.shape
        P = self._P
        u2 = u.reshape(B * L, m).contiguous()
        fused = self._gemm_scan(B, L)
        pk = self._coef_pack(fused=fused)
        if fused[0]:
            x, bu = ops.mimo_fused_fwd(pk["wbf"], pk["wbf_lo"], u2, pk["abar"], pk["scale"], B, L, want_bu=False)
        else:
            if self._tc(m, B * L):
                bu2 = ops.gemm_f32(u2, pk["wbt"], Bt_lo=pk["wbt_lo"])
            else:
                bu2 = u2 @ pk["wb"]
            bu = torch.view_as_complex(bu2.reshape(B, L, P, 2))
            x = ops.mimo_scan_fwd(pk["abar"], pk["scale"], bu)
        x2 = torch.view_as_real(x).reshape(B * L, 2 * P)
        if self._tc(2 * P, B * L):  # y = OUT Re(C x) + D u, the D u skip fused into the epilogue
            y = ops.gemm_f32(x2, pk["wct"], Bt_lo=pk["wct_lo"], Cin=u2, colscale=self.D.contiguous(),
                             alpha=self.OUT_SCALE).reshape(B, L, m)
        else:
            y = torch.addmm((self.D * u).reshape(B * L, m), x2, pk["wct"].T, alpha=self.OUT_SCALE).reshape(B, L, m)
        saved = {"u": u, "x": x, "bu": bu, "deltas": None, "pk": pk} if keep else {}
        return y, saved, x[:, -1]

    def _backward_fused(self, s, gy):
        u, x, bu, pk, host = s["u"], s["x"], s["bu"], s["pk"], s["host"]
        B, L, m = u.shape
        P = self._P
        gy = self._gy(gy, u.shape)
        gy2, u2 = gy.reshape(B * L, m).contiguous(), u.reshape(B * L, m).contiguous()
        x2 = torch.view_as_real(x).reshape(B * L, 2 * P)
        gD = ops.reduce_rows(gy2, B * L, m, other=u2)  # sum_t gy u per channel
        tn = self._tc(m, B * L) and self._tc(2 * P, B * L)
        R = ops.gemm_f32_tn(gy2, x2) if tn else gy2.T @ x2     # [m, 2P]
        if "wgf" in pk:
            gbu, ga = ops.mimo_fused_bwd(pk["wgf"], pk["wgf_lo"], gy2, self.OUT_SCALE, pk["abar"], pk["scale"], x,
                                         reduce=False)
            gsc = None
        else:
            if self._tc(m, B * L):
                gx2 = ops.gemm_f32(gy2, pk["wgt"], Bt_lo=pk["wgt_lo"], alpha=self.OUT_SCALE)
            else:
                gx2 = self.OUT_SCALE * (gy2 @ pk["wct"])
            gx = torch.view_as_complex(gx2.reshape(B, L, P, 2))
            gbu, ga, gsc = ops.mimo_scan_bwd(pk["abar"], pk["scale"], bu, x, gx, reduce=False)
        gbu2 = torch.view_as_real(gbu).reshape(B * L, 2 * P)
        R2 = ops.gemm_f32_tn(gbu2, u2) if tn else gbu2.T @ u2  # [2P, m]
        if self._tc(2 * P, B * L):  # gu = D gy + Re(g conj(B)), the skip fused into the epilogue
            gu = ops.gemm_f32(gbu2, pk["wb"], Bt_lo=pk["wb_lo"], Cin=gy2, colscale=self.D.contiguous()).reshape(B, L, m)
        else:
            gu = gy * self.D + (gbu2 @ pk["wbt"]).reshape(B, L, m)
        grads = self._coef_grads_fused(pk, ga, gsc, R, R2)
        grads["D"] = gD
        return self._out({k: grads[k] for k in self.parameters()}, gu, host)

    # -- step mode (layers.py:708-783) ----------------------------------------
    def _zero_state(self, batch):
        return torch.zeros((batch, self._P), dtype=self.tcdt, device=self.device)

    def _step_coef(self):
        abar, scale, extra = self._abar_scale(None)
        return {"abar": abar.contiguous(), "scale": scale.contiguous(), "extra": extra,
                "B": (self.B_re.contiguous(), self.B_im.contiguous()),
                "C": (self.C_re.contiguous(), self.C_im.contiguous()), "D": self.D.contiguous()}

    def _step(self, st, uk, delta_k):
        cf = st.coef
        abar, scale = cf["abar"], cf["scale"]
        if delta_k is not None:
            if self.discretization != "dirac":
                raise NotImplementedError("per-step deltas in step mode require the dirac scheme")
            ex = cf["extra"]
            a_k, s_k = scheme_factors("dirac", ex["lam"], ex["delta"] * float(delta_k))
            abar, scale = a_k.to(self.tcdt).contiguous(), s_k.to(self.tcdt).contiguous()
        y = torch.empty((st.batch, self.d_model), dtype=self.tdt, device=self.device)
        _lib.check(_lib.lib().lrx_mimo_step(
            _lib.code_of(self.tcdt), _lib.ptr(st.x), _lib.ptr(abar), _lib.ptr(scale), _lib.ptr(cf["B"][0]),
            _lib.ptr(cf["B"][1]), _lib.ptr(cf["C"][0]), _lib.ptr(cf["C"][1]), _lib.ptr(cf["D"]), _lib.ptr(uk),
            _lib.ptr(y), float(self.OUT_SCALE), st.batch, self._P, self.d_model, _lib.stream()))
        return y

    def _ps_args(self, deltas):
        """(lam [P], delta [P], deltas [B, L], scheme) for the per-step kernels."""
        lam = torch.complex(-torch.exp(self.lambda_re_log), self.lambda_im).to(self.tcdt).contiguous()
        return lam, torch.exp(self.log_delta).contiguous(), deltas.to(self.tdt).contiguous(), self.discretization

    def _scan_backward(self, x, bu, gx, abar, scale, deltas):
        """(gbu [B,L,P], gabar, gscale) of the constant-step scan."""
        return ops.mimo_scan_bwd(abar, scale, bu, x, gx)

    def _backward(self, s, gy):
        if "pk" in s:
            return self._backward_fused(s, gy)
        u, x, bu, deltas, host = s["u"], s["x"], s["bu"], s["deltas"], s["host"]
        B, L, m = u.shape
        P = self._P
        gy = self._gy(gy, u.shape)
        gy2, u2 = gy.reshape(B * L, m), u.reshape(B * L, m)
        x2 = torch.view_as_real(x).reshape(B * L, 2 * P)
        osc = self.OUT_SCALE
        gD = ops.reduce_rows(gy2.contiguous(), B * L, m, other=u2.contiguous())  # sum_t gy u per channel
        tn = self._tc(m, B * L) and self._tc(2 * P, B * L)
        R = ops.gemm_f32_tn(gy2.contiguous(), x2) if tn else gy2.T @ x2     # [m, 2P]
        gC_re, gC_im = osc * R[:, 0::2], -osc * R[:, 1::2]
        wg = torch.stack((self.C_re, -self.C_im), dim=-1).reshape(m, 2 * P)
        if self._tc(m, B * L):
            gx = torch.view_as_complex(ops.gemm_f32(gy2.contiguous(), wg.T.contiguous(), alpha=osc).reshape(B, L, P, 2))
        else:
            gx = torch.view_as_complex((osc * (gy2 @ wg)).reshape(B, L, P, 2)).contiguous()
        if deltas is None:
            abar, scale, extra = self._abar_scale(deltas)
            gbu, ga, gsc = self._scan_backward(x, bu, gx, abar, scale, deltas)
            coef = {k: v.to(self.tdt) for k, v in self._coef_grads(ga, gsc, extra, deltas).items()}
        else:  # the kernel accumulates the per-step scheme partials (autograd.py:186-211)
            gbu, glam, glog_delta = ops.mimo_scan_bwd_ps(*self._ps_args(deltas), bu, x, gx.contiguous())
            coef = {"lambda_re_log": (-torch.exp(self.lambda_re_log) * glam.real).to(self.tdt),
                    "lambda_im": glam.imag.to(self.tdt).contiguous(), "log_delta": glog_delta.to(self.tdt)}
        gbu2 = torch.view_as_real(gbu.contiguous()).reshape(B * L, 2 * P)
        R2 = ops.gemm_f32_tn(gbu2, u2.contiguous()) if tn else gbu2.T @ u2  # [2P, m]
        if self._tc(2 * P, B * L):  # gu = D gy + Re(g conj(B)), the skip fused into the epilogue
            gu = ops.gemm_f32(gbu2, self._wb(), Cin=gy2.contiguous(), colscale=self.D.contiguous()).reshape(B, L, m)
        else:
            gu = gy * self.D + (gbu2 @ self._wb().T).reshape(B, L, m)
        grads = coef
        grads.update({"B.re": R2[0::2].contiguous(), "B.im": R2[1::2].contiguous(),
                      "C.re": gC_re.contiguous(), "C.im": gC_im.contiguous(), "D": gD})
        return self._out({k: grads[k] for k in self.parameters()}, gu, host)


class S5(_MIMOBase):
    """MIMO SSM, conjugate-pair storage, y = 2 Re(C x) + D u (layers.py:786-895)."""

    kind = "s5"
    lti = True
    continuous = True
    OUT_SCALE = 2.0

    def __init__(self, d_model, d_state=None, discretization=None, *, asynchronous=False, dtype="f64", rng=None,
                 seed=0, device=None):
        d_state = 64 if d_state is None else d_state
        if d_state % 2:
            raise ValueError(f"s5 stores conjugate pairs and needs even d_state, got {d_state}")
        super().__init__(d_model, d_state, discretization, asynchronous, dtype, device)
        rng = rng if rng is not None else Rng(seed)
        r_b, r_c, r_d = rng.split(3)
        m, P, dt = self.d_model, d_state // 2, self.rdt
        self.lambda_re_log = self._p(np.full((P,), np.log(0.5), dt))
        self.lambda_im = self._p(np.pi * np.arange(P, dtype=dt))
        Br, Bi = _pair(r_b, (P, m), 1.0 / np.sqrt(m), dt)
        Cr, Ci = _pair(r_c, (m, P), 1.0 / np.sqrt(P), dt)
        self.B_re, self.B_im, self.C_re, self.C_im = map(self._p, (Br, Bi, Cr, Ci))
        self.D = self._p(np.ones(m, dt))
        self.log_delta = self._p(_log_delta_init(r_d, P, dt))

    _KIND_CODE = 0
    _coef_keys = ("lambda_re_log", "lambda_im", "log_delta")

    @property
    def _P(self):
        return self.d_state // 2

    def _coef_params(self):
        return self.lambda_re_log, self.lambda_im, self.log_delta

    def parameters(self):
        return {"lambda_re_log": self.lambda_re_log, "lambda_im": self.lambda_im, "B.re": self.B_re,
                "B.im": self.B_im, "C.re": self.C_re, "C.im": self.C_im, "D": self.D, "log_delta": self.log_delta}

    def _abar_scale(self, deltas):
        # parameter-sized discretisation in f64 (the f32 ZOH partial
        # (delta abar lam - (abar - 1)) / lam^2 cancels catastrophically)
        lam = torch.complex(-torch.exp(self.lambda_re_log.double()), self.lambda_im.double())
        delta = torch.exp(self.log_delta.double())
        d_arg = delta if deltas is None else deltas.double()[:, :, None] * delta
        abar, scale = scheme_factors(self.discretization, lam, d_arg)
        return abar.to(self.tcdt), scale.to(self.tcdt), {"lam": lam, "delta": delta, "d_arg": d_arg,
                                                         "abar": abar, "scale": scale}

    def _coef_grads(self, ga, gsc, extra, deltas):
        lam, delta, d_arg = extra["lam"], extra["delta"], extra["d_arg"]
        ga, gsc = ga.to(torch.complex128), gsc.to(torch.complex128)
        # constant steps (per-step deltas accumulate these partials in lrx_mimo_bwd_ps)
        dal, dad, dsl, dsd = scheme_partials(self.discretization, lam, d_arg, extra["abar"], extra["scale"])
        glam = dal.conj() * ga + dsl.conj() * gsc
        gdel = (dad.conj() * ga).real + (dsd.conj() * gsc).real
        glog_delta = gdel * delta
        return {"lambda_re_log": -torch.exp(self.lambda_re_log.double()) * glam.real,
                "lambda_im": glam.imag.contiguous(), "log_delta": glog_delta}


class LRU(_MIMOBase):
    """Linear recurrent unit, ring parameterisation (layers.py:898-980)."""

    kind = "lru"
    lti = True
    continuous = False
    OUT_SCALE = 1.0

    def __init__(self, d_model, d_state=None, discretization=None, *, asynchronous=False, dtype="f64", rng=None,
                 seed=0, r_min=0.9, r_max=0.999, max_phase=np.pi / 10, device=None):
        super().__init__(d_model, 64 if d_state is None else d_state, discretization, asynchronous, dtype, device)
        rng = rng if rng is not None else Rng(seed)
        r_mag, r_ph, r_b, r_c = rng.split(4)
        m, n, dt = self.d_model, self.d_state, self.rdt
        mag = np.asarray(r_mag.uniform(r_min, r_max, n), dt)
        phase = np.maximum(np.asarray(r_ph.uniform(0.0, max_phase, n), dt), 1e-9)
        self.nu_log = self._p(np.asarray(np.log(-np.log(mag)), dt))
        self.theta_log = self._p(np.asarray(np.log(phase), dt))
        self.gamma_log = self._p(np.asarray(0.5 * np.log(1.0 - mag.astype(np.float64) ** 2), dt))
        Br, Bi = _pair(r_b, (n, m), 1.0 / np.sqrt(m), dt)
        Cr, Ci = _pair(r_c, (m, n), 1.0 / np.sqrt(n), dt)
        self.B_re, self.B_im, self.C_re, self.C_im = map(self._p, (Br, Bi, Cr, Ci))
        self.D = self._p(np.ones(m, dt))

    _KIND_CODE = 1
    _coef_keys = ("nu_log", "theta_log", "gamma_log")

    @property
    def _P(self):
        return self.d_state

    def _coef_params(self):
        return self.nu_log, self.theta_log, self.gamma_log

    def parameters(self):
        return {"nu_log": self.nu_log, "theta_log": self.theta_log, "gamma_log": self.gamma_log,
                "B.re": self.B_re, "B.im": self.B_im, "C.re": self.C_re, "C.im": self.C_im, "D": self.D}

    def _abar_scale(self, deltas):
        # lambda in f64, then rounded to the layer dtype (layers.py:936-940)
        z = torch.complex(-torch.exp(self.nu_log.double()), torch.exp(self.theta_log.double()))
        lam64 = torch.exp(z)
        gamma = torch.exp(self.gamma_log)
        return lam64.to(self.tcdt), torch.complex(gamma, torch.zeros_like(gamma)), {"lam": lam64}

    def _coef_grads(self, ga, gsc, extra, deltas):
        cl = extra["lam"].conj() * ga.to(torch.complex128)
        return {"nu_log": -torch.exp(self.nu_log.double()) * cl.real,
                "theta_log": torch.exp(self.theta_log.double()) * cl.imag,
                "gamma_log": torch.exp(self.gamma_log.double()) * gsc.real.double()}


# ---------------------------------------------------------------------------
# S6


class S6(LinearRecurrence):
    """Selective SISO recurrence (layers.py:983-1168)."""

    kind = "s6"
    lti = False
    continuous = False
    bf16_ok = True

    def __init__(self, d_model, d_state=None, discretization=None, *, asynchronous=False, dtype="f64", rng=None,
                 seed=0, d_rank=None, device=None, seq_group=None):
        """`seq_group`: a torch.distributed process group (or "world") for
        sequence parallelism -- every rank passes its contiguous slice
        [B, L_r, d_model] of the sequence (in rank order) to forward; the state
        and cotangent carries cross ranks through distributed.LongS6, and
        layer_backward returns the complete parameter gradients (summed over
        the ranks in a fixed order) on every rank, the slice's grad u."""
        super().__init__(d_model, 64 if d_state is None else d_state, discretization, asynchronous, dtype, device)
        self.seq_group = seq_group
        self._long = None
        if seq_group is not None:
            if self.dtype == "f64" or self.d_state % 16 or d_model % (8 if self.dtype == "bf16" else 4):
                raise ValueError("seq_group needs the v3 kernels: f32 / bf16 I/O, d_state a multiple of 16 and "
                                 "d_model a multiple of 4 (f32) / 8 (bf16)")
            from .distributed import LongS6
            self._long = LongS6(None if seq_group == "world" else seq_group)
        rng = rng if rng is not None else Rng(seed)
        r_b, r_c, r_dn, r_up, r_dt = rng.split(5)
        m, n, dt = self.d_model, self.d_state, self.rdt
        self.d_rank = int(d_rank) if d_rank else max(1, -(-m // 16))
        r = self.d_rank
        self.a_log = self._p(np.broadcast_to(np.log(np.arange(1, n + 1, dtype=dt)), (m, n)))
        self.W_B = self._p(np.asarray(r_b.normal((n, m)) / np.sqrt(m), dt))
        self.W_C = self._p(np.asarray(r_c.normal((n, m)) / np.sqrt(m), dt))
        self.W_delta = self._p(np.asarray(r_dn.normal((m, r)) / np.sqrt(m), dt))
        self.W_delta_proj = self._p(np.asarray(r_up.normal((r, m)) / np.sqrt(r), dt))
        d0 = np.exp(r_dt.uniform(np.log(1e-3), np.log(1e-1), m))
        self.b_delta = self._p(np.asarray(np.log(np.expm1(d0)), dt))
        self.D = self._p(np.ones(m, dt))

    def parameters(self):
        return {"a_log": self.a_log, "W_B": self.W_B, "W_C": self.W_C, "W_delta": self.W_delta,
                "W_delta_proj": self.W_delta_proj, "b_delta": self.b_delta, "D": self.D}

    def _delta_in(self, p1):
        """The delta projection's softplus rides the tcgen05 GEMM epilogue when
        that GEMM runs on the tensor cores and the scan is a v3 kernel."""
        m = self.d_model
        v3 = self.d_state % 16 == 0 and (m % 8 == 0 if self.io_dtype == torch.bfloat16 else m % 4 == 0)
        return (v3 and self.tdt == torch.float32 and _tc_ok(p1, p1.shape[1], m)
                and os.environ.get("LRX_S6_DELTA_IN") != "0")

    def _wcat(self):
        """[W_delta^T; W_B; W_C] ([r + 2n, m]): the three input projections of
        layers.py:1020-1027 as ONE GEMM that reads u once."""
        return torch.cat((self.W_delta.T, self.W_B, self.W_C), 0).contiguous()

    def _forward(self, u, deltas, keep):
        B, L, m = u.shape
        n, r = self.d_state, self.d_rank
        u2 = u.reshape(B * L, m)
        P = _proj(u2, self._wcat())                                    # [T, r + 2n] fp32
        # own (aligned) storage for each part: the kernels' TMA maps need 16-byte bases
        p1 = P[:, :r].clone()
        Bk = P[:, r:r + n].clone().reshape(B, L, n)
        Ck = P[:, r + n:].clone().reshape(B, L, n)
        flags = 0
        if self._long is None and self._delta_in(p1):
            # delta = softplus(p1 W_delta_proj + b_delta) in the GEMM epilogue
            # (layers.py:1020-1027): the scan reads delta (LRX_S6_DELTA_IN)
            pre = ops.gemm_f32(p1, self.W_delta_proj.T.contiguous(), bias=self.b_delta,
                               act=ops.ACT_SOFTPLUS).reshape(B, L, m)
            flags = ops.S6_DELTA_IN
        else:
            pre = _proj(p1, self.W_delta_proj.T).reshape(B, L, m)
        if self._long is not None:  # sequence parallel: this rank's slice
            y, lctx = self._long.forward(u, pre, self.b_delta, self.a_log, Bk, Ck, self.D)
            saved = {"u": u, "p1": p1, "pre": pre, "Bk": Bk, "Ck": Ck, "ckpt": None, "lctx": lctx}
            cks = [c["ckpt"] for c in lctx.get("groups", [lctx])]
            return y, saved, torch.cat([c[:, -1] for c in cks], dim=-1)
        # inference (no tape, no returned state) skips the checkpoint stores
        y, ckpt = ops.s6_scan_fwd(u, pre, self.b_delta, self.a_log, Bk, Ck, self.D, ckpt=keep, flags=flags)
        if not keep:
            return y, {}, None
        saved = {"u": u, "p1": p1, "pre": pre, "Bk": Bk, "Ck": Ck, "ckpt": ckpt, "flags": flags}
        return y, saved, ckpt[:, -1]

    # -- step mode (layers.py:1120-1168) --------------------------------------
    def _zero_state(self, batch):
        return torch.zeros((batch, self.d_model, self.d_state), dtype=self.tdt, device=self.device)

    def _step(self, st, uk, delta_k):
        if self.tdt == torch.float32 and st.batch <= 16 and st.batch * self.d_model * 4 <= 190 * 1024 and \
                (st.batch * self.d_model * uk.element_size()) % 16 == 0:
            # projections + update in two kernels (fp32 weights read once per token)
            y = torch.empty((st.batch, self.d_model), dtype=self.io_dtype, device=self.device)
            ws = torch.empty((st.batch, self.d_rank + 2 * self.d_state), dtype=torch.float32, device=self.device)
            _lib.check(_lib.lib().lrx_s6_step_fused(
                _lib.code_of(self.io_dtype), _lib.ptr(st.x), _lib.ptr(uk), _lib.ptr(self.W_delta),
                _lib.ptr(self.W_delta_proj), _lib.ptr(self.W_B), _lib.ptr(self.W_C), _lib.ptr(self.b_delta),
                _lib.ptr(self.a_log), _lib.ptr(self.D), _lib.ptr(y), _lib.ptr(ws), st.batch, self.d_model,
                self.d_rank, self.d_state, _lib.stream()))
            return y
        p1 = _mm(uk, self.W_delta)
        pre = (p1 @ self.W_delta_proj).contiguous()
        Bk = _mm(uk, self.W_B.T).contiguous()
        Ck = _mm(uk, self.W_C.T).contiguous()
        y = torch.empty((st.batch, self.d_model), dtype=self.io_dtype, device=self.device)
        _lib.check(_lib.lib().lrx_s6_step(
            _lib.code_of(self.io_dtype), _lib.ptr(st.x), _lib.ptr(uk), _lib.ptr(pre), _lib.ptr(Bk), _lib.ptr(Ck),
            _lib.ptr(self.b_delta), _lib.ptr(self.a_log), _lib.ptr(self.D), _lib.ptr(y), st.batch, self.d_model,
            self.d_state, _lib.stream()))
        return y

    def _backward(self, s, gy):
        u, p1, pre, Bk, Ck, ckpt, host = (s[k] for k in ("u", "p1", "pre", "Bk", "Ck", "ckpt", "host"))
        B, L, m = u.shape
        n = self.d_state
        gy = self._gy(gy, u.shape)
        lctx = s.get("lctx")
        if lctx is not None:
            r = self._long.backward(lctx, u, pre, self.b_delta, self.a_log, Bk, Ck, self.D, gy, reduce=False)
        else:
            r = ops.s6_scan_bwd(u, pre, self.b_delta, self.a_log, Bk, Ck, self.D, ckpt, gy, flags=s.get("flags", 0))
        # projection GEMMs (layers.py:1100-1112), compute precision; the three
        # input projections share one GEMM each way: G = [gp1 | gB_k | gC_k]
        c = self.tdt
        rk = self.d_rank
        u2 = ops.cast(u.reshape(B * L, m), c)
        gpre2 = r["gpre"].reshape(B * L, m)
        gp1 = _proj(gpre2, self.W_delta_proj)
        G = torch.cat((gp1, r["gBk"].reshape(B * L, n).to(c), r["gCk"].reshape(B * L, n).to(c)), 1)
        gu = ops.cast(r["gu_local"].reshape(B * L, m), c)
        gu = _proj_acc(gu, G, self._wcat().T)                          # gu += G [W_delta^T; W_B; W_C]
        gW = _wgrad(G, u2)                                             # [r + 2n, m]
        grads = {"a_log": r["ga_log"], "W_B": gW[rk:rk + n].contiguous(), "W_C": gW[rk + n:].contiguous(),
                 "W_delta": gW[:rk].T.contiguous(), "W_delta_proj": _wgrad(p1.to(c), gpre2),
                 "b_delta": r["gb_delta"], "D": r["gD"]}
        if lctx is not None:  # every gradient is a sum over the whole sequence: one fixed-order reduction
            from .distributed import reduce_fixed_order
            grads = dict(zip(grads, reduce_fixed_order(list(grads.values()), self._long.group)))
        return self._out(grads, ops.cast(gu, self.io_dtype).reshape(B, L, m), host)


# ---------------------------------------------------------------------------
# RG-LRU


class RGLRU(LinearRecurrence):
    """Gated real recurrence of width d_model, y = x (layers.py:1171-1336)."""

    kind = "rglru"
    lti = False
    continuous = False
    bf16_ok = True
    GATE_POWER = 8.0

    def __init__(self, d_model, d_state=None, discretization=None, *, asynchronous=False, dtype="f64", rng=None,
                 seed=0, a_min=0.9, a_max=0.999, device=None):
        if d_state is not None and d_state != d_model:
            warnings.warn(f"rglru's recurrence width is structurally d_model={d_model}; d_state={d_state} is ignored")
        super().__init__(d_model, d_model, discretization, asynchronous, dtype, device)
        rng = rng if rng is not None else Rng(seed)
        r_a, r_r, r_i = rng.split(3)
        m, dt = self.d_model, self.rdt
        a0 = np.asarray(r_a.uniform(a_min, a_max, m), np.float64)
        self.lambda_param = self._p(np.asarray(np.log(a0) - np.log1p(-a0), dt))
        self.W_r = self._p(np.asarray(r_r.normal((m, m)) / np.sqrt(m), dt))
        self.b_r = self._p(np.zeros(m, dt))
        self.W_i = self._p(np.asarray(r_i.normal((m, m)) / np.sqrt(m), dt))
        self.b_i = self._p(np.zeros(m, dt))

    def parameters(self):
        return {"lambda_param": self.lambda_param, "W_r": self.W_r, "b_r": self.b_r, "W_i": self.W_i,
                "b_i": self.b_i}

    def _forward(self, u, deltas, keep):
        B, L, W = u.shape
        u2 = u.reshape(B * L, W)
        qr = _proj(u2, self._w(self.W_r), _mm_io).reshape(B, L, W)
        qi = _proj(u2, self._w(self.W_i), _mm_io).reshape(B, L, W)
        y, ckpt = ops.rglru_scan_fwd(u, qr, qi, self.lambda_param, self.b_r, self.b_i)
        saved = {"u": u, "qr": qr, "qi": qi, "ckpt": ckpt, "y": y} if keep else {}
        return y, saved, y[:, -1].to(self.tdt)

    # -- step mode (layers.py:1293-1336) --------------------------------------
    def _zero_state(self, batch):
        return torch.zeros((batch, self.d_model), dtype=self.tdt, device=self.device)

    def _step(self, st, uk, delta_k):
        if self.tdt == torch.float32 and st.batch <= 16 and self.d_model % 8 == 0 and \
                st.batch * self.d_model * 4 <= 190 * 1024:
            # gate GEMVs + update in one kernel (fp32 weights read once per token)
            y = torch.empty((st.batch, self.d_model), dtype=self.io_dtype, device=self.device)
            _lib.check(_lib.lib().lrx_rglru_step_fused(
                _lib.code_of(self.io_dtype), _lib.ptr(st.x), _lib.ptr(uk), _lib.ptr(self.W_r), _lib.ptr(self.W_i),
                _lib.ptr(self.lambda_param), _lib.ptr(self.b_r), _lib.ptr(self.b_i), _lib.ptr(y), st.batch,
                self.d_model, _lib.stream()))
            return y
        qr = (uk @ self._w(self.W_r).T).contiguous()
        qi = (uk @ self._w(self.W_i).T).contiguous()
        y = torch.empty((st.batch, self.d_model), dtype=self.io_dtype, device=self.device)
        _lib.check(_lib.lib().lrx_rglru_step(
            _lib.code_of(self.io_dtype), _lib.ptr(st.x), _lib.ptr(uk), _lib.ptr(qr), _lib.ptr(qi),
            _lib.ptr(self.lambda_param), _lib.ptr(self.b_r), _lib.ptr(self.b_i), _lib.ptr(y), st.batch,
            self.d_model, _lib.stream()))
        return y

    def _backward(self, s, gy):
        u, qr, qi, ckpt, host = s["u"], s["qr"], s["qi"], s["ckpt"], s["host"]
        B, L, W = u.shape
        gy = self._gy(gy, u.shape)
        r = ops.rglru_scan_bwd(u, qr, qi, self.lambda_param, self.b_r, self.b_i, ckpt, gy, y=s["y"])
        c = self.tdt
        u2 = ops.cast(u.reshape(B * L, W), c)
        gqr2, gqi2 = ops.cast(r["gqr"].reshape(B * L, W), c), ops.cast(r["gqi"].reshape(B * L, W), c)
        gu = _proj_acc(ops.cast(r["gu_local"].reshape(B * L, W), c), gqr2, self.W_r.T)
        gu = _proj_acc(gu, gqi2, self.W_i.T)
        grads = {"lambda_param": sigmoid(-self.lambda_param) * r["gla"], "W_r": _wgrad(gqr2, u2), "b_r": r["gb_r"],
                 "W_i": _wgrad(gqi2, u2), "b_i": r["gb_i"]}
        return self._out(grads, ops.cast(gu, self.io_dtype).reshape(B, L, W), host)


# ---------------------------------------------------------------------------
# registry (layers.py:1343-1383)

_REGISTRY = {"s4d": S4D, "s5": S5, "lru": LRU, "s6": S6, "rglru": RGLRU}


def make_layer(kind, d_model, d_state=None, discretization=None, *, asynchronous=False, dtype="f64", rng=None,
               seed=0, **extras):
    try:
        cls = _REGISTRY[kind]
    except KeyError:
        raise UnknownLayer(f"unknown layer kind {kind!r}; registered kinds: {sorted(_REGISTRY)}") from None
    return cls(d_model, d_state=d_state, discretization=discretization, asynchronous=asynchronous, dtype=dtype,
               rng=rng, seed=seed, **extras)


def init_layer(kind, cfg: LayerConfig, rng: Rng):
    return make_layer(kind, cfg.d_model, d_state=cfg.d_state, discretization=cfg.discretization,
                      asynchronous=cfg.asynchronous, dtype=cfg.dtype, rng=rng, **cfg.extras)


def lti_forward(layer, u, mode="sequential", *, workers=1, deltas=None, **kw):
    if not layer.lti:
        raise ValueError(f"{layer.kind} is time-varying; use ltv_forward")
    return layer.forward(u, mode, workers=workers, deltas=deltas, **kw)


def ltv_forward(layer, u, mode="sequential", *, workers=1, **kw):
    if layer.lti:
        raise ValueError(f"{layer.kind} is time-invariant; use lti_forward")
    return layer.forward(u, mode, workers=workers, **kw)


def layer_step(layer, state, u_k, delta_k=None):
    return layer.step(state, u_k, delta_k)
