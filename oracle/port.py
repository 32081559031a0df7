"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

A CPU restatement of the reference's diagonal-recurrence hot path:

  * numerics: Philox `Rng`, overflow-safe softplus/sigmoid
      (pkg/src/linrec/numerics.py:36-39, 86-105, 180-204)
  * discretization factors and their partials
      (discretize.py:39-44, 59-93, 136-142; autograd.py:186-211)
  * the scan operator: `_prepare`, sequential scan, the three-phase chunked
      parallel scan over a thread pool, `plan_chunks`
      (scan.py:44, 62-75, 87-201) — the inner loops are the plain-C
      restatement in oracle/scan_loops.c (of _scan_kernels.py:17-153)
  * the reverse-mode scan pullback (autograd.py:113-179)
  * parameter initialisation, taped forward and analytic backward of the five
      layer kinds s4d / s5 / lru / s6 / rglru (layers.py:352-1336)

The reference is CPU-only numpy+numba; this module keeps its arithmetic (same
formulas, same operation order where it matters for rounding) but is laid out
as plain functions over a parameter dict instead of the reference's class
hierarchy.  It runs in float64 (the ground truth used by the parity tests) or
float32 (the reference's f32 path, for the CPU-baseline timing).
"""
from __future__ import annotations

import ctypes
import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

# ---------------------------------------------------------------------------
# numerics (numerics.py)

SOFTPLUS_THRESHOLD = {np.dtype(np.float32): 30.0, np.dtype(np.float64): 50.0}  # numerics.py:36-39
ZOH_SMALL_POLE_EPS = {np.dtype(np.float64): 1e-8, np.dtype(np.float32): 1e-4}  # discretize.py:39-42
BILINEAR_SINGULAR_TOL = 1e-6                                                   # discretize.py:44
MIN_CHUNK_LEN = 256                                                            # scan.py:44
GATE_POWER = 8.0                                                               # layers.py:1177


class ShapeError(ValueError):
    pass


class SingularBilinear(ValueError):
    pass


def rdtype(spec):
    return {"f32": np.dtype(np.float32), "f64": np.dtype(np.float64)}[spec]


def cdtype(spec):
    return {"f32": np.dtype(np.complex64), "f64": np.dtype(np.complex128)}[spec]


def _real_of(dt):
    dt = np.dtype(dt)
    return {np.dtype(np.complex64): np.dtype(np.float32),
            np.dtype(np.complex128): np.dtype(np.float64)}.get(dt, dt)


def softplus(x):
    """log1p(exp(min(x,t))) with identity above t (numerics.py:86-94)."""
    x = np.asarray(x)
    if x.dtype not in SOFTPLUS_THRESHOLD:
        x = x.astype(np.float64)
    t = SOFTPLUS_THRESHOLD[x.dtype]
    return np.where(x > t, x, np.log1p(np.exp(np.minimum(x, t))))


def sigmoid(x):
    """Branch-free stable logistic (numerics.py:97-105)."""
    x = np.asarray(x)
    if x.dtype not in SOFTPLUS_THRESHOLD:
        x = x.astype(np.float64)
    pos = x >= 0
    e = np.exp(np.where(pos, -x, x))
    return np.where(pos, 1.0 / (1.0 + e), e / (1.0 + e))


class Rng:
    """Philox generator over a SeedSequence, split by spawn (numerics.py:180-204)."""

    def __init__(self, seed=0, _seq=None):
        self._seq = np.random.SeedSequence(seed) if _seq is None else _seq
        self._gen = np.random.Generator(np.random.Philox(self._seq))

    def normal(self, shape=(), dtype="f64"):
        return self._gen.standard_normal(shape, dtype=rdtype(dtype))

    def uniform(self, low=0.0, high=1.0, shape=(), dtype="f64"):
        out = self._gen.uniform(low, high, shape)
        if np.ndim(out) == 0:
            return np.asarray(out, dtype=rdtype(dtype))[()]
        return out.astype(rdtype(dtype), copy=False)

    def split(self, n):
        return [Rng(_seq=s) for s in self._seq.spawn(n)]


# ---------------------------------------------------------------------------
# discretization (discretize.py:59-142) and partials (autograd.py:186-211)

def scheme_factors(scheme, a, delta):
    a = np.asarray(a)
    delta = np.asarray(delta)
    if scheme == "zoh":
        abar = np.exp(delta * a)
        small = np.abs(a) < ZOH_SMALL_POLE_EPS[_real_of(a.dtype)]
        a_safe = np.where(small, np.ones_like(a), a)
        scale = np.where(small, delta * np.ones_like(abar), (abar - 1.0) / a_safe)
        return abar, scale
    if scheme == "bilinear":
        half = 0.5 * delta * a
        den = 1.0 - half
        if np.any(np.abs(den) <= BILINEAR_SINGULAR_TOL * (1.0 + np.abs(half))):
            raise SingularBilinear("bilinear transform singular")
        return (1.0 + half) / den, delta / den
    if scheme == "dirac":
        abar = np.exp(delta * a)
        return abar, np.ones_like(abar)
    raise ValueError(f"unknown discretization scheme {scheme!r}")


def scheme_partials(scheme, lam, delta, abar, scale):
    """(dabar/dlam, dabar/ddelta, dscale/dlam, dscale/ddelta)."""
    if scheme == "zoh":
        eps = ZOH_SMALL_POLE_EPS[_real_of(np.asarray(lam).dtype)]
        small = np.abs(lam) < eps
        lam_safe = np.where(small, 1.0, lam)
        dsl = np.where(small, delta * delta / 2.0,
                       (delta * abar * lam - (abar - 1.0)) / (lam_safe * lam_safe))
        return delta * abar, lam * abar, dsl, np.where(small, np.ones_like(abar), abar)
    if scheme == "bilinear":
        den = 1.0 - 0.5 * delta * lam
        den2 = den * den
        return delta / den2, lam / den2, delta * delta / (2.0 * den2), 1.0 / den2
    if scheme == "dirac":
        z = np.zeros_like(abar)
        return delta * abar, lam * abar, z, z
    raise ValueError(f"unknown discretization scheme {scheme!r}")


# ---------------------------------------------------------------------------
# native loops (oracle/scan_loops.c, restating _scan_kernels.py)

_SUFFIX = {np.dtype(np.float32): "f32", np.dtype(np.float64): "f64",
           np.dtype(np.complex64): "c64", np.dtype(np.complex128): "c128"}
_lib = None
_lib_lock = threading.Lock()


def loops_path():
    return os.path.join(_HERE, "_build", "liboracle_loops.so")


def build_loops(force=False):
    """Compile scan_loops.c with gcc (strict IEEE, no contraction)."""
    out = loops_path()
    src = os.path.join(_HERE, "scan_loops.c")
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    import subprocess
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11",
                           "-fno-fast-math", "-ffp-contract=off", "-fcx-limited-range",
                           src, "-o", out])
    return out


def _loops():
    global _lib
    with _lib_lock:
        if _lib is None:
            path = loops_path()
            if not os.path.exists(path):
                build_loops()
            _lib = ctypes.CDLL(path)
        return _lib


def _call(name, dt, *arrays_then_dims):
    fn = getattr(_loops(), f"{name}_{_SUFFIX[np.dtype(dt)]}")
    args = []
    for v in arrays_then_dims:
        if isinstance(v, np.ndarray):
            assert v.flags.c_contiguous and v.dtype == dt, (name, v.dtype, dt)
            args.append(ctypes.c_void_p(v.ctypes.data))
        else:
            args.append(ctypes.c_int64(int(v)))
    fn(*args)


# ---------------------------------------------------------------------------
# scan operator (scan.py)

_pools = {}
_pools_lock = threading.Lock()


def _pool(workers):
    with _pools_lock:
        p = _pools.get(workers)
        if p is None:
            p = _pools[workers] = ThreadPoolExecutor(max_workers=workers)
        return p


def combine(first, second):
    """(a1,b1) then (a2,b2) -> (a2 a1, a2 b1 + b2)  (scan.py:62-75)."""
    a1, b1 = map(np.asarray, first)
    a2, b2 = map(np.asarray, second)
    if not (a1.shape == b1.shape == a2.shape == b2.shape):
        raise ShapeError("combine operands must share a shape")
    return a2 * a1, a2 * b1 + b2


def plan_chunks(length, workers):
    """(scan.py:139-149)"""
    if length < 1:
        raise ValueError("length must be >= 1")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    size = max(MIN_CHUNK_LEN, -(-length // workers))
    return [(s, min(s + size, length)) for s in range(0, length, size)]


def prepare(a, b, x0):
    """Normalise to time-major [L, N] of one dtype (scan.py:87-124)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if b.ndim < 1 or b.shape[0] < 1:
        raise ShapeError("b must be [length, *lanes] with length >= 1")
    lanes = b.shape[1:]
    if a.ndim == b.ndim:
        if a.shape != b.shape:
            raise ShapeError("per-step a must match b")
        per_step = True
    elif a.ndim == b.ndim - 1:
        if a.shape != lanes:
            raise ShapeError("constant a must match b's lane shape")
        per_step = False
    else:
        raise ShapeError("a must be [*lanes] or [length, *lanes]")
    parts = [a, b] if x0 is None else [a, b, np.asarray(x0)]
    dt = np.result_type(*parts)
    if dt not in _SUFFIX:
        dt = np.result_type(dt, np.float64)
    L = b.shape[0]
    N = int(np.prod(lanes, dtype=np.int64)) if lanes else 1
    b2 = np.ascontiguousarray(b, dtype=dt).reshape(L, N)
    a2 = np.ascontiguousarray(a, dtype=dt).reshape((L, N) if per_step else (N,))
    if x0 is None:
        x02 = np.zeros(N, dt)
    else:
        x02 = np.asarray(x0)
        if x02.shape != lanes:
            raise ShapeError("x0 must have the lane shape")
        x02 = np.ascontiguousarray(x02, dtype=dt).reshape(N)
    return a2, per_step, b2, x02, dt, lanes


def _seq2(a2, per_step, b2, x02):
    out = np.empty_like(b2)
    L, N = b2.shape
    _call("scan_var" if per_step else "scan_const", b2.dtype, a2, b2, x02, out, L, N)
    return out


def _par2(a2, per_step, b2, x02, workers):
    L, N = b2.shape
    dt = b2.dtype
    chunks = plan_chunks(L, workers)
    if len(chunks) == 1:
        return _seq2(a2, per_step, b2, x02)
    out = np.empty_like(b2)
    C = len(chunks)
    prods = np.empty((C, N), dt)
    pool = _pool(workers)

    def phase1(c):  # scan.py:175-182
        s, e = chunks[c]
        aa = np.ascontiguousarray(a2[s:e]) if per_step else a2
        o = np.empty((e - s, N), dt)
        _call("local_scan_var" if per_step else "local_scan_const", dt,
              aa, np.ascontiguousarray(b2[s:e]), o, prods[c], e - s, N)
        out[s:e] = o

    list(pool.map(phase1, range(C)))
    entering = np.empty((C, N), dt)
    entering[0] = x02
    for c in range(1, C):  # scan.py:184-189
        entering[c] = prods[c - 1] * entering[c - 1] + out[chunks[c - 1][1] - 1]

    def phase3(c):  # scan.py:191-200
        s, e = chunks[c]
        if not entering[c].any():
            return
        aa = np.ascontiguousarray(a2[s:e]) if per_step else a2
        o = np.ascontiguousarray(out[s:e])
        _call("fixup_var" if per_step else "fixup_const", dt,
              aa, np.ascontiguousarray(entering[c]), o, e - s, N)
        out[s:e] = o

    list(pool.map(phase3, range(C)))
    return out


def scan_sequential(a, b, x0=None):
    a2, per_step, b2, x02, dt, lanes = prepare(a, b, x0)
    return _seq2(a2, per_step, b2, x02).reshape(b2.shape[0], *lanes)


def scan_parallel(a, b, x0=None, workers=1):
    a2, per_step, b2, x02, dt, lanes = prepare(a, b, x0)
    return _par2(a2, per_step, b2, x02, workers).reshape(b2.shape[0], *lanes)


def _run(mode, workers, a2, per_step, b2):
    x0 = np.zeros(b2.shape[1], b2.dtype)
    if mode == "parallel":
        return _par2(a2, per_step, b2, x0, workers)
    return _seq2(a2, per_step, b2, x0)


def pullback(a2, per_step, x2, x02, gx2):
    """Reverse recurrence with conj(a) (autograd.py:113-140)."""
    L, N = gx2.shape
    dt = gx2.dtype
    g = np.empty_like(gx2)
    ac = np.ascontiguousarray(np.conj(a2), dtype=dt)
    _call("backward_var" if per_step else "backward_const", dt, ac,
          np.ascontiguousarray(gx2), g, L, N)
    xprev = np.empty_like(x2)
    xprev[0] = 0 if x02 is None else x02
    xprev[1:] = x2[:-1]
    xprev = np.conj(xprev)
    if per_step:
        return g, g * xprev, np.conj(a2[0]) * g[0]
    return g, np.einsum("ln,ln->n", g, xprev, optimize=True), np.conj(a2) * g[0]


def scan_backward(a, states, x0, grad_states):
    """(grad_a, grad_b, grad_x0) of a recorded scan (autograd.py:143-179)."""
    a = np.asarray(a)
    gx = np.asarray(grad_states)
    if gx.shape != states.shape:
        raise ShapeError("grad_states shape does not match states")
    L = states.shape[0]
    lanes = states.shape[1:]
    per_step = a.ndim == states.ndim
    a2 = np.ascontiguousarray(a.reshape(L, -1) if per_step
                              else np.broadcast_to(a, lanes).reshape(-1), dtype=states.dtype)
    x02 = None if x0 is None else np.broadcast_to(np.asarray(x0, states.dtype), lanes).reshape(-1)
    g, ga, gx0 = pullback(a2, per_step, states.reshape(L, -1), x02,
                          np.ascontiguousarray(gx.reshape(L, -1), dtype=states.dtype))
    grad_a = ga.reshape(states.shape) if per_step else ga.reshape(lanes)
    if not per_step and a.shape != lanes:
        keep = tuple(range(len(lanes) - a.ndim))
        grad_a = grad_a.sum(axis=keep) if keep else grad_a
    return grad_a, g.reshape(states.shape), gx0.reshape(lanes)


# ---------------------------------------------------------------------------
# layers: parameter initialisation (layers.py:325-1196)

def _tm(x):
    """[B, L, ...] -> contiguous time-major [L, B*...] (layers.py:115-118)."""
    xt = np.ascontiguousarray(np.moveaxis(x, 1, 0))
    return xt.reshape(xt.shape[0], -1)


def _lanes(arr, B):
    return np.tile(arr.reshape(-1), B)


def _pair(rng, shape, std, dt):
    g = rng.split(2)
    return np.asarray(g[0].normal(shape) * std, dt), np.asarray(g[1].normal(shape) * std, dt)


def default_scheme(kind, asynchronous=False):
    if kind in ("s4d", "s5"):
        return "dirac" if asynchronous else "zoh"
    return None


def init_params(kind, d_model, d_state=None, *, dtype="f64", seed=0, **extras):
    """Parameters of make_layer(kind, d_model, d_state, dtype=dtype, seed=seed)."""
    dt = rdtype(dtype)
    rng = Rng(seed)
    m = int(d_model)
    if kind == "s4d":  # layers.py:358-372
        n = 64 if d_state is None else int(d_state)
        r_b, r_c, r_d = rng.split(3)
        br, bi = _pair(r_b, (m, n), 1.0, dt)
        cr, ci = _pair(r_c, (m, n), 1.0 / np.sqrt(n), dt)
        return {"lambda_re_log": np.full((m, n), np.log(0.5), dt),
                "lambda_im": np.broadcast_to(np.pi * np.arange(n, dtype=dt), (m, n)).copy(),
                "b.re": br, "b.im": bi, "c.re": cr, "c.im": ci,
                "d": np.ones(m, dt),
                "log_delta": np.asarray(r_d.uniform(np.log(1e-3), np.log(1e-1), m), dt)}
    if kind == "s5":  # layers.py:794-813
        ds = 64 if d_state is None else int(d_state)
        if ds % 2:
            raise ValueError("s5 needs even d_state")
        P = ds // 2
        r_b, r_c, r_d = rng.split(3)
        Br, Bi = _pair(r_b, (P, m), 1.0 / np.sqrt(m), dt)
        Cr, Ci = _pair(r_c, (m, P), 1.0 / np.sqrt(P), dt)
        return {"lambda_re_log": np.full((P,), np.log(0.5), dt),
                "lambda_im": np.pi * np.arange(P, dtype=dt),
                "B.re": Br, "B.im": Bi, "C.re": Cr, "C.im": Ci,
                "D": np.ones(m, dt),
                "log_delta": np.asarray(r_d.uniform(np.log(1e-3), np.log(1e-1), P), dt)}
    if kind == "lru":  # layers.py:904-934
        n = 64 if d_state is None else int(d_state)
        r_min = extras.get("r_min", 0.9)
        r_max = extras.get("r_max", 0.999)
        max_phase = extras.get("max_phase", np.pi / 10)
        r_mag, r_ph, r_b, r_c = rng.split(4)
        mag = np.asarray(r_mag.uniform(r_min, r_max, n), dt)
        phase = np.maximum(np.asarray(r_ph.uniform(0.0, max_phase, n), dt), 1e-9)
        Br, Bi = _pair(r_b, (n, m), 1.0 / np.sqrt(m), dt)
        Cr, Ci = _pair(r_c, (m, n), 1.0 / np.sqrt(n), dt)
        return {"nu_log": np.asarray(np.log(-np.log(mag)), dt),
                "theta_log": np.asarray(np.log(phase), dt),
                "gamma_log": np.asarray(0.5 * np.log(1.0 - mag.astype(np.float64) ** 2), dt),
                "B.re": Br, "B.im": Bi, "C.re": Cr, "C.im": Ci, "D": np.ones(m, dt)}
    if kind == "s6":  # layers.py:990-1015
        n = 64 if d_state is None else int(d_state)
        r_b, r_c, r_dn, r_up, r_dt = rng.split(5)
        r = int(extras["d_rank"]) if extras.get("d_rank") else max(1, -(-m // 16))
        d0 = np.exp(r_dt.uniform(np.log(1e-3), np.log(1e-1), m))
        return {"a_log": np.broadcast_to(np.log(np.arange(1, n + 1, dtype=dt)), (m, n)).copy(),
                "W_B": np.asarray(r_b.normal((n, m)) / np.sqrt(m), dt),
                "W_C": np.asarray(r_c.normal((n, m)) / np.sqrt(m), dt),
                "W_delta": np.asarray(r_dn.normal((m, r)) / np.sqrt(m), dt),
                "W_delta_proj": np.asarray(r_up.normal((r, m)) / np.sqrt(r), dt),
                "b_delta": np.asarray(np.log(np.expm1(d0)), dt),
                "D": np.ones(m, dt)}
    if kind == "rglru":  # layers.py:1179-1203
        a_min = extras.get("a_min", 0.9)
        a_max = extras.get("a_max", 0.999)
        r_a, r_r, r_i = rng.split(3)
        a0 = np.asarray(r_a.uniform(a_min, a_max, m), np.float64)
        return {"lambda_param": np.asarray(np.log(a0) - np.log1p(-a0), dt),
                "W_r": np.asarray(r_r.normal((m, m)) / np.sqrt(m), dt),
                "b_r": np.zeros(m, dt),
                "W_i": np.asarray(r_i.normal((m, m)) / np.sqrt(m), dt),
                "b_i": np.zeros(m, dt)}
    raise ValueError(f"unknown layer kind {kind!r}")


# ---------------------------------------------------------------------------
# layers: taped forward + analytic backward

def _complex(re, im):
    z = np.empty(re.shape, {np.dtype(np.float32): np.complex64,
                           np.dtype(np.float64): np.complex128}[re.dtype])
    z.real, z.imag = re, im
    return z


class Layer:
    """Functional view of one reference layer: params dict + kind + scheme."""

    def __init__(self, kind, params, scheme=None, asynchronous=False):
        self.kind = kind
        self.p = params
        self.rdt = next(iter(params.values())).dtype
        self.cdt = np.dtype(np.complex64) if self.rdt == np.float32 else np.dtype(np.complex128)
        self.scheme = scheme if scheme is not None else default_scheme(kind, asynchronous)

    # -- LTI coefficient assembly ------------------------------------------
    def _lam_s(self):  # S4D/S5 lambda = -exp(re_log) + i im (layers.py:382-386, 823-827)
        lam = np.empty(self.p["lambda_re_log"].shape, self.cdt)
        lam.real = -np.exp(self.p["lambda_re_log"])
        lam.imag = self.p["lambda_im"]
        return lam

    def _lru_lambda(self):  # f64 then rounded (layers.py:936-940)
        z = -np.exp(self.p["nu_log"].astype(np.float64)) + 1j * np.exp(self.p["theta_log"].astype(np.float64))
        lam = np.empty(z.shape, self.cdt)
        lam[...] = np.exp(z)
        return lam

    # -- forward --------------------------------------------------------------
    def forward(self, u, mode="sequential", workers=1, deltas=None):
        u = np.ascontiguousarray(u, self.rdt)
        B, L, m = u.shape
        k = self.kind
        if deltas is not None:
            d = np.asarray(deltas, self.rdt)
            deltas = np.broadcast_to(d[None, :], (B, L)) if d.ndim == 1 else d
        if k == "s4d":
            return self._fwd_s4d(u, mode, workers, deltas)
        if k in ("s5", "lru"):
            return self._fwd_mimo(u, mode, workers, deltas)
        if k == "s6":
            return self._fwd_s6(u, mode, workers)
        if k == "rglru":
            return self._fwd_rglru(u, mode, workers)
        raise ValueError(k)

    def _fwd_s4d(self, u, mode, workers, deltas):  # layers.py:453-473
        B, L, m = u.shape
        p = self.p
        n = p["b.re"].shape[1]
        lam = self._lam_s()
        delta = np.exp(p["log_delta"])
        b = _complex(p["b.re"], p["b.im"])
        if deltas is None:
            abar, scale = scheme_factors(self.scheme, lam, delta[:, None])
            abar, scale = np.asarray(abar, self.cdt), np.asarray(scale, self.cdt)
            w = (scale * b) * u[..., None]
            a2, per = _lanes(abar, B), False
        else:
            deff = (deltas * 1.0)[:, :, None] * delta
            abar_k, sc_k = scheme_factors(self.scheme, lam, deff[..., None])
            w = (np.asarray(sc_k, self.cdt) * b) * u[..., None]
            a2, per = _tm(np.asarray(abar_k, self.cdt)), True
        xt = _run(mode, workers, np.ascontiguousarray(a2, self.cdt), per, _tm(w).astype(self.cdt))
        xt = xt.reshape(L, B, m, n)
        c = _complex(p["c.re"], p["c.im"])
        y = np.einsum("lbhn,hn->blh", xt, c, optimize=True).real + p["d"] * u
        return np.ascontiguousarray(y, self.rdt), {"u": u, "xt": xt, "deltas": deltas}

    def _mimo(self):
        p = self.p
        Bm = _complex(p["B.re"], p["B.im"])
        Cm = _complex(p["C.re"], p["C.im"])
        if self.kind == "lru":
            return Bm, Cm, 1.0, self._lru_lambda(), np.exp(p["gamma_log"]), None, None
        lam = self._lam_s()
        delta = np.exp(p["log_delta"])
        abar, scale = scheme_factors(self.scheme, lam, delta)
        return Bm, Cm, 2.0, np.asarray(abar, self.cdt), np.asarray(scale, self.cdt), lam, delta

    def _fwd_mimo(self, u, mode, workers, deltas):  # layers.py:666-686
        B, L, m = u.shape
        Bm, Cm, osc, abar, scale, lam, delta = self._mimo()
        bu = u @ Bm.T
        if deltas is None:
            v = np.asarray(scale) * bu
            a2, per = _lanes(abar, B), False
        else:
            deff = deltas[:, :, None] * delta
            abar_k, sc_k = scheme_factors(self.scheme, lam, deff)
            v = np.asarray(sc_k, self.cdt) * bu
            a2, per = _tm(np.asarray(abar_k, self.cdt)), True
        xt = _run(mode, workers, np.ascontiguousarray(a2, self.cdt), per, _tm(v).astype(self.cdt))
        P = Bm.shape[0]
        xt = xt.reshape(L, B, P)
        y = osc * np.einsum("lbp,hp->blh", xt, Cm, optimize=True).real + self.p["D"] * u
        return np.ascontiguousarray(y, self.rdt), {"u": u, "xt": xt, "bu": bu, "deltas": deltas}

    def _s6_proj(self, u):  # layers.py:1020-1027
        p = self.p
        p1 = u @ p["W_delta"]
        pre = p1 @ p["W_delta_proj"] + p["b_delta"]
        return softplus(pre), u @ p["W_B"].T, u @ p["W_C"].T, p1, pre

    def _fwd_s6(self, u, mode, workers):  # layers.py:1051-1066
        B, L, m = u.shape
        p = self.p
        n = p["W_B"].shape[0]
        a = -np.exp(p["a_log"])
        delta, bk, ck, p1, pre = self._s6_proj(u)
        abar = np.exp(delta[..., None] * a)
        w = (delta * u)[..., None] * bk[:, :, None, :]
        xt = _run(mode, workers, _tm(abar), True, _tm(w)).reshape(L, B, m, n)
        y = np.einsum("lbhn,bln->blh", xt, ck, optimize=True) + p["D"] * u
        return np.ascontiguousarray(y, self.rdt), dict(u=u, xt=xt, delta=delta, bk=bk, ck=ck, p1=p1, pre=pre)

    def _rg_gates(self, u):  # layers.py:1208-1218
        p = self.p
        r = sigmoid(u @ p["W_r"].T + p["b_r"])
        ig = sigmoid(u @ p["W_i"].T + p["b_i"])
        loga = GATE_POWER * r * (-softplus(-p["lambda_param"]))
        return r, ig, np.exp(loga), np.sqrt(-np.expm1(2.0 * loga))

    def _fwd_rglru(self, u, mode, workers):  # layers.py:1239-1250
        B, L, m = u.shape
        r, ig, ak, s = self._rg_gates(u)
        xt = _run(mode, workers, _tm(ak), True, _tm(s * ig * u)).reshape(L, B, m)
        y = np.ascontiguousarray(np.moveaxis(xt, 0, 1), self.rdt)
        return y, dict(u=u, xt=xt, r=r, ig=ig, ak=ak, s=s)

    # -- backward -------------------------------------------------------------
    def backward(self, saved, gy):
        gy = np.asarray(gy, self.rdt)
        k = self.kind
        if k == "s4d":
            return self._bwd_s4d(saved, gy)
        if k in ("s5", "lru"):
            return self._bwd_mimo(saved, gy)
        if k == "s6":
            return self._bwd_s6(saved, gy)
        return self._bwd_rglru(saved, gy)

    def _bwd_s4d(self, s, gy):  # layers.py:477-546
        u, xt, deltas = s["u"], s["xt"], s["deltas"]
        p = self.p
        B, L, m = u.shape
        n = p["b.re"].shape[1]
        lam = self._lam_s()
        delta = np.exp(p["log_delta"])
        b = _complex(p["b.re"], p["b.im"])
        c = _complex(p["c.re"], p["c.im"])
        gd = np.einsum("blh,blh->h", gy, u, optimize=True)
        gu = gy * p["d"]
        gyt = np.moveaxis(gy, 1, 0)
        gc = np.einsum("lbh,lbhn->hn", gyt, np.conj(xt), optimize=True)
        gxt = gyt[..., None] * np.conj(c)
        per = deltas is not None
        if per:
            deff = deltas[:, :, None] * delta
            abar_k, sc_k = scheme_factors(self.scheme, lam, deff[..., None])
            abar_k, sc_k = np.asarray(abar_k, self.cdt), np.asarray(sc_k, self.cdt)
            a2 = _tm(abar_k)
        else:
            abar, scale = scheme_factors(self.scheme, lam, delta[:, None])
            abar, scale = np.asarray(abar, self.cdt), np.asarray(scale, self.cdt)
            a2 = _lanes(abar, B)
        g2, ga, _ = pullback(np.ascontiguousarray(a2, self.cdt), per, xt.reshape(L, -1), None,
                             np.ascontiguousarray(gxt.reshape(L, -1)))
        gw = g2.reshape(L, B, m, n)
        if not per:
            gabar = ga.reshape(B, m, n).sum(axis=0)
            gpsi = np.einsum("lbhn,blh->hn", gw, u, optimize=True)
            gu = gu + np.einsum("lbhn,hn->blh", gw, np.conj(scale * b), optimize=True).real
            gscale = np.conj(b) * gpsi
            gb = np.conj(scale) * gpsi
            dal, dad, dsl, dsd = scheme_partials(self.scheme, lam, delta[:, None], abar, scale)
            glam = np.conj(dal) * gabar + np.conj(dsl) * gscale
            gdel = ((np.conj(dad) * gabar).real + (np.conj(dsd) * gscale).real).sum(-1)
            glog_delta = gdel * delta
        else:
            ga_k = np.moveaxis(ga.reshape(L, B, m, n), 0, 1)
            gw_b = np.moveaxis(gw, 0, 1)
            gpsi_k = gw_b * u[..., None]
            gu = gu + np.einsum("blhn,blhn->blh", gw_b, np.conj(sc_k * b), optimize=True).real
            gscale_k = np.conj(b) * gpsi_k
            gb = (np.conj(sc_k) * gpsi_k).sum(axis=(0, 1))
            dal, dad, dsl, dsd = scheme_partials(self.scheme, lam, deff[..., None], abar_k, sc_k)
            glam = (np.conj(dal) * ga_k + np.conj(dsl) * gscale_k).sum(axis=(0, 1))
            gdeff = ((np.conj(dad) * ga_k).real + (np.conj(dsd) * gscale_k).real).sum(-1)
            glog_delta = np.einsum("blh,bl->h", gdeff, deltas, optimize=True) * delta
        grads = {"lambda_re_log": -np.exp(p["lambda_re_log"]) * glam.real,
                 "lambda_im": np.ascontiguousarray(glam.imag),
                 "b.re": np.ascontiguousarray(gb.real), "b.im": np.ascontiguousarray(gb.imag),
                 "c.re": np.ascontiguousarray(gc.real), "c.im": np.ascontiguousarray(gc.imag),
                 "d": gd, "log_delta": glog_delta}
        return grads, gu

    def _bwd_mimo(self, s, gy):  # layers.py:691-704, 836-895, 945-980
        u, xt, bu, deltas = s["u"], s["xt"], s["bu"], s["deltas"]
        p = self.p
        B, L, m = u.shape
        Bm, Cm, osc, abar, scale, lam, delta = self._mimo()
        P = Bm.shape[0]
        gD = np.einsum("blh,blh->h", gy, u, optimize=True)
        gu = gy * p["D"]
        gC = osc * np.einsum("blh,lbp->hp", gy, np.conj(xt), optimize=True)
        gxt = osc * np.einsum("blh,hp->lbp", gy, np.conj(Cm), optimize=True)
        per = deltas is not None
        if per:
            deff = deltas[:, :, None] * delta
            abar_k, sc_k = scheme_factors(self.scheme, lam, deff)
            abar_k, sc_k = np.asarray(abar_k, self.cdt), np.asarray(sc_k, self.cdt)
            a2 = _tm(abar_k)
        else:
            a2 = _lanes(abar, B)
        g2, ga, _ = pullback(np.ascontiguousarray(a2, self.cdt), per, xt.reshape(L, -1), None,
                             np.ascontiguousarray(gxt.reshape(L, -1)))
        gv = g2.reshape(L, B, P)
        grads = {}
        if self.kind == "lru":
            glam = ga.reshape(B, P).sum(axis=0)
            gbu = scale * gv
            ggamma = np.einsum("blp,lbp->p", np.conj(bu), gv, optimize=True).real
            cl = np.conj(abar) * glam
            grads["nu_log"] = -np.exp(p["nu_log"]) * cl.real
            grads["theta_log"] = np.exp(p["theta_log"]) * cl.imag
            grads["gamma_log"] = scale * ggamma
        else:
            if not per:
                gabar = ga.reshape(B, P).sum(axis=0)
                gbu = np.conj(scale) * gv
                gscale = np.einsum("blp,lbp->p", np.conj(bu), gv, optimize=True)
                dal, dad, dsl, dsd = scheme_partials(self.scheme, lam, delta, abar, scale)
                glam = np.conj(dal) * gabar + np.conj(dsl) * gscale
                gdel = (np.conj(dad) * gabar).real + (np.conj(dsd) * gscale).real
                glog_delta = gdel * delta
            else:
                ga_k = np.moveaxis(ga.reshape(L, B, P), 0, 1)
                gv_b = np.moveaxis(gv, 0, 1)
                gbu = np.moveaxis(np.conj(sc_k) * gv_b, 1, 0)
                gscale_k = np.conj(bu) * gv_b
                dal, dad, dsl, dsd = scheme_partials(self.scheme, lam, deff, abar_k, sc_k)
                glam = (np.conj(dal) * ga_k + np.conj(dsl) * gscale_k).sum(axis=(0, 1))
                gdeff = (np.conj(dad) * ga_k).real + (np.conj(dsd) * gscale_k).real
                glog_delta = np.einsum("blp,bl->p", gdeff, deltas, optimize=True) * delta
            grads["lambda_re_log"] = -np.exp(p["lambda_re_log"]) * glam.real
            grads["lambda_im"] = np.ascontiguousarray(glam.imag)
        gB = np.einsum("lbp,blh->ph", gbu, u, optimize=True)
        gu = gu + np.einsum("lbp,ph->blh", gbu, np.conj(Bm), optimize=True).real
        grads.update({"B.re": np.ascontiguousarray(gB.real), "B.im": np.ascontiguousarray(gB.imag),
                      "C.re": np.ascontiguousarray(gC.real), "C.im": np.ascontiguousarray(gC.imag),
                      "D": gD})
        if self.kind == "s5":
            grads["log_delta"] = glog_delta
        return grads, gu

    def _bwd_s6(self, s, gy):  # layers.py:1068-1118
        u, xt = s["u"], s["xt"]
        delta, bk, ck, p1, pre = (s[k] for k in ("delta", "bk", "ck", "p1", "pre"))
        p = self.p
        B, L, m = u.shape
        n = p["W_B"].shape[0]
        a = -np.exp(p["a_log"])
        gD = np.einsum("blh,blh->h", gy, u, optimize=True)
        gu = gy * p["D"]
        gck = np.einsum("blh,lbhn->bln", gy, xt, optimize=True)
        gxt = np.moveaxis(gy, 1, 0)[..., None] * np.moveaxis(ck, 1, 0)[:, :, None, :]
        abar = np.exp(delta[..., None] * a)
        g2, ga, _ = pullback(_tm(abar), True, xt.reshape(L, -1), None,
                             np.ascontiguousarray(gxt.reshape(L, -1)))
        gw = np.moveaxis(g2.reshape(L, B, m, n), 0, 1)
        t = abar * np.moveaxis(ga.reshape(L, B, m, n), 0, 1)
        gdelta = np.einsum("blhn,hn->blh", t, a, optimize=True)
        ga_mat = np.einsum("blhn,blh->hn", t, delta, optimize=True)
        s1 = np.einsum("blhn,bln->blh", gw, bk, optimize=True)
        gdelta = gdelta + s1 * u
        gu = gu + delta * s1
        gbk = np.einsum("blhn,blh->bln", gw, delta * u, optimize=True)
        gpre = sigmoid(pre) * gdelta
        gp1 = gpre @ p["W_delta_proj"].T
        gu = gu + gp1 @ p["W_delta"].T + gbk @ p["W_B"] + gck @ p["W_C"]
        grads = {"a_log": a * ga_mat,
                 "W_B": np.einsum("bln,blh->nh", gbk, u, optimize=True),
                 "W_C": np.einsum("bln,blh->nh", gck, u, optimize=True),
                 "W_delta": np.einsum("blh,blr->hr", u, gp1, optimize=True),
                 "W_delta_proj": np.einsum("blr,blh->rh", p1, gpre, optimize=True),
                 "b_delta": gpre.sum(axis=(0, 1)), "D": gD}
        return grads, gu

    def _bwd_rglru(self, s, gy):  # layers.py:1252-1291
        u, xt = s["u"], s["xt"]
        r, ig, ak, sq = (s[k] for k in ("r", "ig", "ak", "s"))
        p = self.p
        B, L, m = u.shape
        la = -softplus(-p["lambda_param"])
        gxt = np.ascontiguousarray(np.moveaxis(gy, 1, 0).reshape(L, -1))
        g2, ga, _ = pullback(_tm(ak), True, xt.reshape(L, -1), None, gxt)
        g = np.moveaxis(g2.reshape(L, B, m), 0, 1)
        gak = np.moveaxis(ga.reshape(L, B, m), 0, 1)
        gloga = ak * gak - (ak * ak / sq) * (ig * u * g)
        gqr = r * (1.0 - r) * (GATE_POWER * la * gloga)
        gqi = ig * (1.0 - ig) * (sq * u * g)
        gu = gqr @ p["W_r"] + gqi @ p["W_i"] + sq * ig * g
        grads = {"lambda_param": sigmoid(-p["lambda_param"]) * (GATE_POWER * r * gloga).sum(axis=(0, 1)),
                 "W_r": np.einsum("blj,blh->jh", gqr, u, optimize=True), "b_r": gqr.sum(axis=(0, 1)),
                 "W_i": np.einsum("blj,blh->jh", gqi, u, optimize=True), "b_i": gqi.sum(axis=(0, 1))}
        return grads, gu


def make_layer(kind, d_model, d_state=None, discretization=None, *, asynchronous=False,
               dtype="f64", seed=0, **extras):
    return Layer(kind, init_params(kind, d_model, d_state, dtype=dtype, seed=seed, **extras),
                 discretization, asynchronous)


def naive_forward(kind, params, u, scheme=None, deltas=None):
    """Independent per-step loop reference (mirrors test_layers.py:21-87)."""
    p = {k: np.asarray(v, np.float64) for k, v in params.items()}
    u = np.asarray(u, np.float64)
    B, L, m = u.shape
    y = np.zeros((B, L, m))
    scheme = scheme or default_scheme(kind, deltas is not None)
    for bi in range(B):
        if kind == "s4d":
            lam = -np.exp(p["lambda_re_log"]) + 1j * p["lambda_im"]
            b = p["b.re"] + 1j * p["b.im"]
            c = p["c.re"] + 1j * p["c.im"]
            x = np.zeros(lam.shape, complex)
            for k in range(L):
                dk = np.exp(p["log_delta"]) * (1.0 if deltas is None else deltas[bi, k])
                ab, sc = scheme_factors(scheme, lam, dk[:, None])
                x = ab * x + sc * b * u[bi, k][:, None]
                y[bi, k] = (c * x).sum(-1).real + p["d"] * u[bi, k]
        elif kind in ("s5", "lru"):
            Bm = p["B.re"] + 1j * p["B.im"]
            Cm = p["C.re"] + 1j * p["C.im"]
            x = np.zeros(Bm.shape[0], complex)
            for k in range(L):
                if kind == "lru":
                    ab = np.exp(-np.exp(p["nu_log"]) + 1j * np.exp(p["theta_log"]))
                    sc = np.exp(p["gamma_log"])
                    osc = 1.0
                else:
                    lam = -np.exp(p["lambda_re_log"]) + 1j * p["lambda_im"]
                    dk = np.exp(p["log_delta"]) * (1.0 if deltas is None else deltas[bi, k])
                    ab, sc = scheme_factors(scheme, lam, dk)
                    osc = 2.0
                x = ab * x + sc * (Bm @ u[bi, k])
                y[bi, k] = osc * (Cm @ x).real + p["D"] * u[bi, k]
        elif kind == "s6":
            a = -np.exp(p["a_log"])
            x = np.zeros(a.shape)
            for k in range(L):
                uk = u[bi, k]
                dl = softplus(uk @ p["W_delta"] @ p["W_delta_proj"] + p["b_delta"])
                x = np.exp(dl[:, None] * a) * x + (dl * uk)[:, None] * (p["W_B"] @ uk)[None, :]
                y[bi, k] = x @ (p["W_C"] @ uk) + p["D"] * uk
        elif kind == "rglru":
            la = -softplus(-p["lambda_param"])
            x = np.zeros(m)
            for k in range(L):
                uk = u[bi, k]
                r = sigmoid(p["W_r"] @ uk + p["b_r"])
                ig = sigmoid(p["W_i"] @ uk + p["b_i"])
                loga = GATE_POWER * r * la
                x = np.exp(loga) * x + np.sqrt(-np.expm1(2 * loga)) * ig * uk
                y[bi, k] = x
    return y


def rel_err(got, ref):
    """max|got-ref| / max|ref| (bench.py:239-241)."""
    got = np.asarray(got, np.complex128 if np.iscomplexobj(got) else np.float64)
    ref = np.asarray(ref, np.complex128 if np.iscomplexobj(ref) else np.float64)
    return float(np.max(np.abs(got - ref))) / max(float(np.max(np.abs(ref))), 1e-30)


# ---------------------------------------------------------------------------
# scan-level operators (the benchmark unit): the layer math between the dense
# projections, restated from the same reference lines, for the CPU baseline.

def rglru_scan(u, qr, qi, lam, b_r, b_i, gy, mode="parallel", workers=1):
    """RG-LRU gates + scan + pullback from gate pre-activations
    (layers.py:1208-1218, 1239-1291 without the W_r / W_i GEMMs)."""
    B, L, W = u.shape
    r = sigmoid(qr + b_r)
    ig = sigmoid(qi + b_i)
    la = -softplus(-lam)
    loga = GATE_POWER * r * la
    ak = np.exp(loga)
    sq = np.sqrt(-np.expm1(2.0 * loga))
    a2 = _tm(ak)
    xt = _run(mode, workers, a2, True, _tm(sq * ig * u)).reshape(L, B, W)
    y = np.moveaxis(xt, 0, 1)
    g2, ga, _ = pullback(a2, True, xt.reshape(L, -1), None, np.ascontiguousarray(_tm(gy)))
    g = np.moveaxis(g2.reshape(L, B, W), 0, 1)
    gak = np.moveaxis(ga.reshape(L, B, W), 0, 1)
    gloga = ak * gak - (ak * ak / sq) * (ig * u * g)
    gqr = r * (1.0 - r) * (GATE_POWER * la * gloga)
    gqi = ig * (1.0 - ig) * (sq * u * g)
    return y, {"gu_local": sq * ig * g, "gqr": gqr, "gqi": gqi,
               "gla": (GATE_POWER * r * gloga).sum(axis=(0, 1)), "gb_r": gqr.sum(axis=(0, 1)),
               "gb_i": gqi.sum(axis=(0, 1))}


def s6_scan(u, pre, b_delta, a_log, Bk, Ck, D, gy, mode="parallel", workers=1):
    """S6 selective scan fwd + pullback from the projection outputs
    (layers.py:1041-1042, 1051-1066, 1068-1098 without the projection GEMMs)."""
    B, L, m = u.shape
    n = Bk.shape[-1]
    a = -np.exp(a_log)
    pre_b = pre + b_delta
    delta = softplus(pre_b)
    abar = np.exp(delta[..., None] * a)
    a2 = _tm(abar)
    xt = _run(mode, workers, a2, True, _tm((delta * u)[..., None] * Bk[:, :, None, :])).reshape(L, B, m, n)
    y = np.einsum("lbhn,bln->blh", xt, Ck, optimize=True) + D * u
    gxt = np.moveaxis(gy, 1, 0)[..., None] * np.moveaxis(Ck, 1, 0)[:, :, None, :]
    g2, ga, _ = pullback(a2, True, xt.reshape(L, -1), None, np.ascontiguousarray(gxt.reshape(L, -1)))
    gw = np.moveaxis(g2.reshape(L, B, m, n), 0, 1)
    t = abar * np.moveaxis(ga.reshape(L, B, m, n), 0, 1)
    s1 = np.einsum("blhn,bln->blh", gw, Bk, optimize=True)
    gdelta = np.einsum("blhn,hn->blh", t, a, optimize=True) + s1 * u
    gpre = sigmoid(pre_b) * gdelta
    return y, {"gu_local": gy * D + delta * s1, "gpre": gpre,
               "gBk": np.einsum("blhn,blh->bln", gw, delta * u, optimize=True),
               "gCk": np.einsum("blh,lbhn->bln", gy, xt, optimize=True),
               "ga_log": a * np.einsum("blhn,blh->hn", t, delta, optimize=True),
               "gD": np.einsum("blh,blh->h", gy, u, optimize=True), "gb_delta": gpre.sum(axis=(0, 1))}


def s6_layer_blocked(params, u, gy, block=128):
    """The S6 layer's taped forward + analytic backward (layers.py:1020-1027,
    1051-1118) with the scan part run over blocks of `block` channels: the
    recurrence is per channel, only gB_k / gC_k (layers.py:1080, 1098) sum
    over channels, so they are accumulated over the blocks.  Same arithmetic
    as Layer("s6").forward/backward with a bounded [L, B, block, N] footprint
    (full-length C3 rows).  Returns (y, grads, gu, {gBk, gCk})."""
    p = {k: np.asarray(v, np.float64) for k, v in params.items()}
    u, gy = np.asarray(u, np.float64), np.asarray(gy, np.float64)
    m = u.shape[-1]
    p1 = u @ p["W_delta"]
    pre0 = p1 @ p["W_delta_proj"]  # s6_scan adds b_delta
    bk, ck = u @ p["W_B"].T, u @ p["W_C"].T
    y = np.empty_like(u)
    gu, gpre = np.empty_like(u), np.empty_like(u)
    gbk, gck = np.zeros_like(bk), np.zeros_like(ck)
    ga_log, gD, gb = np.empty_like(p["a_log"]), np.empty(m), np.empty(m)
    for h0 in range(0, m, block):
        hs = slice(h0, min(m, h0 + block))
        yb, r = s6_scan(u[..., hs], pre0[..., hs], p["b_delta"][hs], p["a_log"][hs], bk, ck, p["D"][hs],
                        gy[..., hs], "sequential", 1)
        y[..., hs], gu[..., hs], gpre[..., hs] = yb, r["gu_local"], r["gpre"]
        gbk += r["gBk"]
        gck += r["gCk"]
        ga_log[hs], gD[hs], gb[hs] = r["ga_log"], r["gD"], r["gb_delta"]
    gp1 = gpre @ p["W_delta_proj"].T
    gu = gu + gp1 @ p["W_delta"].T + gbk @ p["W_B"] + gck @ p["W_C"]
    grads = {"a_log": ga_log,
             "W_B": np.einsum("bln,blh->nh", gbk, u, optimize=True),
             "W_C": np.einsum("bln,blh->nh", gck, u, optimize=True),
             "W_delta": np.einsum("blh,blr->hr", u, gp1, optimize=True),
             "W_delta_proj": np.einsum("blr,blh->rh", p1, gpre, optimize=True),
             "b_delta": gb, "D": gD}
    return y, grads, gu, {"gBk": gbk, "gCk": gck}
