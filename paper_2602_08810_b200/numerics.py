"""Numeric substrate of the drop-in API (mirrors pkg/src/linrec/numerics.py).

Host-side helpers only: the dtype policy, the exception type, the Philox RNG
used for parameter initialisation (so `make_layer(..., seed=s)` yields the
reference's exact parameters), and softplus / sigmoid for either numpy arrays
or torch tensors.  The scan itself never runs here.
"""
from __future__ import annotations

import numpy as np
import torch

__all__ = ["REAL_DTYPES", "SOFTPLUS_THRESHOLD", "ShapeError", "real_dtype", "complex_dtype",
           "torch_real", "torch_complex", "softplus", "sigmoid", "Rng", "as_tensor", "complex_exp",
           "ComplexPair", "alloc", "allocation_count"]

REAL_DTYPES = {"f32": np.dtype(np.float32), "f64": np.dtype(np.float64)}
# numerics.py:36-39
SOFTPLUS_THRESHOLD = {np.dtype(np.float32): 30.0, np.dtype(np.float64): 50.0}

_T_REAL = {"f32": torch.float32, "f64": torch.float64, "bf16": torch.float32}
_T_CPLX = {"f32": torch.complex64, "f64": torch.complex128, "bf16": torch.complex64}


class ShapeError(ValueError):
    """An array's shape violates an operation's contract (numerics.py:42)."""


def real_dtype(spec) -> np.dtype:
    if isinstance(spec, str):
        if spec == "bf16":
            return np.dtype(np.float32)
        try:
            return REAL_DTYPES[spec]
        except KeyError:
            raise ValueError(f"unknown dtype spec {spec!r}; expected 'f32', 'f64' or 'bf16'") from None
    dt = np.dtype(spec)
    return {np.dtype(np.complex64): np.dtype(np.float32),
            np.dtype(np.complex128): np.dtype(np.float64)}.get(dt, dt)


def complex_dtype(spec) -> np.dtype:
    return {np.dtype(np.float32): np.dtype(np.complex64),
            np.dtype(np.float64): np.dtype(np.complex128)}[real_dtype(spec)]


def torch_real(spec) -> torch.dtype:
    return _T_REAL[spec]


def torch_complex(spec) -> torch.dtype:
    return _T_CPLX[spec]


def _thr(dtype):
    return 50.0 if dtype in (torch.float64, np.float64) else 30.0


def softplus(x):
    """ln(1+e^x), identity above the per-dtype threshold (numerics.py:86-94)."""
    if isinstance(x, torch.Tensor):
        t = _thr(x.dtype)
        return torch.where(x > t, x, torch.log1p(torch.exp(torch.clamp(x, max=t))))
    x = np.asarray(x)
    if x.dtype not in SOFTPLUS_THRESHOLD:
        x = x.astype(np.float64)
    t = SOFTPLUS_THRESHOLD[x.dtype]
    out = np.where(x > t, x, np.log1p(np.exp(np.minimum(x, t))))
    return out[()] if out.ndim == 0 else out


def sigmoid(x):
    """Overflow-free logistic (numerics.py:97-105)."""
    if isinstance(x, torch.Tensor):
        e = torch.exp(torch.where(x >= 0, -x, x))
        return torch.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e))
    x = np.asarray(x)
    if x.dtype not in SOFTPLUS_THRESHOLD:
        x = x.astype(np.float64)
    pos = x >= 0
    e = np.exp(np.where(pos, -x, x))
    out = np.where(pos, 1.0 / (1.0 + e), e / (1.0 + e))
    return out[()] if out.ndim == 0 else out


class Rng:
    """Splittable counter-based RNG (Philox over a SeedSequence), identical in
    stream layout to the reference's Rng (numerics.py:180-204)."""

    def __init__(self, seed: int = 0, *, _seq=None):
        self._seq = np.random.SeedSequence(seed) if _seq is None else _seq
        self._gen = np.random.Generator(np.random.Philox(self._seq))
        self.seed = seed if _seq is None else None

    def normal(self, shape=(), dtype="f64"):
        return self._gen.standard_normal(shape, dtype=real_dtype(dtype))

    def uniform(self, low=0.0, high=1.0, shape=(), dtype="f64"):
        out = self._gen.uniform(low, high, shape)
        if np.ndim(out) == 0:
            return np.asarray(out, dtype=real_dtype(dtype))[()]
        return out.astype(real_dtype(dtype), copy=False)

    def integers(self, low, high=None, shape=()):
        return self._gen.integers(low, high, size=shape)

    def split(self, n: int):
        return [Rng(_seq=s) for s in self._seq.spawn(n)]


# ---------------------------------------------------------------------------
# host array helpers of the reference's public numerics API (numerics.py:67-175)

_CPLX_OF = {np.dtype(np.float32): np.dtype(np.complex64), np.dtype(np.float64): np.dtype(np.complex128)}
_SUPPORTED = set(_CPLX_OF) | set(_CPLX_OF.values())


def as_tensor(values, dtype=None) -> np.ndarray:
    """C-contiguous array in a supported dtype (f32/f64/c64/c128); integer or
    bool input becomes float64, other complex input complex128 (numerics.py:67-83)."""
    arr = np.asarray(values)
    if dtype is not None:
        dt = REAL_DTYPES[dtype] if isinstance(dtype, str) and dtype in REAL_DTYPES else np.dtype(dtype)
    elif arr.dtype in _SUPPORTED:
        dt = arr.dtype
    else:
        dt = np.dtype(np.complex128 if np.issubdtype(arr.dtype, np.complexfloating) else np.float64)
    if dt not in _SUPPORTED:
        raise ValueError(f"unsupported tensor dtype {dt}")
    return np.ascontiguousarray(arr, dtype=dt)


def complex_exp(re, im=None):
    """e^z.  One complex argument -> complex result; two real planes (re, im)
    -> the planes (e^re cos im, e^re sin im) (numerics.py:108-128)."""
    if im is None:
        z = np.asarray(re)
        r = np.exp(z.real)
        out = (r * np.cos(z.imag) + 1j * (r * np.sin(z.imag))).astype(_CPLX_OF.get(np.asarray(r).dtype,
                                                                                     np.dtype(np.complex128)))
        return out[()] if out.ndim == 0 else out
    re, im = np.asarray(re), np.asarray(im)
    if re.shape != im.shape:
        raise ShapeError(f"plane shapes differ: {re.shape} vs {im.shape}")
    r = np.exp(re)
    return r * np.cos(im), r * np.sin(im)


class ComplexPair:
    """A complex array held as two real planes of one shape (numerics.py:131-154)."""

    __slots__ = ("re", "im")

    def __init__(self, re, im):
        if np.shape(re) != np.shape(im):
            raise ShapeError(f"plane shapes differ: {np.shape(re)} vs {np.shape(im)}")
        object.__setattr__(self, "re", re)
        object.__setattr__(self, "im", im)

    def __setattr__(self, name, value):  # frozen, like the reference's dataclass
        raise AttributeError("ComplexPair is immutable")

    @property
    def shape(self):
        return np.shape(self.re)

    def to_complex(self) -> np.ndarray:
        re = np.asarray(self.re)
        return (re + 1j * np.asarray(self.im)).astype(_CPLX_OF[np.dtype(re.dtype)])

    @classmethod
    def from_complex(cls, z) -> "ComplexPair":
        z = np.asarray(z)
        return cls(np.ascontiguousarray(z.real), np.ascontiguousarray(z.imag))


_ALLOCATIONS = [0]


def alloc(shape, dtype) -> np.ndarray:
    """Uninitialised host buffer, counted (numerics.py:165-169).  The device
    paths allocate through torch; step mode (Layer.step / StepGraph) allocates
    no host buffers per token."""
    _ALLOCATIONS[0] += 1
    return np.empty(shape, dtype)


def allocation_count() -> int:
    """alloc() calls since import (compare deltas; numerics.py:172-174)."""
    return _ALLOCATIONS[0]

