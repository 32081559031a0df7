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
           "torch_real", "torch_complex", "softplus", "sigmoid", "Rng"]

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
