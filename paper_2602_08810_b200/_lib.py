"""ctypes binding of liblrx.so, the sm_100a C-ABI declared in include/lrx.h.

There is no fallback: if the shared object is missing, fails to load, or no
CUDA device is present, every compute entry point raises.  Status codes map to
the reference's exception types (numerics.ShapeError, ValueError,
discretize.SingularBilinear).
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblrx.so")

F32, F64, C64, C128, BF16 = 0, 1, 2, 3, 4
OK, ERR_SHAPE, ERR_VALUE, ERR_SINGULAR, ERR_CUDA, ERR_UNSUPPORTED = range(6)

_vp, _i, _i64, _sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
_P64 = ctypes.POINTER(ctypes.c_int64)

# name -> (restype, argtypes); must mirror include/lrx.h exactly
SIGNATURES = {
    "lrx_last_error": (ctypes.c_char_p, []),
    "lrx_version": (_i, []),
    "lrx_launch_count": (_i64, []),
    "lrx_scan_workspace_bytes": (_sz, [_i, _i64, _i64]),
    "lrx_scan_fwd": (_i, [_i, _i, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _sz, _vp]),
    "lrx_scan_bwd_workspace_bytes": (_sz, [_i, _i64, _i64]),
    "lrx_scan_bwd": (_i, [_i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _sz, _vp]),
    "lrx_rglru_chunking": (_i, [_i, _i64, _P64, _P64]),
    "lrx_rglru_workspace_bytes": (_sz, [_i, _i64, _i64, _i64]),
    "lrx_rglru_fwd": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp]),
    "lrx_rglru_bwd": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                           _i64, _i64, _i64, _vp, _sz, _vp]),
    "lrx_s6_geometry": (_i, [_i, _i64, _i64, _i64, _i64, _P64]),
    "lrx_s6_fwd": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _i64,
                        _i, _vp]),
    "lrx_s6_bwd": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                        _vp, _i64, _i64, _i64, _i64, _vp, _i64, _i, _vp]),
    "lrx_s6_fwd_carry": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _i64, _vp]),
    "lrx_s6_bwd_carry": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _i64, _vp]),
    "lrx_mimo_chunking": (_i, [_i, _i64, _i64, _i64, _P64, _P64]),
    "lrx_mimo_workspace_bytes": (_sz, [_i, _i64, _i64, _i64]),
    "lrx_mimo_fwd": (_i, [_i, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp]),
    "lrx_mimo_bwd_workspace_bytes": (_sz, [_i, _i64, _i64, _i64]),
    "lrx_mimo_bwd": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp]),
    "lrx_mimo_ps_workspace_bytes": (_sz, [_i, _i64, _i64, _i64]),
    "lrx_mimo_fwd_ps": (_i, [_i, _vp, _vp, _vp, _i, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp]),
    "lrx_mimo_bwd_ps": (_i, [_i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp]),
    "lrx_mimo_fused_workspace_bytes": (_i, [_i64, _i64, _i64, _P64]),
    "lrx_mimo_fused_units": (_i, [_i64, _i64, _P64]),
    "lrx_mimo_fused_fwd": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _sz, _vp]),
    "lrx_mimo_fused_bwd": (_i, [_vp, _vp, _vp, ctypes.c_float, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64,
                                _vp, _sz, _vp]),
    "lrx_reduce_rows": (_i, [_i, _vp, _vp, _i64, _i64, _vp]),
    "lrx_reduce_rows_ws_bytes": (_sz, [_i, _i64, _i64]),
    "lrx_reduce_rows_ws": (_i, [_i, _vp, _vp, _vp, _i64, _i64, _vp, _sz, _vp]),
    "lrx_scan_step": (_i, [_i, _vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "lrx_s4d_step": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "lrx_mimo_step": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_double, _i64, _i64,
                           _i64, _vp]),
    "lrx_s6_step": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "lrx_rglru_step": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp]),
    "lrx_s6_step_fused": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64,
                               _vp]),
    "lrx_rglru_step_fused": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp]),
    "lrx_gemm_f32": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i64, _i64, _i64, ctypes.c_float, ctypes.c_float,
                          _vp]),
    "lrx_gemm_f32_tn_splits": (_i, [_i64, _i64, _i64, _P64]),
    "lrx_gemm_f32_tn": (_i, [_vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_float, _vp]),
    "lrx_s4d_coef": (_i, [_i, _i, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "lrx_s4d_coef_grads": (_i, [_i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "lrx_cast": (_i, [_i, _i, _vp, _vp, _i64, _vp]),
    "lrx_gemm_bf16": (_i, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_float, ctypes.c_float, _i, _i, _vp]),
    "lrx_s4d_chunking": (_i, [_i64, _P64, _P64]),
    "lrx_s4d_geometry": (_i, [_i, _i64, _i64, _i64, _i64, _P64]),
    "lrx_s4d_fwd": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64,
                         _vp, _sz, _vp]),
    "lrx_s4d_bwd": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                         _vp, _i64, _i64, _i64, _i64, _vp, _sz, _vp]),
    "lrx_mimo_coef": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                           _vp, _vp, _vp, _i, _vp]),
    "lrx_mimo_coef_grads": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp,
                                 ctypes.c_double, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp]),
}

_lib = None
_lock = threading.Lock()


class LrxError(RuntimeError):
    """A CUDA-side failure inside liblrx."""


def load(require_gpu=True):
    """Load liblrx.so (and check for a CUDA device unless require_gpu=False)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2602_08810_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_gpu and not torch.cuda.is_available():
        raise RuntimeError("liblrx needs a CUDA device (B200, sm_100a); none is visible")
    return _lib


def lib():
    return load(True)


def _exc(rc, msg):
    from .discretize import SingularBilinear
    from .numerics import ShapeError
    if rc == ERR_SHAPE:
        return ShapeError(msg)
    if rc == ERR_VALUE:
        return ValueError(msg)
    if rc == ERR_SINGULAR:
        return SingularBilinear(msg)
    if rc == ERR_UNSUPPORTED:
        return NotImplementedError(msg)
    return LrxError(msg)


def check(rc):
    if rc != OK:
        raise _exc(rc, load(False).lrx_last_error().decode(errors="replace"))


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def workspace(nbytes, device):
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def launch_count():
    return int(load(False).lrx_launch_count())


def code_of(dtype: torch.dtype) -> int:
    return {torch.float32: F32, torch.float64: F64, torch.complex64: C64,
            torch.complex128: C128, torch.bfloat16: BF16}[dtype]


def i64():
    return ctypes.c_int64(0)


def ref(x):
    return ctypes.byref(x)
