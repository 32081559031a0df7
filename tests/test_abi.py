"""The C-ABI library loads and exports exactly what include/lrx.h declares
(no compute calls: this runs without a GPU)."""
import ctypes
import os
import re

from paper_2602_08810_b200 import _lib
from tests.conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "lrx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(lrx_\w+)\s*\(", src))


def test_library_exports_every_declared_symbol():
    lib = _lib.load(require_gpu=False)
    names = _declared()
    assert len(names) >= 20
    for n in sorted(names):
        assert hasattr(lib, n), n


def test_binding_table_matches_header():
    assert set(_lib.SIGNATURES) == _declared()


def test_header_argument_counts_match_binding():
    src = open(os.path.join(ROOT, "include", "lrx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    for name, args in re.findall(r"\b(lrx_\w+)\s*\(([^)]*)\)\s*;", src, flags=re.S):
        n = 0 if args.strip() in ("", "void") else args.count(",") + 1
        assert n == len(_lib.SIGNATURES[name][1]), name


def test_host_queries_without_gpu():
    lib = _lib.load(require_gpu=False)
    assert lib.lrx_version() == 1
    assert lib.lrx_scan_workspace_bytes(_lib.F32, 1000, 4096) > 1000 * 4096 // 32
    ck, nc = ctypes.c_int64(), ctypes.c_int64()
    assert lib.lrx_rglru_chunking(_lib.F32, 1000, ctypes.byref(ck), ctypes.byref(nc)) == 0
    assert ck.value * nc.value >= 1000
    geo = (ctypes.c_int64 * 6)()
    assert lib.lrx_s6_geometry(_lib.BF16, 16, 8192, 1536, 16, geo) == 0
    ck, nck, ndb, nseg, prow, ws = geo
    assert nck == -(-8192 // ck) + 1 and ndb == 1536 // 64 and prow == nseg * 16 and ws > 0
    # B=1 long sequence: time segments fill the GPU
    assert lib.lrx_s6_geometry(_lib.BF16, 1, 2 ** 20, 2048, 16, geo) == 0
    assert geo[3] > 1 and geo[4] == geo[3]
    # f64 runs the generic kernels (one segment, no workspace)
    assert lib.lrx_s6_geometry(_lib.F64, 2, 100, 24, 16, geo) == 0
    assert geo[3] == 1 and geo[4] == 2 and geo[5] == 0
    # d_state beyond the compiled range is a loud, typed error
    assert lib.lrx_s6_geometry(_lib.F32, 1, 10, 10, 65, geo) == _lib.ERR_UNSUPPORTED
    assert b"65" in lib.lrx_last_error()


def test_shape_errors_are_reported_before_launch():
    lib = _lib.load(require_gpu=False)
    rc = lib.lrx_scan_fwd(_lib.F32, 0, None, None, None, None, 0, 4, None, 0, None)
    assert rc == _lib.ERR_SHAPE
    assert b"length" in lib.lrx_last_error()


def test_gemm_wrappers_reject_mismatched_operands():
    import pytest
    import torch

    from paper_2602_08810_b200 import ops
    a, bt = torch.zeros(8, 16), torch.zeros(4, 12)
    with pytest.raises(ValueError, match="disagree on K"):
        ops.gemm_f32(a, bt)
    with pytest.raises(ValueError, match="disagree on K"):
        ops.gemm_bf16(a.bfloat16(), bt.bfloat16())
    with pytest.raises(ValueError, match="disagree on K"):
        ops.gemm_f32_tn(a, torch.zeros(7, 4))
    with pytest.raises(ValueError, match="not \\[M, N\\]"):
        ops.gemm_f32(a, torch.zeros(4, 16), Cin=torch.zeros(8, 5))
