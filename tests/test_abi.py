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
    ndb = ctypes.c_int64()
    assert lib.lrx_s6_ckpt_len(_lib.BF16, 8192, 1536, 16, ctypes.byref(ck), ctypes.byref(nc), ctypes.byref(ndb)) == 0
    assert nc.value == -(-8192 // ck.value) + 1 and ndb.value >= 1
    # d_state beyond the compiled range is a loud, typed error
    assert lib.lrx_s6_ckpt_len(_lib.F32, 10, 10, 65, ctypes.byref(ck), ctypes.byref(nc),
                               ctypes.byref(ndb)) == _lib.ERR_UNSUPPORTED
    assert b"65" in lib.lrx_last_error()


def test_shape_errors_are_reported_before_launch():
    lib = _lib.load(require_gpu=False)
    rc = lib.lrx_scan_fwd(_lib.F32, 0, None, None, None, None, 0, 4, None, 0, None)
    assert rc == _lib.ERR_SHAPE
    assert b"length" in lib.lrx_last_error()
