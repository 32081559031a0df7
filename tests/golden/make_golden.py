"""Generate golden vectors by running the REAL reference (`linrec`) here.

Run in the build container only (the reference tree does not exist on the GPU
box):

    python tests/golden/make_golden.py

It imports linrec from /root/reference/pkg/src with a scratch NUMBA_CACHE_DIR
and PYTHONDONTWRITEBYTECODE so that nothing is written into the read-only
reference tree, then records inputs, parameters, outputs and gradients of the
reference's own public API (make_layer / Layer.forward / layer_backward,
scan_sequential / scan_parallel / scan_forward / scan_backward) into small
.npz fixtures beside this script.  tests/test_oracle_golden.py pins the oracle
restatement (oracle/port.py) to these files, and the GPU parity tests reuse
them as fixed inputs.
"""
from __future__ import annotations

import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "lrx_numba_cache"))
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

import linrec  # noqa: E402
from linrec import layer_backward, make_layer  # noqa: E402
from linrec.numerics import Rng  # noqa: E402
from linrec.scan import scan_parallel, scan_sequential  # noqa: E402
from linrec.autograd import scan_backward, scan_forward  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

LAYER_CASES = [
    # name, kind, scheme, d_model, d_state, B, L, dtype, async
    ("s4d_zoh", "s4d", "zoh", 3, 4, 2, 40, "f64", False),
    ("s4d_bilinear", "s4d", "bilinear", 3, 4, 2, 40, "f64", False),
    ("s4d_dirac", "s4d", "dirac", 3, 4, 2, 40, "f64", False),
    ("s5_zoh", "s5", "zoh", 3, 4, 2, 40, "f64", False),
    ("s5_bilinear", "s5", "bilinear", 3, 4, 2, 40, "f64", False),
    ("s5_dirac", "s5", "dirac", 3, 4, 2, 40, "f64", False),
    ("lru", "lru", None, 3, 4, 2, 40, "f64", False),
    ("s6", "s6", None, 3, 4, 2, 40, "f64", False),
    ("rglru", "rglru", None, 3, None, 2, 40, "f64", False),
    # async event-stream deltas (continuous-time LTI kinds only)
    ("s4d_zoh_async", "s4d", "zoh", 3, 4, 2, 30, "f64", True),
    ("s4d_bilinear_async", "s4d", "bilinear", 3, 4, 2, 30, "f64", True),
    ("s4d_dirac_async", "s4d", "dirac", 3, 4, 2, 30, "f64", True),
    ("s5_zoh_async", "s5", "zoh", 3, 4, 2, 30, "f64", True),
    ("s5_bilinear_async", "s5", "bilinear", 3, 4, 2, 30, "f64", True),
    ("s5_dirac_async", "s5", "dirac", 3, 4, 2, 30, "f64", True),
    # wider / longer cases crossing the 256-step chunk floor and warp widths
    ("lru_wide", "lru", None, 16, 24, 2, 260, "f64", False),
    ("s5_wide", "s5", "zoh", 16, 48, 2, 260, "f64", False),
    ("s6_wide", "s6", None, 20, 16, 2, 260, "f64", False),
    ("rglru_wide", "rglru", None, 40, None, 2, 260, "f64", False),
    ("s4d_wide", "s4d", "zoh", 12, 8, 2, 260, "f64", False),
    # the reference's own f32 path
    ("lru_f32", "lru", None, 16, 24, 2, 260, "f32", False),
    ("s5_f32", "s5", "zoh", 16, 48, 2, 260, "f32", False),
    ("s6_f32", "s6", None, 20, 16, 2, 260, "f32", False),
    ("rglru_f32", "rglru", None, 40, None, 2, 260, "f32", False),
]


def layer_case(name, kind, scheme, m, n, B, L, dtype, asyn):
    layer = make_layer(kind, m, d_state=n, discretization=scheme,
                       asynchronous=asyn, dtype=dtype, seed=11)
    rng = Rng(sum(map(ord, name)))
    u = np.asarray(rng.normal((B, L, m)), layer.rdt)
    gy = np.asarray(rng.normal((B, L, m)), layer.rdt)
    deltas = np.asarray(rng.uniform(0.1, 3.0, (B, L)), layer.rdt) if asyn else None
    y, tape = layer.forward(u, "sequential", deltas=deltas, tape=True)
    g = layer_backward(layer, tape, gy)
    y_par = layer.forward(u, "parallel", workers=3, deltas=deltas)
    rec = {"kind": kind, "scheme": scheme or "", "d_model": m,
           "d_state": -1 if n is None else n, "dtype": dtype, "seed": 11,
           "u": u, "gy": gy, "y": y, "gu": g.u}
    if L <= 64:
        rec["y_par"] = y_par
    if deltas is not None:
        rec["deltas"] = deltas
    for k, v in layer.parameters().items():
        rec["param:" + k] = v
    for k, v in g.params.items():
        rec["grad:" + k] = v
    np.savez_compressed(os.path.join(OUT, f"layer_{name}.npz"), **rec)


def scan_cases():
    rec = {}
    rng = Rng(2024)
    # real / complex x const / per-step, with and without x0; L crosses 256
    for tag, cplx in (("real", False), ("cplx", True)):
        for per in (False, True):
            L, N = 300, 7
            shape_a = (L, N) if per else (N,)
            if cplx:
                a = 0.95 * np.exp(1j * rng.normal(shape_a) * 0.3) * rng.uniform(0.5, 1.0, shape_a)
                b = rng.normal((L, N)) + 1j * rng.normal((L, N))
                x0 = rng.normal(N) + 1j * rng.normal(N)
            else:
                a = rng.uniform(0.3, 0.99, shape_a) * np.sign(rng.normal(shape_a))
                b = rng.normal((L, N))
                x0 = rng.normal(N)
            key = f"{tag}_{'var' if per else 'const'}"
            rec[key + ":a"] = a
            rec[key + ":b"] = b
            rec[key + ":x0"] = x0
            rec[key + ":seq"] = scan_sequential(a, b, x0=x0)
            rec[key + ":par3"] = scan_parallel(a, b, x0=x0, workers=3)
            gx = rng.normal((L, N)) + (1j * rng.normal((L, N)) if cplx else 0)
            _, tape = scan_forward(a, b, x0)
            ga, gb, gx0 = scan_backward(tape, gx)
            rec[key + ":gx"] = gx
            rec[key + ":ga"] = ga
            rec[key + ":gb"] = gb
            rec[key + ":gx0"] = gx0
    np.savez_compressed(os.path.join(OUT, "scan_ops.npz"), **rec)


def main():
    for case in LAYER_CASES:
        layer_case(*case)
    scan_cases()
    with open(os.path.join(OUT, "PROVENANCE.txt"), "w") as f:
        f.write(f"generated by tests/golden/make_golden.py from linrec {linrec.__version__} "
                f"at {REF}; numpy {np.__version__}\n")
    print("wrote", len(LAYER_CASES) + 1, "fixtures to", OUT)


if __name__ == "__main__":
    main()
