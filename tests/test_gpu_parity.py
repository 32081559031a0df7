"""GPU parity: the sm_100a kernels (through the drop-in API / C-ABI) against the
reference's golden outputs and the f64 oracle restatement.

Error metric everywhere: max|got - ref| / max|ref| (reference bench.py:239-241).
Tolerances (north_star): fp32 1e-4, bf16 I/O with fp32 accumulation 1e-2;
f64 kernels are held to 1e-10 (the reference's own mode-equivalence bar).
"""
import glob
import os

import numpy as np
import pytest
import torch

from oracle import port
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-10, "f32": 1e-4, "bf16": 1e-2}
LAYER_FILES = sorted(glob.glob(os.path.join(GOLDEN, "layer_*.npz")))


@pytest.fixture(scope="module")
def lrx():
    import paper_2602_08810_b200 as m
    return m


def rel(got, ref):
    if isinstance(got, torch.Tensor):
        got = got.detach().float().cpu().numpy() if got.dtype == torch.bfloat16 else got.detach().cpu().numpy()
    return port.rel_err(got, ref)


def _golden(path):
    z = np.load(path)
    rec = {k: z[k] for k in z.files}
    n = int(rec["d_state"])
    return rec, str(rec["kind"]), (str(rec["scheme"]) or None), (None if n < 0 else n)


def _oracle_f64(kind, scheme, params, u, gy, deltas=None, asyn=False):
    p64 = {k: np.asarray(v, np.float64) for k, v in params.items()}
    lay = port.Layer(kind, p64, scheme, asynchronous=asyn)
    y, saved = lay.forward(np.asarray(u, np.float64), deltas=None if deltas is None else np.asarray(deltas, np.float64))
    g, gu = lay.backward(saved, np.asarray(gy, np.float64))
    return y, g, gu


@pytest.mark.parametrize("path", LAYER_FILES, ids=lambda p: os.path.basename(p)[6:-4])
def test_layer_matches_reference_golden(lrx, path):
    rec, kind, scheme, n = _golden(path)
    dtype = str(rec["dtype"])
    asyn = "deltas" in rec
    layer = lrx.make_layer(kind, int(rec["d_model"]), n, scheme, asynchronous=asyn, dtype=dtype, seed=11)
    deltas = rec.get("deltas")
    for mode in ("sequential", "parallel"):
        y, tape = layer.forward(rec["u"], mode, workers=3, deltas=deltas, tape=True)
        g = lrx.layer_backward(layer, tape, rec["gy"])
        assert isinstance(y, np.ndarray) and y.dtype == layer.rdt
        if dtype == "f64":
            ref_y, ref_g, ref_gu = rec["y"], {k[5:]: rec[k] for k in rec if k.startswith("grad:")}, rec["gu"]
        else:  # f32 path is judged against the f64 ground truth on the same inputs
            params = {k[6:]: rec[k] for k in rec if k.startswith("param:")}
            ref_y, ref_g, ref_gu = _oracle_f64(kind, scheme, params, rec["u"], rec["gy"], deltas, asyn)
        tol = TOL[dtype]
        assert rel(y, ref_y) < tol, (mode, rel(y, ref_y))
        assert rel(g.u, ref_gu) < tol, (mode, rel(g.u, ref_gu))
        assert list(g.params) == list(layer.parameters())
        for k, v in ref_g.items():
            assert g.params[k].shape == v.shape, k
            assert rel(g.params[k], v) < tol, (mode, k, rel(g.params[k], v))


def test_modes_agree_bitwise_and_runs_are_deterministic(lrx):
    for kind, n in (("s6", 16), ("rglru", None), ("s5", 32), ("lru", 16), ("s4d", 8)):
        layer = lrx.make_layer(kind, 24, n, dtype="f32", seed=3)
        u = port.Rng(5).normal((2, 700, 24)).astype(np.float32)
        gy = port.Rng(6).normal((2, 700, 24)).astype(np.float32)
        outs = []
        for mode in ("sequential", "parallel", "parallel"):
            y, tape = layer.forward(u, mode, workers=7, tape=True)
            g = lrx.layer_backward(layer, tape, gy)
            outs.append((y, g.u, g.params))
        for y, gu, gp in outs[1:]:
            np.testing.assert_array_equal(y, outs[0][0])
            np.testing.assert_array_equal(gu, outs[0][1])
            for k in gp:
                np.testing.assert_array_equal(gp[k], outs[0][2][k], err_msg=f"{kind}:{k}")


def test_lti_ltv_entry_points(lrx):
    """lti_forward / ltv_forward route to forward and refuse the other family
    (reference test_layers.py:318-329)."""
    u = port.Rng(71).normal((2, 9, 3))
    layer = lrx.make_layer("s5", 3, 4)
    np.testing.assert_array_equal(lrx.lti_forward(layer, u), layer.forward(u))
    with pytest.raises(ValueError):
        lrx.lti_forward(lrx.make_layer("s6", 3, 2), u)
    ltv = lrx.make_layer("rglru", 3)
    np.testing.assert_array_equal(lrx.ltv_forward(ltv, u), ltv.forward(u))
    with pytest.raises(ValueError):
        lrx.ltv_forward(layer, u)


@pytest.mark.parametrize("kind", ["s4d", "s5", "lru", "s6", "rglru"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_validation_grid(lrx, kind, dtype):
    """The reference's validation grid (bench.py:185-190, run_validation):
    L in {1, 2, 257, 1024} x B in {1, 4} x H in {1, 8} x N in {2, 16}, every
    output and gradient against the f64 oracle."""
    tol = TOL[dtype]
    for L in (1, 2, 257, 1024):
        for B in (1, 4):
            for H in (1, 8):
                for N in (2, 16):
                    layer = lrx.make_layer(kind, H, None if kind == "rglru" else N, dtype=dtype, seed=L + B + H + N)
                    u = port.Rng(L * 7 + B).normal((B, L, H)).astype(layer.rdt)
                    gy = port.Rng(L * 7 + B + 1).normal((B, L, H)).astype(layer.rdt)
                    y, tape = layer.forward(u, tape=True)
                    g = lrx.layer_backward(layer, tape, gy)
                    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
                    ry, rg, rgu = _oracle_f64(kind, layer.discretization, params, u, gy)
                    case = (L, B, H, N)
                    assert rel(y, ry) < tol, case
                    assert rel(g.u, rgu) < tol, case
                    for k in rg:
                        assert rel(g.params[k], rg[k]) < tol, (case, k, rel(g.params[k], rg[k]))


@pytest.mark.parametrize("kind,m,n,B,L", [
    ("s6", 40, 16, 2, 1500), ("s6", 33, 4, 3, 70), ("s6", 16, 8, 1, 129), ("s6", 8, 32, 2, 100),
    ("s6", 12, 64, 1, 80), ("s6", 20, 13, 2, 65),
    ("rglru", 200, None, 3, 1111), ("rglru", 7, None, 1, 1), ("rglru", 130, None, 2, 33),
    ("s5", 64, 128, 2, 1024), ("s5", 10, 6, 3, 2), ("lru", 128, 64, 2, 1024), ("lru", 5, 3, 1, 17),
    ("lru", 128, 64, 8, 1024), ("s5", 64, 128, 4, 1100),  # >= 4096 tokens: tcgen05 projections
    ("rglru", 64, None, 2, 2100), ("s6", 256, 16, 2, 2100),
    ("s4d", 6, 10, 2, 300),
])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_layer_matches_oracle_multichunk(lrx, kind, m, n, B, L, dtype):
    layer = lrx.make_layer(kind, m, n, dtype=dtype, seed=17)
    u = port.Rng(1).normal((B, L, m)).astype(layer.rdt)
    gy = port.Rng(2).normal((B, L, m)).astype(layer.rdt)
    y, tape = layer.forward(u, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64(kind, layer.discretization, params, u, gy)
    tol = TOL[dtype]
    assert rel(y, ry) < tol
    assert rel(g.u, rgu) < tol
    for k in rg:
        assert rel(g.params[k], rg[k]) < tol, (k, rel(g.params[k], rg[k]))


@pytest.mark.parametrize("n", [32, 64])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_s6_wide_state_groups_match_oracle(lrx, n, dtype):
    """d_state 32 / 64 run as 16-state groups on the v3 kernels (fp32 sums over
    the groups); prefill state for step mode comes from the grouped checkpoints."""
    m, B, L = 24, 2, 700
    layer = lrx.make_layer("s6", m, n, dtype=dtype, seed=81)
    io = torch.bfloat16 if dtype == "bf16" else torch.float32
    u = torch.from_numpy(port.Rng(82).normal((B, L, m))).to("cuda", io)
    gy = torch.from_numpy(port.Rng(83).normal((B, L, m))).to("cuda", io)
    y, tape = layer.forward(u, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64("s6", None, params, u.float().cpu().numpy(), gy.float().cpu().numpy())
    tol = TOL[dtype]
    assert rel(y, ry) < tol
    assert rel(g.u, rgu) < tol
    for k in rg:
        assert rel(g.params[k], rg[k]) < tol, (k, rel(g.params[k], rg[k]))
    _, st = layer.forward(u[:, :300], return_state=True)
    yk, st = layer.step(st, u[:, 300])
    assert rel(yk.float(), ry[:, 300]) < tol


@pytest.mark.parametrize("kind", ["s6", "rglru"])
def test_bf16_io_matches_f64_oracle(lrx, kind):
    m, n, B, L = (64, 16, 2, 1200) if kind == "s6" else (256, None, 2, 1500)
    layer = lrx.make_layer(kind, m, n, dtype="bf16", seed=23)
    u = torch.from_numpy(port.Rng(3).normal((B, L, m))).to("cuda", torch.bfloat16)
    gy = torch.from_numpy(port.Rng(4).normal((B, L, m))).to("cuda", torch.bfloat16)
    y, tape = layer.forward(u, tape=True)
    assert y.dtype == torch.bfloat16 and y.is_cuda
    g = lrx.layer_backward(layer, tape, gy)
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64(kind, None, params, u.float().cpu().numpy(), gy.float().cpu().numpy())
    assert rel(y, ry) < TOL["bf16"]
    assert rel(g.u, rgu) < TOL["bf16"]
    for k in rg:
        assert rel(g.params[k], rg[k]) < TOL["bf16"], (k, rel(g.params[k], rg[k]))


@pytest.mark.parametrize("key", ["real_const", "real_var", "cplx_const", "cplx_var"])
def test_scan_operator_matches_reference(lrx, key):
    z = np.load(os.path.join(GOLDEN, "scan_ops.npz"))
    a, b, x0 = z[key + ":a"], z[key + ":b"], z[key + ":x0"]
    assert rel(lrx.scan_sequential(a, b, x0), z[key + ":seq"]) < 1e-13
    assert rel(lrx.scan_parallel(a, b, x0, workers=3), z[key + ":par3"]) < 1e-13
    states, tape = lrx.scan_forward(a, b, x0)
    ga, gb, gx0 = lrx.scan_backward(tape, z[key + ":gx"])
    assert rel(ga, z[key + ":ga"]) < 1e-12
    assert rel(gb, z[key + ":gb"]) < 1e-12
    assert rel(gx0, z[key + ":gx0"]) < 1e-12
    with pytest.raises(lrx.TapeConsumed):
        lrx.scan_backward(tape, z[key + ":gx"])


@pytest.mark.parametrize("stream", ["0", "1"])  # chunked look-back / one-pass streaming walk
@pytest.mark.parametrize("dt", [np.float32, np.float64, np.complex64, np.complex128])
@pytest.mark.parametrize("L,N", [(1, 1), (2, 3), (255, 129), (4097, 300), (33, 5000)])
def test_scan_operator_sizes_vs_oracle(lrx, monkeypatch, dt, L, N, stream):
    monkeypatch.setenv("LRX_SCAN_STREAM", stream)
    rng = port.Rng(L * 7 + N)
    cplx = np.dtype(dt).kind == "c"

    def draw(shape):
        x = rng.normal(shape)
        return (x + 1j * rng.normal(shape)) if cplx else x

    for per in (False, True):
        a = (0.97 * np.exp(1j * rng.normal((L, N) if per else N)) if cplx else
             rng.uniform(-0.99, 0.99, (L, N) if per else N)).astype(dt)
        b, x0, gx = draw((L, N)).astype(dt), draw(N).astype(dt), draw((L, N)).astype(dt)
        tol = 1e-5 if np.dtype(dt) in (np.float32, np.complex64) else 1e-12
        ref = port.scan_sequential(a.astype(np.complex128 if cplx else np.float64),
                                   b.astype(np.complex128 if cplx else np.float64), x0)
        assert rel(lrx.scan_sequential(a, b, x0), ref) < tol
        st, tape = lrx.scan_forward(a, b, x0)
        ga, gb, gx0 = lrx.scan_backward(tape, gx)
        ra, rb, rx0 = port.scan_backward(a.astype(ref.dtype), ref, x0.astype(ref.dtype), gx.astype(ref.dtype))
        assert rel(gb, rb) < tol and rel(gx0, rx0) < tol and rel(ga, ra) < tol * 10


def test_known_answers(lrx):  # reference test_scan.py:19-30, 112-117, 155-160
    np.testing.assert_array_equal(lrx.scan_sequential(np.array(0.5), np.ones(3)), [1.0, 1.5, 1.75])
    np.testing.assert_array_equal(lrx.scan_sequential(np.array(0.5), np.ones(3), x0=np.array(1.0)),
                                  [1.5, 1.75, 1.875])
    out = lrx.scan_sequential(np.array([0.5]), np.zeros((4, 1)), x0=np.array([16.0]))
    np.testing.assert_array_equal(out[:, 0], [8.0, 4.0, 2.0, 1.0])
    out = lrx.scan_sequential(np.array([0.5], np.float32), np.array([[2.0]], np.float32))
    assert out.dtype == np.float32 and out[0, 0] == 2.0
    with pytest.raises(lrx.ShapeError):
        lrx.scan_sequential(np.ones(3), np.ones((10, 4)))
    with pytest.raises(lrx.ShapeError):
        lrx.scan_sequential(np.ones((9, 3)), np.ones((10, 3)))


def test_api_contract(lrx):
    layer = lrx.make_layer("lru", 2, 4, seed=3)
    u = port.Rng(4).normal((1, 8, 2))
    y, tape = layer.forward(u, tape=True)
    lrx.layer_backward(layer, tape, np.ones_like(y))
    with pytest.raises(lrx.TapeConsumed):
        lrx.layer_backward(layer, tape, np.ones_like(y))
    with pytest.raises(lrx.ShapeError):
        layer.forward(np.zeros((1, 8, 3)))
    with pytest.raises(ValueError):
        layer.forward(u, "turbo")
    with pytest.raises(ValueError):
        layer.forward(u, deltas=np.ones(8))  # LRU is discrete-time
    y, st = layer.forward(u, return_state=True)
    assert st.k == 8 and tuple(st.x.shape) == (1, 4)
    with pytest.raises(lrx.SingularBilinear):  # reference test_discretize.py:97-99
        lrx.scheme_factors("bilinear", torch.tensor([2.0 + 0j], device="cuda"), torch.tensor([1.0], device="cuda"))


def test_fault_hook_is_detected(lrx):
    from paper_2602_08810_b200 import autograd as ag
    layer = lrx.make_layer("lru", 2, 4, seed=3)
    u = port.Rng(4).normal((1, 6, 2))
    _, t1 = layer.forward(u, tape=True)
    clean = lrx.layer_backward(layer, t1, np.ones((1, 6, 2)))
    ag._grad_fault = "nu_log"
    try:
        _, t2 = layer.forward(u, tape=True)
        dirty = lrx.layer_backward(layer, t2, np.ones((1, 6, 2)))
    finally:
        ag._grad_fault = None
    np.testing.assert_allclose(dirty.params["nu_log"], 1.01 * clean.params["nu_log"], rtol=1e-12)
    np.testing.assert_array_equal(dirty.params["D"], clean.params["D"])


@pytest.mark.parametrize("kind", ["s4d", "s5", "lru", "s6", "rglru"])
def test_finite_differences_on_device(lrx, kind):  # reference test_autograd.py:238-254
    layer = lrx.make_layer(kind, 3, None if kind == "rglru" else 4, seed=31)
    u = port.Rng(32).normal((2, 10, 3))
    rep = lrx.check_layer_gradients(layer, u, rng=lrx.Rng(33))
    assert rep.passed, str(rep)


def test_native_kernels_ran(lrx):
    from paper_2602_08810_b200 import _lib
    before = _lib.launch_count()
    layer = lrx.make_layer("s6", 16, 16, dtype="f32")
    y, tape = layer.forward(np.ones((1, 5, 16), np.float32), tape=True)
    lrx.layer_backward(layer, tape, np.ones_like(y))
    assert _lib.launch_count() > before


def _s6_inputs(lrx, m, n, L, seed=5, dtype="f32"):
    from paper_2602_08810_b200.layers import _mm
    layer = lrx.make_layer("s6", m, n, dtype=dtype, seed=seed)
    g = torch.Generator(device="cuda").manual_seed(seed)
    u = torch.randn((1, L, m), generator=g, device="cuda").to(layer.io_dtype)
    gy = torch.randn((1, L, m), generator=g, device="cuda").to(layer.io_dtype)
    u2 = u.reshape(L, m)
    pre = (_mm(u2, layer.W_delta) @ layer.W_delta_proj).reshape(1, L, m)
    Bk = _mm(u2, layer.W_B.T).reshape(1, L, n)
    Ck = _mm(u2, layer.W_C.T).reshape(1, L, n)
    return layer, (u, pre, layer.b_delta, layer.a_log, Bk, Ck, layer.D), gy


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_long_sequence_parallel_matches_single_pass(lrx, dtype):
    from paper_2602_08810_b200 import ops
    from paper_2602_08810_b200.distributed import LongS6
    layer, args, gy = _s6_inputs(lrx, 64, 16, 4096, dtype=dtype)
    y_ref, ck = ops.s6_scan_fwd(*args)
    r_ref = ops.s6_scan_bwd(*args, ck, gy)
    tol = 1e-5 if dtype == "f32" else 1e-2
    for G in (1, 3):
        y, r = LongS6.simulate(G, *args, gy)
        assert rel(y, y_ref.float().cpu().numpy()) < tol
        for k in ("gu_local", "gpre", "gBk", "gCk", "ga_log", "gD", "gb_delta"):
            assert rel(r[k], r_ref[k].float().cpu().numpy()) < tol, (G, k)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_grouped_carries_match_single_pass(lrx, dtype):
    """d_state 64 (the layer default: 16-state groups) with the state carry
    x0 and the cotangent carry h_in / h_out across a sequence cut: the two
    halves stitched by their carries equal one pass (the grouped
    path used to refuse carries)."""
    from paper_2602_08810_b200 import ops
    layer, args, gy = _s6_inputs(lrx, 64, 64, 3000, dtype=dtype)
    u, pre, bd, al, Bk, Ck, D = args
    y_ref, ck = ops.s6_scan_fwd(*args)
    r_ref = ops.s6_scan_bwd(*args, ck, gy, want_h_out=True)
    c = 1234
    h0 = lambda t: t[:, :c].contiguous()  # noqa: E731
    h1 = lambda t: t[:, c:].contiguous()  # noqa: E731
    y0, ck0 = ops.s6_scan_fwd(h0(u), h0(pre), bd, al, h0(Bk), h0(Ck), D)
    y1, ck1 = ops.s6_scan_fwd(h1(u), h1(pre), bd, al, h1(Bk), h1(Ck), D, x0=ck0[:, -1].contiguous())
    r1 = ops.s6_scan_bwd(h1(u), h1(pre), bd, al, h1(Bk), h1(Ck), D, ck1, h1(gy), want_h_out=True)
    r0 = ops.s6_scan_bwd(h0(u), h0(pre), bd, al, h0(Bk), h0(Ck), D, ck0, h0(gy), h_in=r1["h_out"],
                         want_h_out=True)
    tol = 1e-5 if dtype == "f32" else 1e-2
    assert rel(torch.cat((y0, y1), 1), y_ref.float().cpu().numpy()) < tol
    for k in ("gu_local", "gpre", "gBk", "gCk"):
        assert rel(torch.cat((r0[k], r1[k]), 1), r_ref[k].float().cpu().numpy()) < tol, k
    for k in ("ga_log", "gb_delta"):
        assert rel(r0[k] + r1[k], r_ref[k].cpu().numpy()) < tol, k
    assert rel(r0["h_out"], r_ref["h_out"].cpu().numpy()) < tol


# ---- S6 v3 (TMA tiles, channel pairs, in-kernel time segments) -------------

@pytest.mark.parametrize("segs", ["1", "3", "auto"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("B,L,m", [(3, 1000, 72), (2, 37, 136), (1, 4099, 64), (2, 16, 8)])
def test_s6_segments_match_oracle(lrx, monkeypatch, segs, dtype, B, L, m):
    """Every segment count gives the f64 oracle's outputs and gradients
    (ragged L, D not a multiple of the 64-channel block)."""
    if segs == "auto":
        monkeypatch.delenv("LRX_S6_SEGS", raising=False)
    else:
        monkeypatch.setenv("LRX_S6_SEGS", segs)
    layer = lrx.make_layer("s6", m, 16, dtype=dtype, seed=41)
    io = torch.bfloat16 if dtype == "bf16" else torch.float32
    u = torch.from_numpy(port.Rng(8).normal((B, L, m))).to("cuda", io)
    gy = torch.from_numpy(port.Rng(9).normal((B, L, m))).to("cuda", io)
    y, tape = layer.forward(u, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64("s6", None, params, u.float().cpu().numpy(), gy.float().cpu().numpy())
    tol = TOL[dtype]
    assert rel(y, ry) < tol
    assert rel(g.u, rgu) < tol
    for k in rg:
        assert rel(g.params[k], rg[k]) < tol, (k, rel(g.params[k], rg[k]))


def test_s6_geometry_and_carries(lrx, monkeypatch):
    """x0 / h_in seeds, final state and h_out through the scan operator, with
    and without segments, against a split-sequence composition."""
    from paper_2602_08810_b200 import ops
    layer, args, gy = _s6_inputs(lrx, 64, 16, 2000, dtype="f32")
    u, pre, bd, al, Bk, Ck, Dk = args
    for segs in ("1", "5"):
        monkeypatch.setenv("LRX_S6_SEGS", segs)
        geo = ops.s6_geometry(u.dtype, 1, 2000, 64, 16)
        assert geo["ckpt_len"] == 8 and geo["n_seg"] == int(segs)
        y, ck = ops.s6_scan_fwd(*args)
        r = ops.s6_scan_bwd(*args, ck, gy, want_h_out=True)
        # split at t=1200: the right half continues from the left half's final state
        cut = 1200
        L_ = lambda t: t[:, :cut].contiguous()
        R_ = lambda t: t[:, cut:].contiguous()
        yl, ckl = ops.s6_scan_fwd(L_(u), L_(pre), bd, al, L_(Bk), L_(Ck), Dk)
        yr, ckr = ops.s6_scan_fwd(R_(u), R_(pre), bd, al, R_(Bk), R_(Ck), Dk, x0=ckl[:, -1].contiguous())
        assert rel(torch.cat((yl, yr), 1), y.cpu().numpy()) < 1e-5
        assert rel(ckr[:, -1], ck[:, -1].cpu().numpy()) < 1e-5
        rr = ops.s6_scan_bwd(R_(u), R_(pre), bd, al, R_(Bk), R_(Ck), Dk, ckr, R_(gy), want_h_out=True)
        rl = ops.s6_scan_bwd(L_(u), L_(pre), bd, al, L_(Bk), L_(Ck), Dk, ckl, L_(gy), h_in=rr["h_out"],
                             want_h_out=True)
        assert rel(torch.cat((rl["gpre"], rr["gpre"]), 1), r["gpre"].cpu().numpy()) < 1e-5
        assert rel(rl["h_out"], r["h_out"].cpu().numpy()) < 1e-5
        assert rel(rl["ga_log"] + rr["ga_log"], r["ga_log"].cpu().numpy()) < 1e-5


def test_s6_carry_api_matches_full_scan(lrx, monkeypatch):
    """lrx_s6_{fwd,bwd}_carry slice maps reproduce the final state / h_out."""
    from paper_2602_08810_b200 import ops
    monkeypatch.setenv("LRX_S6_SEGS", "4")
    layer, args, gy = _s6_inputs(lrx, 64, 16, 3000, dtype="bf16")
    u, pre, bd, al, Bk, Ck, Dk = args
    y, ck = ops.s6_scan_fwd(*args)
    r = ops.s6_scan_bwd(*args, ck, gy, want_h_out=True)
    x_agg, sd, ws = ops.s6_fwd_carry(u, pre, bd, al, Bk)
    assert rel(x_agg, ck[:, -1].cpu().numpy()) < 1e-5
    h_agg, sd2, _ = ops.s6_bwd_carry(gy, pre, bd, al, Ck)
    assert rel(h_agg, r["h_out"].cpu().numpy()) < 1e-5
    ref_sd = torch.nn.functional.softplus(pre.double() + bd.double()).sum(1)
    assert rel(sd, ref_sd.cpu().numpy()) < 1e-5 and rel(sd2, ref_sd.cpu().numpy()) < 1e-5
    # reusing the workspace maps gives the same result as recomputing them
    y2, ck2 = ops.s6_scan_fwd(*args, ws=ws, flags=ops.S6_REUSE_AGG)
    assert torch.equal(y2, y) and torch.equal(ck2, ck)


def test_s6_is_deterministic_with_segments(lrx, monkeypatch):
    from paper_2602_08810_b200 import ops
    monkeypatch.setenv("LRX_S6_SEGS", "6")
    layer, args, gy = _s6_inputs(lrx, 128, 16, 1500, dtype="bf16")
    outs = []
    for _ in range(2):
        y, ck = ops.s6_scan_fwd(*args)
        r = ops.s6_scan_bwd(*args, ck, gy)
        outs.append((y, r))
    assert torch.equal(outs[0][0], outs[1][0])
    for k in outs[0][1]:
        assert torch.equal(outs[0][1][k], outs[1][1][k]), k


@pytest.mark.parametrize("R,N", [(24, 2_000_000), (3, 600_004), (33, 151_552), (4096, 100), (10_000, 7),
                                 (5, 31)])
def test_reduce_rows_matches_f64_and_is_deterministic(lrx, R, N):
    """Fixed-order row reductions (every launch shape: wide float4, row-lane
    tree, two-stage) against an f64 sum; bitwise equal on a re-run."""
    from paper_2602_08810_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(R * 7 + N)
    part = torch.randn((R, N), generator=g, device="cuda")
    out = ops.reduce_rows(part, R, N)
    ref = part.double().sum(0)
    assert float((out.double() - ref).abs().max()) <= 1e-5 * max(1.0, float(ref.abs().max()))
    assert torch.equal(out, ops.reduce_rows(part, R, N))


# ---- tcgen05 3xTF32 GEMM ---------------------------------------------------

@pytest.mark.parametrize("M,N,K", [(128, 256, 256), (1000, 256, 256), (4096, 128, 256), (300, 64, 36),
                                   (131072, 256, 256), (257, 200, 64), (640, 96, 2560)])
def test_gemm_f32_tcgen05_matches_f64(lrx, M, N, K):
    from paper_2602_08810_b200 import ops
    # the tensor core's fp32 accumulation is not round-to-nearest: ~6e-8 per
    # 8-wide K step (K = 2560: 1.5e-5 measured), still far inside 1e-4
    tol = 1e-5 if K <= 1024 else 3e-5
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn((M, K), generator=g, device="cuda")
    Bt = torch.randn((N, K), generator=g, device="cuda")
    Cin = torch.randn((M, N), generator=g, device="cuda")
    cs = torch.randn(N, generator=g, device="cuda")
    ref = A.double() @ Bt.double().T
    C = ops.gemm_f32(A, Bt)
    assert rel(C, ref.cpu().numpy()) < tol
    C2 = ops.gemm_f32(A, Bt, Cin=Cin, colscale=cs, alpha=2.0)
    ref2 = 2.0 * ref + cs.double() * Cin.double()
    assert rel(C2, ref2.cpu().numpy()) < tol
    C3 = ops.gemm_f32(A, Bt, Cin=Cin, beta=-0.5)
    assert rel(C3, (ref - 0.5 * Cin.double()).cpu().numpy()) < tol


@pytest.mark.parametrize("K,M,N", [(4096, 256, 256), (131072, 256, 256), (1000, 128, 64), (77, 64, 192),
                                   (8192, 128, 128), (1 << 20, 64, 64)])
def test_gemm_f32_tn_tcgen05_matches_f64(lrx, K, M, N):
    from paper_2602_08810_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(K + M + N)
    A = torch.randn((K, M), generator=g, device="cuda")
    B = torch.randn((K, N), generator=g, device="cuda")
    ref = (A.double().T @ B.double()) * 1.5
    C = ops.gemm_f32_tn(A, B, alpha=1.5)
    # bar 3e-5: the tensor core's fp32 accumulation is not round-to-nearest, so
    # the error grows with the K span one CTA accumulates in TMEM (measured for
    # K = 131072 over 148 CTAs: 1.25e-5; 296 CTAs: 7e-6 at +30% time).  Still
    # 3x inside the 1e-4 parity bar; a 1xTF32 GEMM would be ~1e-3.
    assert rel(C, ref.cpu().numpy()) < 3e-5
    C2 = ops.gemm_f32_tn(A, B, alpha=1.5)
    assert torch.equal(C, C2)  # deterministic split-K


@pytest.mark.parametrize("n", [16, 64])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_s6_layer_delta_epilogue_matches_oracle(lrx, monkeypatch, n, dtype):
    """S6 layer with >= 4096 tokens: delta = softplus(p1 W_delta_proj + b_delta)
    in the tcgen05 GEMM epilogue and the scan in delta-input mode
    (LRX_S6_DELTA_IN; sigmoid(pre) = 1 - exp(-delta) in the backward) against
    the oracle -- and against the pre-activation path (LRX_S6_DELTA_IN=0)."""
    m, B, L = 256, 2, 2500  # d_rank 16: the delta GEMM's K qualifies for the tensor cores
    layer = lrx.make_layer("s6", m, n, dtype=dtype, seed=81)
    u = torch.from_numpy(port.Rng(82).normal((B, L, m))).to("cuda", layer.io_dtype)
    gy = torch.from_numpy(port.Rng(83).normal((B, L, m))).to("cuda", layer.io_dtype)
    y, tape = layer.forward(u, tape=True)
    assert tape._saved["flags"] == 2
    g = lrx.layer_backward(layer, tape, gy)
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64("s6", None, params, u.float().cpu().numpy(), gy.float().cpu().numpy())
    tol = TOL[dtype]
    assert rel(y, ry) < tol
    assert rel(g.u, rgu) < tol
    for k in rg:
        assert rel(g.params[k], rg[k]) < tol, (k, rel(g.params[k], rg[k]))
    monkeypatch.setenv("LRX_S6_DELTA_IN", "0")
    y0, tape0 = layer.forward(u, tape=True)
    assert tape0._saved["flags"] == 0
    assert rel(y, y0.float().cpu().numpy()) < (1e-5 if dtype == "f32" else 1e-2)


@pytest.mark.parametrize("n", [0, 5, 8, 1003, 1 << 20])
def test_cast_matches_torch_bitwise(lrx, n):
    """lrx_cast (bf16 <-> fp32 planes, ragged tail) gives torch's conversion bits."""
    from paper_2602_08810_b200 import ops
    x = torch.randn(n, device="cuda") * 3
    b = ops.cast(x, torch.bfloat16)
    assert b.dtype == torch.bfloat16 and torch.equal(b, x.to(torch.bfloat16))
    f = ops.cast(b, torch.float32)
    assert f.dtype == torch.float32 and torch.equal(f, b.float())


@pytest.mark.parametrize("M,N,K", [(131072, 128, 1536), (4096, 16, 1536), (1000, 96, 72), (300, 256, 64),
                                   (5, 32, 8), (2049, 300, 264)])
def test_gemm_bf16_tcgen05_matches_fp64(lrx, M, N, K):
    """bf16 tcgen05 GEMM (kind::f16, fp32 accumulation) with its fused epilogue
    (bias + identity / softplus / sigmoid, + beta Cin) against an fp64 GEMM of
    the same bf16-rounded operands.  The products are exact in fp32, so only
    the accumulation rounds: bar 1e-5."""
    from paper_2602_08810_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = (0.5 * torch.randn((M, K), generator=g, device="cuda")).to(torch.bfloat16)
    Bt = (torch.randn((N, K), generator=g, device="cuda") / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, generator=g, device="cuda")
    Cin = torch.randn((M, N), generator=g, device="cuda")
    ref = A.double() @ Bt.double().T
    assert rel(ops.gemm_bf16(A, Bt), ref.cpu().numpy()) < 1e-5
    pre = 1.5 * ref + bias.double()
    sp = torch.where(pre > 30, pre, torch.log1p(torch.exp(pre.clamp(max=30))))
    got = ops.gemm_bf16(A, Bt, bias=bias, act=ops.ACT_SOFTPLUS, alpha=1.5)
    assert rel(got, sp.cpu().numpy()) < 1e-5
    got = ops.gemm_bf16(A, Bt, bias=bias, act=ops.ACT_SIGMOID, Cin=Cin, beta=-0.5)
    want = torch.sigmoid(ref + bias.double()) - 0.5 * Cin.double()
    assert rel(got, want.cpu().numpy()) < 1e-5
    assert torch.equal(ops.gemm_bf16(A, Bt), ops.gemm_bf16(A, Bt))
    # bf16 output (RG-LRU gate pre-activations; 16-byte rows: N % 8 == 0): the fp32 result rounded once
    if N % 8:
        with pytest.raises(ValueError):
            ops.gemm_bf16(A, Bt, out_dtype=torch.bfloat16)
        return
    got16 = ops.gemm_bf16(A, Bt, bias=bias, act=ops.ACT_SIGMOID, out_dtype=torch.bfloat16)
    assert got16.dtype == torch.bfloat16
    assert torch.equal(got16, ops.gemm_bf16(A, Bt, bias=bias, act=ops.ACT_SIGMOID).to(torch.bfloat16))


@pytest.mark.parametrize("n", [8, 16, 32, 64])
@pytest.mark.parametrize("scheme", ["zoh", "bilinear", "dirac"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_s4d_fused_kernel_matches_oracle(lrx, n, scheme, dtype):
    """The fused S4D kernel (d_state in {8, 16, 32, 64}, ragged L) against the
    oracle; prefill state and the kernel's launch are checked too."""
    from paper_2602_08810_b200 import _lib
    m, B, L = 12, 3, 301
    layer = lrx.make_layer("s4d", m, n, scheme, dtype=dtype, seed=61)
    u = port.Rng(62).normal((B, L, m)).astype(layer.rdt)
    gy = port.Rng(63).normal((B, L, m)).astype(layer.rdt)
    before = _lib.launch_count()
    y, tape = layer.forward(u, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    assert _lib.launch_count() > before
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64("s4d", scheme, params, u, gy)
    tol = TOL[dtype]
    assert rel(y, ry) < tol
    assert rel(g.u, rgu) < tol
    for k in rg:
        assert rel(g.params[k], rg[k]) < tol, (k, rel(g.params[k], rg[k]))
    # prefill -> decode continues from the fused kernel's final state
    _, st = layer.forward(u[:, :200], return_state=True)
    for k in range(200, 204):
        yk, st = layer.step(st, u[:, k])
        assert rel(yk, ry[:, k]) < tol


@pytest.mark.parametrize("n", [8, 32, 64])
@pytest.mark.parametrize("scheme", ["zoh", "bilinear", "dirac"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_s4d_async_fused_matches_oracle(lrx, n, scheme, dtype):
    """Asynchronous S4D (per-step deltas [B, L], layers.py:402-440) on the
    fused kernel: abar_k / scale_k discretised in the kernel, the coefficient
    gradients through the scheme partials accumulated per lane (no [B, L, m, n]
    planes) -- against the oracle, every parameter gradient."""
    m, B, L = 6, 2, 203
    layer = lrx.make_layer("s4d", m, n, scheme, asynchronous=True, dtype=dtype, seed=64)
    u = port.Rng(65).normal((B, L, m)).astype(layer.rdt)
    gy = port.Rng(66).normal((B, L, m)).astype(layer.rdt)
    deltas = port.Rng(67).uniform(0.1, 3.0, (B, L)).astype(layer.rdt)
    y, tape = layer.forward(u, deltas=deltas, tape=True)
    assert tape._saved.get("fused")
    g = lrx.layer_backward(layer, tape, gy)
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64("s4d", scheme, params, u, gy, deltas=deltas, asyn=True)
    tol = TOL[dtype]
    assert rel(y, ry) < tol
    assert rel(g.u, rgu) < tol
    for k in rg:
        assert rel(g.params[k], rg[k]) < tol, (k, rel(g.params[k], rg[k]))


@pytest.mark.parametrize("seg", ["16", "auto"])
@pytest.mark.parametrize("scheme", ["zoh", "bilinear", "dirac"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_s5_async_fused_matches_oracle(lrx, monkeypatch, seg, scheme, dtype):
    """Asynchronous S5 (per-step deltas, layers.py:650-658): the MIMO scan
    discretises every step in the kernel and accumulates the coefficient
    gradients through the scheme partials -- against the oracle, every
    parameter gradient, with forced short segments too."""
    if seg != "auto":
        monkeypatch.setenv("LRX_MIMO_SEG", seg)
    m, B, L = 8, 3, 157
    layer = lrx.make_layer("s5", m, 12, scheme, asynchronous=True, dtype=dtype, seed=72)
    u = port.Rng(73).normal((B, L, m)).astype(layer.rdt)
    gy = port.Rng(74).normal((B, L, m)).astype(layer.rdt)
    deltas = port.Rng(75).uniform(0.05, 3.0, (B, L)).astype(layer.rdt)
    y, tape = layer.forward(u, deltas=deltas, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64("s5", scheme, params, u, gy, deltas=deltas, asyn=True)
    tol = TOL[dtype]
    assert rel(y, ry) < tol
    assert rel(g.u, rgu) < tol
    for k in rg:
        assert rel(g.params[k], rg[k]) < tol, (k, rel(g.params[k], rg[k]))


@pytest.mark.parametrize("segs", ["1", "3", "auto"])
@pytest.mark.parametrize("asyn", [False, True])
def test_s4d_time_segments_match_oracle(lrx, monkeypatch, segs, asyn):
    """Fused S4D with the sequence cut into time segments (aggregate maps
    folded in a fixed order; ragged last segment), constant and per-step
    steps, against the oracle; a re-run gives the same bits."""
    if segs != "auto":
        monkeypatch.setenv("LRX_S4D_SEGS", segs)
    m, B, L, n = 3, 1, 1000, 16
    layer = lrx.make_layer("s4d", m, n, "zoh", asynchronous=asyn, dtype="f64", seed=68)
    u = port.Rng(69).normal((B, L, m))
    gy = port.Rng(70).normal((B, L, m))
    deltas = port.Rng(71).uniform(0.1, 2.0, (B, L)) if asyn else None
    y, tape = layer.forward(u, deltas=deltas, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    y2, tape2 = layer.forward(u, deltas=deltas, tape=True)
    g2 = lrx.layer_backward(layer, tape2, gy)
    assert np.array_equal(y, y2) and np.array_equal(g.u, g2.u)
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64("s4d", "zoh", params, u, gy, deltas=deltas, asyn=asyn)
    assert rel(y, ry) < 1e-10
    assert rel(g.u, rgu) < 1e-10
    for k in rg:
        assert rel(g.params[k], rg[k]) < 1e-10, (segs, k)
    _, st = layer.forward(u, deltas=deltas, return_state=True)
    xl = st.x.cpu().numpy()
    assert np.isfinite(xl).all()


@pytest.mark.parametrize("seg", ["16", "128", "1024"])
def test_mimo_segment_lengths_match_oracle(lrx, monkeypatch, seg):
    """MIMO scans with forced segment lengths (LRX_MIMO_SEG; ragged last one)."""
    monkeypatch.setenv("LRX_MIMO_SEG", seg)
    layer = lrx.make_layer("s5", 16, 24, dtype="f32", seed=51)
    u = port.Rng(52).normal((3, 1000, 16)).astype(np.float32)
    gy = port.Rng(53).normal((3, 1000, 16)).astype(np.float32)
    y, tape = layer.forward(u, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64("s5", layer.discretization, params, u, gy)
    assert rel(y, ry) < TOL["f32"]
    assert rel(g.u, rgu) < TOL["f32"]
    for k in rg:
        assert rel(g.params[k], rg[k]) < TOL["f32"], (seg, k)


@pytest.mark.parametrize("kind", ["s5", "lru"])
def test_mimo_layer_on_tensor_cores_matches_oracle(lrx, kind):
    """B*L = 32768 tokens: the projections run on the tcgen05 3xTF32 GEMMs."""
    from paper_2602_08810_b200 import _lib
    m, n, B, L = 64, 64, 8, 4096
    layer = lrx.make_layer(kind, m, n, dtype="f32", seed=19)
    u = port.Rng(11).normal((B, L, m)).astype(np.float32)
    gy = port.Rng(12).normal((B, L, m)).astype(np.float32)
    before = _lib.launch_count()
    y, tape = layer.forward(u, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    assert _lib.launch_count() - before >= 8  # 4 projection GEMMs + 2 reductions + scans
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64(kind, layer.discretization, params, u, gy)
    assert rel(y, ry) < TOL["f32"]
    assert rel(g.u, rgu) < TOL["f32"]
    for k in rg:
        assert rel(g.params[k], rg[k]) < TOL["f32"], (k, rel(g.params[k], rg[k]))


@pytest.mark.parametrize("bwd", ["fused", "separate"])
@pytest.mark.parametrize("kind,m,n,B,L", [("s5", 64, 256, 5, 1000), ("lru", 48, 64, 2, 4096),
                                          ("s5", 128, 64, 40, 128), ("lru", 32, 128, 1, 8192)])
def test_mimo_gemm_scan_fused_matches_oracle(lrx, monkeypatch, kind, m, n, B, L, bwd):
    """The fused projection + scan kernels (bu / gx scanned straight out of
    TMEM, csrc/lrx_mimo_fused.cu): ragged last unit (L = 1000), P = 128 (s5
    d_state 256), zero-padded state rows (P < 128), one batch row of 64 units;
    the backward fused or separate (no bu stored: d scale from the weight
    GEMM).  Oracle in f64, all parameter gradients, same bits on a re-run."""
    from paper_2602_08810_b200 import ops
    monkeypatch.setenv("LRX_MIMO_FUSED", "1")
    monkeypatch.setenv("LRX_MIMO_FUSED_BWD", "1" if bwd == "fused" else "0")
    calls = []
    for name in ("mimo_fused_fwd", "mimo_fused_bwd"):
        f = getattr(ops, name)
        monkeypatch.setattr(ops, name, (lambda f, nm: lambda *a, **k: (calls.append(nm), f(*a, **k))[1])(f, name))
    layer = lrx.make_layer(kind, m, n, dtype="f32", seed=23)
    u = port.Rng(31).normal((B, L, m)).astype(np.float32)
    gy = port.Rng(32).normal((B, L, m)).astype(np.float32)
    y, tape = layer.forward(u, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    assert calls == (["mimo_fused_fwd", "mimo_fused_bwd"] if bwd == "fused" else ["mimo_fused_fwd"])
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64(kind, layer.discretization, params, u, gy)
    assert rel(y, ry) < TOL["f32"]
    assert rel(g.u, rgu) < TOL["f32"]
    for k in rg:
        assert rel(g.params[k], rg[k]) < TOL["f32"], (k, rel(g.params[k], rg[k]))
    y2, tape2 = layer.forward(u, tape=True)
    g2 = lrx.layer_backward(layer, tape2, gy)
    assert np.array_equal(np.asarray(y), np.asarray(y2)) and np.array_equal(np.asarray(g.u), np.asarray(g2.u))
    for k in g.params:
        assert torch.equal(torch.as_tensor(g.params[k]), torch.as_tensor(g2.params[k])), k


def test_mimo_fused_concurrent_streams_match_sequential(lrx, monkeypatch):
    """Two fused projection + scan forwards+backwards on two streams at once:
    units are claimed dynamically, so kernels sharing the GPU cannot wait on
    each other's unlaunched CTAs; results equal the sequential ones bitwise."""
    monkeypatch.setenv("LRX_MIMO_FUSED", "1")
    monkeypatch.setenv("LRX_MIMO_FUSED_BWD", "1")
    layer = lrx.make_layer("s5", 64, 128, dtype="f32", seed=5)
    us = [torch.from_numpy(port.Rng(60 + i).normal((6, 2048, 64)).astype(np.float32)).cuda() for i in range(2)]
    gys = [torch.from_numpy(port.Rng(70 + i).normal((6, 2048, 64)).astype(np.float32)).cuda() for i in range(2)]

    def run(i):
        y, tape = layer.forward(us[i], tape=True)
        g = lrx.layer_backward(layer, tape, gys[i])
        return y, g.u

    ref = [run(0), run(1)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    out = [None, None]
    for _ in range(3):
        for i, st in enumerate(streams):
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                out[i] = run(i)
        torch.cuda.synchronize()
        for i in range(2):
            assert torch.equal(out[i][0], ref[i][0]) and torch.equal(out[i][1], ref[i][1])


@pytest.mark.parametrize("mode", ["tma", "stream", "lookback", "rc", "rev"])
def test_rglru_kernel_variants_match_oracle(lrx, monkeypatch, mode):
    """Every RG-LRU kernel family (LRX_RGLRU_MODE) gives the oracle's answer."""
    monkeypatch.setenv("LRX_RGLRU_MODE", mode)
    m, B, L = 96, 3, 777
    layer = lrx.make_layer("rglru", m, dtype="f32", seed=29)
    u = port.Rng(13).normal((B, L, m)).astype(np.float32)
    gy = port.Rng(14).normal((B, L, m)).astype(np.float32)
    y, tape = layer.forward(u, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64("rglru", None, params, u, gy)
    assert rel(y, ry) < TOL["f32"]
    assert rel(g.u, rgu) < TOL["f32"]
    for k in rg:
        assert rel(g.params[k], rg[k]) < TOL["f32"], (mode, k)


@pytest.mark.parametrize("segs", ["1", "2", "5", "64"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("mode", ["tma", "rev"])
def test_rglru_time_segments_match_oracle(lrx, monkeypatch, segs, dtype, mode):
    """Segmented TMA passes (LRX_RGLRU_SEGS; ragged last segment) give the
    oracle's answer, and the same bits on a second run (y-streaming and
    reverse-reconstruction backward)."""
    monkeypatch.setenv("LRX_RGLRU_MODE", mode)
    monkeypatch.setenv("LRX_RGLRU_SEGS", segs)
    m, B, L = 64, 2, 1000 if dtype == "f32" else 517
    layer = lrx.make_layer("rglru", m, dtype=dtype, seed=37)
    io = torch.bfloat16 if dtype == "bf16" else torch.float32
    u = torch.from_numpy(port.Rng(15).normal((B, L, m))).to("cuda", io)
    gy = torch.from_numpy(port.Rng(16).normal((B, L, m))).to("cuda", io)
    y, tape = layer.forward(u, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    y2, tape2 = layer.forward(u, tape=True)
    g2 = lrx.layer_backward(layer, tape2, gy)
    assert torch.equal(y, y2) and torch.equal(g.u, g2.u)
    params = {k: v.cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu = _oracle_f64("rglru", None, params, u.float().cpu().numpy(), gy.float().cpu().numpy())
    tol = TOL[dtype]
    assert rel(y, ry) < tol
    assert rel(g.u, rgu) < tol
    for k in rg:
        assert rel(g.params[k], rg[k]) < tol, (segs, k)


# ---- step mode (decode), reference test_layers.py:277-315 -------------------

STEP_KINDS = [("s4d", 4), ("s5", 8), ("lru", 4), ("s6", 4), ("rglru", None)]


@pytest.mark.parametrize("kind,n", STEP_KINDS)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_step_matches_forward(lrx, kind, n, dtype):
    m, B, L = 6, 2, 40
    layer = lrx.make_layer(kind, m, n, dtype=dtype, seed=41)
    u = port.Rng(42).normal((B, L, m)).astype(layer.rdt)
    ref = layer.forward(u)
    st = layer.init_state(B)
    tol = 1e-10 if dtype == "f64" else 1e-4
    for k in range(L):
        yk, st = layer.step(st, u[:, k])
        assert isinstance(yk, np.ndarray) and yk.shape == (B, m)
        assert rel(yk, ref[:, k]) < tol, (k, rel(yk, ref[:, k]))
    assert st.k == L
    # prefill half with forward(return_state=True), decode the rest
    _, st2 = layer.forward(u[:, :L // 2], return_state=True)
    assert st2.k == L // 2
    for k in range(L // 2, L):
        yk, st2 = layer.step(st2, u[:, k])
        assert rel(yk, ref[:, k]) < tol


@pytest.mark.parametrize("kind,n", STEP_KINDS)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_step_graph_matches_eager_steps(lrx, kind, n, dtype):
    """StepGraph (CUDA-graph decode) gives the eager step's bits and the
    forward's values; prefill via forward(return_state=True) then decode."""
    if dtype == "bf16" and kind not in ("s6", "rglru"):
        pytest.skip("bf16 I/O exists for S6 / RG-LRU only")
    m, B, L = 32, 3, 24
    layer = lrx.make_layer(kind, m, n, dtype=dtype, seed=45)
    u = torch.from_numpy(port.Rng(46).normal((B, L, m))).to("cuda", layer.io_dtype)
    ref = layer.forward(u).float().cpu().numpy()
    st_e, st_g = layer.init_state(B), layer.init_state(B)
    g = layer.step_graph(st_g)
    for k in range(L):
        ye, st_e = layer.step(st_e, u[:, k])
        yg = g.step(u[:, k])
        assert torch.equal(ye, yg), k
        assert rel(yg.float(), ref[:, k]) < TOL[dtype]
    assert st_g.k == L and torch.equal(st_e.x, st_g.x)
    _, st2 = layer.forward(u[:, :L // 2], return_state=True)
    ys = layer.step_graph(st2).run(u[:, L // 2:])
    assert rel(ys.float(), ref[:, L // 2:]) < TOL[dtype]


@pytest.mark.parametrize("kind", ["s6", "rglru"])
def test_step_bf16_and_device_tensors(lrx, kind):
    m, B, L = 64, 2, 50
    layer = lrx.make_layer(kind, m, 16 if kind == "s6" else None, dtype="bf16", seed=43)
    u = torch.from_numpy(port.Rng(44).normal((B, L, m))).to("cuda", torch.bfloat16)
    ref = layer.forward(u).float()
    st = layer.init_state(B)
    for k in range(L):
        yk, st = layer.step(st, u[:, k])
        assert yk.is_cuda and yk.dtype == torch.bfloat16
        assert rel(yk, ref[:, k].cpu().numpy()) < 1e-2


def test_step_api_contract(lrx):  # reference test_layers.py:277-303
    layer = lrx.make_layer("lru", 2, d_state=4, seed=1)
    u = port.Rng(2).normal((1, 10, 2))
    ref = layer.forward(u)
    s1, s2 = layer.init_state(1), layer.init_state(1)
    for k in range(10):
        y1, s1 = layer.step(s1, u[:, k])
        layer.step(s2, port.Rng(k).normal((1, 2)))  # unrelated traffic
        np.testing.assert_allclose(y1, ref[:, k], atol=1e-12)
    assert s1.k == 10
    rg = lrx.make_layer("rglru", 3, seed=4)
    st = rg.init_state(1)
    y, st = rg.step(st, np.zeros(3))
    assert y.shape == (3,)
    with pytest.raises(lrx.ShapeError):
        rg.step(st, np.zeros((2, 3)))
    with pytest.raises(ValueError):
        rg.step(st, np.zeros(3), delta_k=0.5)
    s4 = lrx.make_layer("s4d", 2, d_state=2, discretization="zoh")
    with pytest.raises(NotImplementedError):
        s4.step(s4.init_state(1), np.zeros((1, 2)), delta_k=0.5)
    y, st = lrx.layer_step(rg, rg.init_state(1), np.zeros((1, 3)))
    assert y.shape == (1, 3)


@pytest.mark.parametrize("kind", ["s4d", "s5"])
def test_async_step_matches_batched_forward(lrx, kind):  # reference test_layers.py:305-315
    layer = lrx.make_layer(kind, 2, d_state=4, asynchronous=True, seed=6)
    u = port.Rng(7).normal((1, 12, 2))
    deltas = port.Rng(8).uniform(0.2, 2.0, 12)
    ref = layer.forward(u, deltas=deltas)
    st = layer.init_state(1)
    for k in range(12):
        yk, st = layer.step(st, u[:, k], delta_k=deltas[k])
        np.testing.assert_allclose(yk, ref[:, k], atol=1e-12)


def test_scan_step_operator(lrx):  # reference test_scan.py:133-146
    rng = port.Rng(5)
    a = 0.9 * np.exp(1j * rng.normal(5))
    bs = rng.normal((7, 5)) + 1j * rng.normal((7, 5))
    ref = port.scan_sequential(a, bs, None)
    st = lrx.init_step_state((5,), np.complex128)
    for k in range(7):
        xk, st = lrx.step(st, a, bs[k])
        np.testing.assert_allclose(xk.cpu().numpy(), ref[k], atol=1e-12)
    assert st.k == 7
    st = lrx.init_step_state((4,), np.float64)
    with pytest.raises(lrx.ShapeError):
        lrx.step(st, np.ones(3), np.ones(3))
    # lane-periodic, scalar and leading-singleton operands against numpy broadcasting
    st = lrx.init_step_state((3, 4), np.float32, x0=np.arange(12, dtype=np.float32).reshape(3, 4))
    x = np.arange(12, dtype=np.float64).reshape(3, 4)
    for a_k, b_k in ((np.full(4, 0.5), np.float64(2.0)), (np.float64(0.25), np.ones((1, 4))),
                     (np.full((3, 1), 0.5), np.ones((3, 4)))):
        xk, st = lrx.step(st, a_k, b_k)
        x = a_k * x + b_k
        np.testing.assert_allclose(xk.cpu().numpy(), x, rtol=1e-6)


@pytest.mark.parametrize("kind,n", STEP_KINDS)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_step_matches_oracle_loop(lrx, kind, n, dtype):
    """Step mode pinned directly to the oracle's independent per-step loop
    (port.naive_forward, the restatement of test_layers.py:21-87) rather than
    to this package's forward; async steps for the kinds that take them."""
    m, B, L = 6, 2, 30
    asyn = kind in ("s4d", "s5")
    layer = lrx.make_layer(kind, m, n, dtype=dtype, seed=47, asynchronous=asyn,
                           **({"discretization": "dirac"} if asyn else {}))
    u = port.Rng(48).normal((B, L, m)).astype(layer.rdt)
    deltas = port.Rng(49).uniform(0.2, 2.0, L) if asyn else None
    params = {k: np.asarray(v.cpu().numpy() if isinstance(v, torch.Tensor) else v, np.float64)
              for k, v in layer.parameters().items()}
    ref = port.naive_forward(kind, params, u.astype(np.float64), scheme=layer.discretization,
                             deltas=None if deltas is None else np.broadcast_to(deltas, (B, L)))
    st = layer.init_state(B)
    tol = 1e-10 if dtype == "f64" else 1e-4
    for k in range(L):
        yk, st = layer.step(st, u[:, k], **({"delta_k": float(deltas[k])} if asyn else {}))
        assert rel(yk, ref[:, k]) < tol, (k, rel(yk, ref[:, k]))
