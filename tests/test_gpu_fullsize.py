"""Parity at BASELINE.json's full sizes (configs C1-C5), where the f64 oracle
cannot run the whole problem: size-independent properties plus oracle spot
checks on independent lanes over the full sequence length.

  * oracle spot check: the lanes of a few channels (all batch rows, the whole
    L) go through oracle/port.py's scan-level restatements (rglru_scan,
    s6_scan: layers.py:1208-1291, 1041-1118) or its layer restatement; errors
    max|d| / max|ref| within the north_star tolerances.
  * linearity in u at fixed gates / projections (the scan is linear in its
    input: y(u1 + 2 u2) = y(u1) + 2 y(u2)) and the adjoint identity
    <gy, J u2> = <J^T gy, u2> between the forward and the backward kernels.
  * bitwise determinism of a re-run (test_acceptance.py:249-250).
The big configs need ~100 GB of HBM (B200: 180 GB)."""
import numpy as np
import pytest
import torch

from oracle import port

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lrx():
    import paper_2602_08810_b200 as m
    return m


@pytest.fixture(autouse=True)
def _free():
    yield
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def rel(got, ref):
    got = got.detach().double().cpu().numpy() if isinstance(got, torch.Tensor) else got
    return port.rel_err(got, ref)


def randn(shape, seed, dtype=torch.float32):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(shape, generator=g, device="cuda", dtype=torch.float32).to(dtype)


def dot(a, b):
    return float((a.double() * b.double()).sum())


def adjoint_gap(gy, y2, gu, u2):
    """|<gy, J u2> - <J^T gy, u2>| relative to |gy| |J u2|."""
    lhs, rhs = dot(gy, y2), dot(gu, u2)
    return abs(lhs - rhs) / (float(gy.double().norm()) * float(y2.double().norm()))


def test_rglru_c4_full_size(lrx):
    """C4: RG-LRU B=64 L=16384 W=2560 fp32 (the bench workload)."""
    from paper_2602_08810_b200 import ops
    B, L, W = 64, 16384, 2560
    layer = lrx.make_layer("rglru", W, dtype="f32", seed=0)
    p = (layer.lambda_param, layer.b_r, layer.b_i)
    u, qr, qi, gy = (randn((B, L, W), s) for s in (1, 2, 3, 4))
    y, ck = ops.rglru_scan_fwd(u, qr, qi, *p)
    r = ops.rglru_scan_bwd(u, qr, qi, *p, ck, gy, y=y)
    # oracle: 5 channels (incl. the most contracting one, where the backward's
    # state reconstruction expands rounding the most), every batch row, the
    # whole sequence
    worst = int(torch.argmin(layer.lambda_param))
    cols = torch.tensor([0, 777, 1500, W - 1, worst], device="cuda")
    sl = lambda t: t.index_select(2, cols).double().cpu().numpy()  # noqa: E731
    pn = [t.index_select(0, cols).double().cpu().numpy() for t in p]
    ry, rg = port.rglru_scan(sl(u), sl(qr), sl(qi), *pn, sl(gy))
    assert rel(y.index_select(2, cols), ry) < 1e-4
    for k in ("gu_local", "gqr", "gqi"):
        assert rel(r[k].index_select(2, cols), rg[k]) < 1e-4, k
    for k, o in (("gla", "gla"), ("gb_r", "gb_r"), ("gb_i", "gb_i")):
        assert rel(r[k].index_select(0, cols), rg[o]) < 1e-4, k
    # determinism
    y_again, _ = ops.rglru_scan_fwd(u, qr, qi, *p)
    assert torch.equal(y, y_again)
    del y_again, ck, r["gqr"], r["gqi"]
    # linearity in u (gates fixed) and the adjoint identity on the u path
    gu = r["gu_local"]
    u2 = randn((B, L, W), 5)
    y2, _ = ops.rglru_scan_fwd(u2, qr, qi, *p)
    assert adjoint_gap(gy, y2, gu, u2) < 1e-5
    u.add_(u2, alpha=2.0)
    y12, _ = ops.rglru_scan_fwd(u, qr, qi, *p)
    y.add_(y2, alpha=2.0)
    assert float((y12 - y).abs().max()) / float(y.abs().max()) < 1e-5


@pytest.mark.parametrize("B", [32, 16, 8, 4])
def test_rglru_per_rank_shares_match_oracle(lrx, B):
    """The per-rank batch shares of an N-GPU C4 job (B = 64/N, W = 2560):
    each lane count takes its own plan (B = 32: tile height 4 capped by the
    occupancy check, 3-stage ring; B = 16: 8 / 16; B <= 8: time segments).
    Oracle on 4 channels x every row at L = 2048 (plans depend on the lane
    count, not on L, except the segment count, capped at L / 256 = 8)."""
    from paper_2602_08810_b200 import ops
    L, W = 2048, 2560
    layer = lrx.make_layer("rglru", W, dtype="f32", seed=3)
    p = (layer.lambda_param, layer.b_r, layer.b_i)
    u, qr, qi, gy = (randn((B, L, W), s) for s in (11, 12, 13, 14))
    y, ck = ops.rglru_scan_fwd(u, qr, qi, *p)
    r = ops.rglru_scan_bwd(u, qr, qi, *p, ck, gy, y=y)
    cols = torch.tensor([0, 1281, W - 2, int(torch.argmin(layer.lambda_param))], device="cuda")
    sl = lambda t: t.index_select(2, cols).double().cpu().numpy()  # noqa: E731
    pn = [t.index_select(0, cols).double().cpu().numpy() for t in p]
    ry, rg = port.rglru_scan(sl(u), sl(qr), sl(qi), *pn, sl(gy))
    assert rel(y.index_select(2, cols), ry) < 1e-4
    for k in ("gu_local", "gqr", "gqi"):
        assert rel(r[k].index_select(2, cols), rg[k]) < 1e-4, k
    for k in ("gla", "gb_r", "gb_i"):
        assert rel(r[k].index_select(0, cols), rg[k]) < 1e-4, k


def test_rglru_c4_bf16_full_size(lrx):
    """C4 shape with bf16 I/O (the optional dtype): the backward reconstructs
    the fp32 states anchored on the forward's checkpoints (y is rounded, so it
    is never read); oracle spot check on 4 channels with the bf16-rounded
    inputs."""
    from paper_2602_08810_b200 import ops
    B, L, W = 64, 16384, 2560
    layer = lrx.make_layer("rglru", W, dtype="f32", seed=0)
    p = (layer.lambda_param, layer.b_r, layer.b_i)
    u, qr, qi, gy = (randn((B, L, W), s, torch.bfloat16) for s in (6, 7, 8, 9))
    y, ck = ops.rglru_scan_fwd(u, qr, qi, *p)
    r = ops.rglru_scan_bwd(u, qr, qi, *p, ck, gy)  # no y: the bf16 state is rounded
    cols = torch.tensor([3, 1024, W - 2, W - 1], device="cuda")
    sl = lambda t: t.index_select(2, cols).double().cpu().numpy()  # noqa: E731
    pn = [t.index_select(0, cols).double().cpu().numpy() for t in p]
    ry, rg = port.rglru_scan(sl(u), sl(qr), sl(qi), *pn, sl(gy))
    assert rel(y.index_select(2, cols), ry) < 1e-2
    for k in ("gu_local", "gqr", "gqi"):
        assert rel(r[k].index_select(2, cols), rg[k]) < 1e-2, k
    for k in ("gla", "gb_r", "gb_i"):
        assert rel(r[k].index_select(0, cols), rg[k]) < 1e-2, k


@pytest.mark.parametrize("io", ["bf16", "f32"])
def test_s6_c3_full_size(lrx, io):
    """C3: S6 B=16 L=8192 D=1536 N=16 (bf16 I/O as configured; f32 I/O for the
    exact linearity / adjoint checks)."""
    from paper_2602_08810_b200 import ops
    B, L, D, N = 16, 8192, 1536, 16
    layer = lrx.make_layer("s6", D, N, dtype="f32", seed=0)
    iod = torch.bfloat16 if io == "bf16" else torch.float32
    u = randn((B, L, D), 11, iod)
    gy = randn((B, L, D), 12, iod)
    pre = randn((B, L, D), 13) * 0.5 - 2.0
    Bk, Ck = randn((B, L, N), 14), randn((B, L, N), 15)
    p = (layer.b_delta, layer.a_log)
    y, ck = ops.s6_scan_fwd(u, pre, *p, Bk, Ck, layer.D)
    r = ops.s6_scan_bwd(u, pre, *p, Bk, Ck, layer.D, ck, gy)
    tol = 1e-2 if io == "bf16" else 1e-4
    cols = torch.tensor([0, 701, D - 1], device="cuda")
    sl = lambda t: t.index_select(2, cols).double().cpu().numpy()  # noqa: E731
    ry, rg = port.s6_scan(sl(u), sl(pre), layer.b_delta.index_select(0, cols).double().cpu().numpy(),
                          layer.a_log.index_select(0, cols).double().cpu().numpy(), Bk.double().cpu().numpy(),
                          Ck.double().cpu().numpy(), layer.D.index_select(0, cols).double().cpu().numpy(), sl(gy))
    assert rel(y.index_select(2, cols), ry) < tol
    for k in ("gu_local", "gpre"):
        assert rel(r[k].index_select(2, cols), rg[k]) < tol, k
    for k in ("ga_log", "gD", "gb_delta"):
        assert rel(r[k].index_select(0, cols), rg[k]) < tol, k
    # the channel sums gB_k / gC_k (layers.py:1080, 1098) of batch row 0 over
    # all 1536 channels and the whole sequence, oracle in channel blocks
    gbk, gck = np.zeros((1, L, N)), np.zeros((1, L, N))
    row = lambda t, hs: t[:1, :, hs].double().cpu().numpy()  # noqa: E731
    Bk0, Ck0 = Bk[:1].double().cpu().numpy(), Ck[:1].double().cpu().numpy()
    for h0 in range(0, D, 256):
        hs = slice(h0, h0 + 256)
        _, rb = port.s6_scan(row(u, hs), row(pre, hs), layer.b_delta[hs].double().cpu().numpy(),
                             layer.a_log[hs].double().cpu().numpy(), Bk0, Ck0,
                             layer.D[hs].double().cpu().numpy(), row(gy, hs), "sequential", 1)
        gbk += rb["gBk"]
        gck += rb["gCk"]
    assert rel(r["gBk"][:1], gbk) < tol
    assert rel(r["gCk"][:1], gck) < tol
    y_again, _ = ops.s6_scan_fwd(u, pre, *p, Bk, Ck, layer.D)
    assert torch.equal(y, y_again)
    if io == "f32":
        u2 = randn((B, L, D), 16)
        y2, _ = ops.s6_scan_fwd(u2, pre, *p, Bk, Ck, layer.D)
        assert adjoint_gap(gy, y2, r["gu_local"], u2) < 1e-5
        y12, _ = ops.s6_scan_fwd(u + 2.0 * u2, pre, *p, Bk, Ck, layer.D)
        assert float((y12 - (y + 2.0 * y2)).abs().max()) / float(y.abs().max()) < 1e-5


def test_s5_c2_full_size(lrx):
    """C2: S5 layer B=32 L=4096 H=256 P=128 ZOH through the drop-in layer API,
    against the f64 oracle on the WHOLE batch: y, gu and every parameter
    gradient (the B*L = 131072-term reductions of layers.py:836-895 run on the
    split-K tensor-core GEMMs); plus forward linearity and the adjoint
    identity with layer_backward."""
    B, L, H = 32, 4096, 256
    layer = lrx.make_layer("s5", H, 256, dtype="f32", seed=0)
    u, u2, gy = randn((B, L, H), 21), randn((B, L, H), 22), randn((B, L, H), 23)
    y, tape = layer.forward(u, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    params = {k: v.double().cpu().numpy() for k, v in layer.parameters().items()}
    lay = port.Layer("s5", params, layer.discretization)
    ry, saved = lay.forward(u.double().cpu().numpy())
    rg, rgu = lay.backward(saved, gy.double().cpu().numpy())
    del saved
    assert rel(y, ry) < 1e-4
    assert rel(g.u, rgu) < 1e-4
    assert set(rg) == set(g.params)
    for k in rg:
        assert rel(g.params[k], rg[k]) < 1e-4, (k, rel(g.params[k], rg[k]))
    y2 = layer.forward(u2)
    assert adjoint_gap(gy, y2, g.u, u2) < 1e-5
    y12 = layer.forward(u + 2.0 * u2)
    assert float((y12 - (y + 2.0 * y2)).abs().max()) / float(y.abs().max()) < 1e-5
    assert torch.equal(layer.forward(u), y)


def test_lru_c1_full_size_against_oracle(lrx):
    """C1: LRU B=8 L=1024 H=128 N=64 -- small enough for the full oracle."""
    B, L, H = 8, 1024, 128
    layer = lrx.make_layer("lru", H, 64, dtype="f32", seed=0)
    u = port.Rng(31).normal((B, L, H)).astype(np.float32)
    gy = port.Rng(32).normal((B, L, H)).astype(np.float32)
    y, tape = layer.forward(u, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    params = {k: v.double().cpu().numpy() for k, v in layer.parameters().items()}
    lay = port.Layer("lru", params, None)
    ry, saved = lay.forward(u.astype(np.float64))
    rg, rgu = lay.backward(saved, gy.astype(np.float64))
    assert rel(y, ry) < 1e-4
    assert rel(g.u, rgu) < 1e-4
    for k in rg:
        assert rel(g.params[k], rg[k]) < 1e-4, k


def test_s6_c5_long_full_size(lrx):
    """C5: S6 B=1 L=2^20 D=2048 N=16 bf16 (one GPU: the in-kernel time
    segments carry the state across the whole million steps)."""
    from paper_2602_08810_b200 import ops
    B, L, D, N = 1, 2 ** 20, 2048, 16
    layer = lrx.make_layer("s6", D, N, dtype="f32", seed=0)
    u, gy = randn((B, L, D), 41, torch.bfloat16), randn((B, L, D), 42, torch.bfloat16)
    pre = randn((B, L, D), 43) * 0.5 - 2.0
    Bk, Ck = randn((B, L, N), 44), randn((B, L, N), 45)
    p = (layer.b_delta, layer.a_log)
    y, ck = ops.s6_scan_fwd(u, pre, *p, Bk, Ck, layer.D)
    r = ops.s6_scan_bwd(u, pre, *p, Bk, Ck, layer.D, ck, gy)
    cols = torch.tensor([5, D - 2], device="cuda")
    sl = lambda t: t.index_select(2, cols).double().cpu().numpy()  # noqa: E731
    ry, rg = port.s6_scan(sl(u), sl(pre), layer.b_delta.index_select(0, cols).double().cpu().numpy(),
                          layer.a_log.index_select(0, cols).double().cpu().numpy(), Bk.double().cpu().numpy(),
                          Ck.double().cpu().numpy(), layer.D.index_select(0, cols).double().cpu().numpy(), sl(gy))
    assert rel(y.index_select(2, cols), ry) < 1e-2
    for k in ("gu_local", "gpre"):
        assert rel(r[k].index_select(2, cols), rg[k]) < 1e-2, k
    for k in ("ga_log", "gb_delta"):
        assert rel(r[k].index_select(0, cols), rg[k]) < 1e-2, k
    y_again, _ = ops.s6_scan_fwd(u, pre, *p, Bk, Ck, layer.D)
    assert torch.equal(y, y_again)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_s6_c3_layer_full_row(lrx, dtype):
    """C3 through the drop-in layer API on one full-length batch row with all
    1536 channels: y, gu and EVERY parameter gradient (W_B / W_C are the
    channel-summed gB_k / gC_k contracted with u, layers.py:1068-1118) against
    the f64 oracle (run in channel blocks)."""
    L, D, N = 8192, 1536, 16
    layer = lrx.make_layer("s6", D, N, dtype=dtype, seed=0)
    u = randn((1, L, D), 51, layer.io_dtype)
    gy = randn((1, L, D), 52, layer.io_dtype)
    y, tape = layer.forward(u, tape=True)
    g = lrx.layer_backward(layer, tape, gy)
    params = {k: v.double().cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu, _ = port.s6_layer_blocked(params, u.double().cpu().numpy(), gy.double().cpu().numpy(), 256)
    tol = 1e-2 if dtype == "bf16" else 1e-4
    assert rel(y, ry) < tol
    assert rel(g.u, rgu) < tol
    assert set(rg) == set(g.params)
    for k in rg:
        assert rel(g.params[k], rg[k]) < tol, (k, rel(g.params[k], rg[k]))
