"""Multi-process host logic on CPU (gloo, world size 2): batch sharding and the
sequence-parallel carry exchange of paper_2602_08810_b200.distributed, with a
test-only torch restatement of the S6 slice scan (x0 / h_in aware) standing in
for the device kernels."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from paper_2602_08810_b200.distributed import compose_prefix, compose_suffix, reduce_fixed_order, shard_range


def test_shard_range_partitions():
    for n in (1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [e - s for s, e in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_carry_composition_matches_sequential():
    rng = np.random.default_rng(0)
    A = torch.tensor(rng.uniform(0.2, 1.0, (4, 3)))
    X = torch.tensor(rng.normal(size=(4, 3)))
    # sequential: x_{r+1} = A_r x_r + X_r from x_0 = 0
    x = torch.zeros(3, dtype=torch.float64)
    for r in range(4):
        assert torch.allclose(compose_prefix(A, X, r), x)
        x = A[r] * x + X[r]
    h = torch.zeros(3, dtype=torch.float64)
    for r in range(3, -1, -1):
        assert torch.allclose(compose_suffix(A, X, r), h)
        h = A[r] * h + X[r]


# ---- test-only torch restatement of the S6 slice scan (layers.py:1038-1098) --

def _fwd(u, pre, b_delta, a_log, Bk, Ck, D, x0=None):
    a = -torch.exp(a_log)
    delta = torch.nn.functional.softplus(pre + b_delta)
    B, L, m = u.shape
    x = torch.zeros((B, m, a.shape[1]), dtype=u.dtype) if x0 is None else x0.clone()
    xs, ys = [], []
    for t in range(L):
        xs.append(x)
        x = torch.exp(delta[:, t, :, None] * a) * x + (delta[:, t] * u[:, t])[..., None] * Bk[:, t, None, :]
        ys.append((x * Ck[:, t, None, :]).sum(-1) + D * u[:, t])
    ckpt = torch.stack(xs + [x], dim=1)          # every state + final (test layout)
    return torch.stack(ys, 1), ckpt


def _bwd(u, pre, b_delta, a_log, Bk, Ck, D, ckpt, gy, h_in=None, want_h_out=False):
    a = -torch.exp(a_log)
    pre_b = pre + b_delta
    delta = torch.nn.functional.softplus(pre_b)
    B, L, m = u.shape
    h = torch.zeros_like(ckpt[:, 0]) if h_in is None else h_in.clone()
    gu = torch.zeros_like(u)
    gpre = torch.zeros_like(u)
    gBk, gCk = torch.zeros_like(Bk), torch.zeros_like(Ck)
    ga = torch.zeros_like(a)
    for t in range(L - 1, -1, -1):
        ab = torch.exp(delta[:, t, :, None] * a)
        g = gy[:, t, :, None] * Ck[:, t, None, :] + h
        term = ab * g * ckpt[:, t]
        s1 = (g * Bk[:, t, None, :]).sum(-1)
        gdelta = (term * a).sum(-1) + s1 * u[:, t]
        gpre[:, t] = torch.sigmoid(pre_b[:, t]) * gdelta
        gu[:, t] = gy[:, t] * D + delta[:, t] * s1
        gBk[:, t] = (g * (delta[:, t] * u[:, t])[..., None]).sum(1)
        gCk[:, t] = (gy[:, t, :, None] * ckpt[:, t + 1]).sum(1)
        ga += (term * delta[:, t, :, None]).sum(0)
        h = ab * g
    out = {"gu_local": gu, "gpre": gpre, "gBk": gBk, "gCk": gCk, "ga_log": a * ga,
           "gD": (gy * u).sum((0, 1)), "gb_delta": gpre.sum((0, 1))}
    if want_h_out:
        out["h_out"] = h
    return out


class _CpuOps:
    """Test-only stand-in for ops.py's carry API (ws / flags are ignored)."""
    S6_REUSE_AGG = 1

    @staticmethod
    def s6_scan_fwd(u, pre, b_delta, a_log, Bk, Ck, D, x0=None, ws=None, flags=0):
        return _fwd(u, pre, b_delta, a_log, Bk, Ck, D, x0=x0)

    @staticmethod
    def s6_scan_bwd(u, pre, b_delta, a_log, Bk, Ck, D, ckpt, gy, h_in=None, ws=None, flags=0):
        return _bwd(u, pre, b_delta, a_log, Bk, Ck, D, ckpt, gy, h_in=h_in)

    @staticmethod
    def s6_fwd_carry(u, pre, b_delta, a_log, Bk, ws=None):
        zero = torch.zeros_like(Bk)
        _, ck = _fwd(u, pre, b_delta, a_log, Bk, zero, torch.zeros(u.shape[-1], dtype=u.dtype))
        return ck[:, -1], torch.nn.functional.softplus(pre + b_delta).sum(1), None

    @staticmethod
    def s6_bwd_carry(gy, pre, b_delta, a_log, Ck, ws=None):
        a = -torch.exp(a_log)
        delta = torch.nn.functional.softplus(pre + b_delta)
        h = torch.zeros((gy.shape[0], gy.shape[2], a.shape[1]), dtype=gy.dtype)
        for t in range(gy.shape[1] - 1, -1, -1):
            h = torch.exp(delta[:, t, :, None] * a) * (gy[:, t, :, None] * Ck[:, t, None, :] + h)
        return h, delta.sum(1), None


def _problem(L=24, m=3, n=4, dt=np.float64):
    p = port.init_params("s6", m, n, seed=3)
    rng = port.Rng(7)
    u = rng.normal((1, L, m))
    pre = (u @ p["W_delta"]) @ p["W_delta_proj"]
    T = lambda x: torch.tensor(np.asarray(x, dt))  # noqa: E731
    return dict(u=T(u), pre=T(pre), b_delta=T(p["b_delta"]), a_log=T(p["a_log"]), Bk=T(u @ p["W_B"].T),
                Ck=T(u @ p["W_C"].T), D=T(p["D"]), gy=T(rng.normal((1, L, m)))), p, u, pre


def _spawn(target, world, *args):
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port_no = sck.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, world, port_no, q) + args) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=120) for _ in range(world)), key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return res


def _worker_reduce(rank, world, port_no, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = torch.full((2, 3), 0.1 * (rank + 1), dtype=torch.float32)
        b = torch.arange(4, dtype=torch.float32) * (rank + 1)
        ra, rb = reduce_fixed_order([a, b])
        q.put((rank, ra.numpy(), rb.numpy()))
    finally:
        dist.destroy_process_group()


def test_reduce_fixed_order_gloo():
    """Rank-order sum, identical bits on every rank (the S6 sequence-parallel
    parameter-gradient reduction)."""
    res = _spawn(_worker_reduce, 3)
    want_a = (np.float32(0.1) + np.float32(0.2)) + np.float32(0.1 * 3)
    for _, ra, rb in res:
        assert ra.shape == (2, 3) and rb.shape == (4,)
        np.testing.assert_array_equal(ra, np.full((2, 3), np.float32(want_a)))
        np.testing.assert_array_equal(rb, np.arange(4, dtype=np.float32) * 6)
    assert all(np.array_equal(res[0][1], r[1]) for r in res)


def _worker_long(rank, world, port_no, q, L, n, dt):
    from paper_2602_08810_b200.distributed import LongS6
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pb, p, u, pre = _problem(L=L, n=n, dt=dt)
        s, e = shard_range(L, world, rank)
        sl = {k: (v[:, s:e].contiguous() if k in ("u", "pre", "Bk", "Ck", "gy") else v) for k, v in pb.items()}
        ls = LongS6(impl=_CpuOps)
        args = (sl["u"], sl["pre"], sl["b_delta"], sl["a_log"], sl["Bk"], sl["Ck"], sl["D"])
        y, ctx = ls.forward(*args)
        r = ls.backward(ctx, *args, sl["gy"])  # parameter gradients reduced inside
        q.put((rank, y.numpy(), {k: v.numpy() for k, v in r.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,dt,tol", [(4, np.float64, 1e-12), (32, np.float32, 2e-5)])
def test_hierarchical_long_sequence_gloo(n, dt, tol):
    """LongS6 over 2 gloo ranks (CPU stand-in kernels): slices stitched by the
    all-gathered carries equal the oracle's single pass; the parameter
    gradients come back complete (and bitwise equal) on every rank; d_state 32
    runs the protocol per 16-state group."""
    L = 36
    res = _spawn(_worker_long, 2, L, n, dt)
    pb, p, u, pre = _problem(L=L, n=n)
    y_ref, o = port.s6_scan(u, pre, p["b_delta"], p["a_log"], u @ p["W_B"].T, u @ p["W_C"].T, p["D"],
                            pb["gy"].numpy())
    assert port.rel_err(np.concatenate([r[1] for r in res], 1), y_ref) < tol
    for k in ("gu_local", "gpre", "gBk", "gCk"):
        assert port.rel_err(np.concatenate([r[2][k] for r in res], 1), o[k]) < tol, k
    for k in ("ga_log", "gD", "gb_delta"):
        assert port.rel_err(res[0][2][k], o[k]) < tol, k
        assert np.array_equal(res[0][2][k], res[1][2][k]), k
