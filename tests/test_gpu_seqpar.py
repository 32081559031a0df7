"""Sequence parallelism through the drop-in S6 layer (make_layer(..., seq_group=)):
two ranks (gloo, both on cuda:0 -- the round's GPU budget is one device) each
forward their contiguous slice of the sequence; the carries cross ranks
through distributed.LongS6 and layer_backward returns the complete parameter
gradients on every rank.  Checked against one single-GPU layer pass over the
whole sequence and against the f64 oracle (reference layers.py:1051-1118,
scan.py:184-189)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port

pytestmark = pytest.mark.gpu

M, B, L = 64, 2, 3000


def _worker(rank, world, port_no, q, n):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2602_08810_b200 as lrx
        from paper_2602_08810_b200.distributed import shard_range
        layer = lrx.make_layer("s6", M, n, dtype="f32", seed=9, seq_group="world")
        u = port.Rng(10).normal((B, L, M)).astype(np.float32)
        gy = port.Rng(11).normal((B, L, M)).astype(np.float32)
        s, e = shard_range(L, world, rank)
        y, tape = layer.forward(np.ascontiguousarray(u[:, s:e]), tape=True)
        g = lrx.layer_backward(layer, tape, np.ascontiguousarray(gy[:, s:e]))
        q.put((rank, y, g.u, g.params))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [16, 64])
def test_s6_layer_sequence_parallel_two_ranks(n):
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port_no = sck.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, q, n)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=300) for _ in range(2)), key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    import paper_2602_08810_b200 as lrx
    layer = lrx.make_layer("s6", M, n, dtype="f32", seed=9)
    u = port.Rng(10).normal((B, L, M)).astype(np.float32)
    gy = port.Rng(11).normal((B, L, M)).astype(np.float32)
    y1, tape = layer.forward(u, tape=True)
    g1 = lrx.layer_backward(layer, tape, gy)
    params = {k: v.double().cpu().numpy() for k, v in layer.parameters().items()}
    ry, rg, rgu, _ = port.s6_layer_blocked(params, u.astype(np.float64), gy.astype(np.float64), 64)
    y = np.concatenate([r[1] for r in res], axis=1)
    gu = np.concatenate([r[2] for r in res], axis=1)
    assert port.rel_err(y, y1) < 1e-5 and port.rel_err(y, ry) < 1e-4
    assert port.rel_err(gu, g1.u) < 1e-5 and port.rel_err(gu, rgu) < 1e-4
    for k in rg:
        assert np.array_equal(res[0][3][k], res[1][3][k]), k  # complete, identical on every rank
        assert port.rel_err(res[0][3][k], g1.params[k]) < 1e-5, k
        assert port.rel_err(res[0][3][k], rg[k]) < 1e-4, k
