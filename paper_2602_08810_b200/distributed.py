"""Multi-GPU execution of the scan: batch sharding and sequence parallelism.

One process per GPU (torchrun, NCCL).  Two modes:

* **Batch sharding** (RG-LRU, S6, S5, LRU): lanes are independent, so each rank
  takes a contiguous batch slice and runs the single-GPU operator — no data-path
  collective.  Parameter gradients are summed by the caller's usual DP
  all-reduce.  `shard_range` is the split.

* **Sequence parallelism** (S6, config C5: B=1, L=2^20): the time axis is split
  into G contiguous slices, one per rank.  The recurrence is affine in its
  carry, so a slice is summarised by (A_r, X_r) with A_r[b,d,n] =
  exp(a[d,n] * sum_t delta_t) (the product of the slice's abar) and X_r = the
  slice's final state from a zero start.  Forward: every rank scans from zero,
  the (A_r, X_r) pairs are all-gathered (2 x B*D*N fp32 per rank, 262 KB for
  C5), each rank composes its exclusive prefix x_in = sum_k<r (prod A) X_k --
  the multi-rank analog of the reference's serial chunk stitch
  (scan.py:184-189, layers.py:167-169) -- and continues its slice from x_in.
  Backward mirrors it right-to-left with the cotangent carry h: the slice maps
  h_in -> h_out = A_r h_in + H_r, so the H_r are all-gathered and composed
  from the right.  Rank r's scan is re-run with the true carry (2x MUFU work on
  the ranks that receive a carry); the fix-up-only variant is next
  (DESIGN.md §8).

The carry algebra is in pure functions (`compose_prefix`, `compose_suffix`) so
it is tested on CPU with gloo, and `SeqParallelS6.simulate` runs the whole
protocol on one GPU (slices processed in turn) for the parity tests.
"""
from __future__ import annotations

import torch

from . import ops
from .numerics import softplus

__all__ = ["shard_range", "compose_prefix", "compose_suffix", "SeqParallelS6", "LongS6"]


def shard_range(n: int, world: int, rank: int):
    """Contiguous [start, stop) of `n` items owned by `rank` (balanced)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def compose_prefix(A, X, rank):
    """State entering slice `rank` from gathered per-slice summaries.

    A, X: [G, ...] (slice products and zero-start final states).  Returns
    sum_{k<rank} (prod_{k<j<rank} A_j) X_k, folded left to right."""
    x = torch.zeros_like(X[0])
    for k in range(rank):
        x = A[k] * x + X[k]
    return x


def compose_suffix(A, H, rank):
    """Cotangent carry entering slice `rank` from the right:
    h = sum_{k>rank} (prod_{rank<j<k} A_j) H_k, folded right to left."""
    h = torch.zeros_like(H[0])
    for k in range(A.shape[0] - 1, rank, -1):
        h = A[k] * h + H[k]
    return h


def _slice_product(pre, b_delta, a_log):
    """A_r = exp(a * sum_t softplus(pre_t + b)) for a [B, L, D] slice -> [B, D, N]."""
    sd = softplus(pre.to(a_log.dtype) + b_delta).sum(dim=1)            # [B, D]
    return torch.exp(-torch.exp(a_log)[None] * sd[..., None])



def _all_gather(t, group):
    """[world, *t.shape]: every rank's t.  NCCL gathers device tensors in place
    (all_gather_into_tensor over NVLink); a gloo group (CPU tests, the
    single-GPU multi-rank bench hook) gathers host copies."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = t.contiguous()
    if dist.get_backend(group) == "gloo":
        parts = [torch.empty_like(t, device="cpu") for _ in range(world)]
        dist.all_gather(parts, t.cpu(), group=group)
        return torch.stack(parts).to(t.device)
    out = torch.empty((world * t.shape[0], *t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t, group=group)
    return out.view(world, *t.shape)

class SeqParallelS6:
    """Sequence-parallel selective scan over a process group (or simulated).

    `scan_fwd(u, pre, b_delta, a_log, Bk, Ck, D, x0=None) -> (y, ckpt)` and
    `scan_bwd(..., ckpt, gy, h_in=None, want_h_out=False) -> dict` default to
    the device operators in ops.py; they are injectable so the exchange
    protocol can be exercised by CPU tests."""

    def __init__(self, group=None, scan_fwd=None, scan_bwd=None):
        self.group = group
        self.scan_fwd = scan_fwd or ops.s6_scan_fwd
        self.scan_bwd = scan_bwd or ops.s6_scan_bwd

    # -- collective helpers -------------------------------------------------
    def _gather(self, t):
        return _all_gather(t, self.group)

    # -- forward / backward on this rank's slice ----------------------------
    def forward(self, u, pre, b_delta, a_log, Bk, Ck, Dskip):
        import torch.distributed as dist
        rank = dist.get_rank(self.group)
        y, ckpt = self.scan_fwd(u, pre, b_delta, a_log, Bk, Ck, Dskip)
        A = _slice_product(pre, b_delta, a_log)
        AX = self._gather(torch.stack((A, ckpt[:, -1])))                   # [G, 2, B, D, N]
        x_in = compose_prefix(AX[:, 0], AX[:, 1], rank)
        if rank > 0:
            y, ckpt = self.scan_fwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, x0=x_in.contiguous())
        return y, {"ckpt": ckpt, "A": AX[:, 0]}

    def backward(self, ctx, u, pre, b_delta, a_log, Bk, Ck, Dskip, gy):
        import torch.distributed as dist
        rank = dist.get_rank(self.group)
        world = dist.get_world_size(self.group)
        r = self.scan_bwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, ctx["ckpt"], gy, want_h_out=True)
        H = self._gather(r["h_out"])
        h_in = compose_suffix(ctx["A"], H, rank)
        if rank < world - 1:
            r = self.scan_bwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, ctx["ckpt"], gy, h_in=h_in.contiguous(),
                              want_h_out=True)
        return r  # per-rank parameter-gradient contributions: sum them across ranks

    # -- single-process simulation (tests, one GPU) ---------------------------
    @staticmethod
    def simulate(G, u, pre, b_delta, a_log, Bk, Ck, Dskip, gy):
        """Run the protocol with the sequence split into G slices on one device.
        Returns (y, grads) assembled over slices, parameter grads summed."""
        L = u.shape[1]
        cuts = [shard_range(L, G, r) for r in range(G)]
        sl = [(lambda t, s=s, e=e: t[:, s:e].contiguous()) for s, e in cuts]
        loc = [ops.s6_scan_fwd(sl[r](u), sl[r](pre), b_delta, a_log, sl[r](Bk), sl[r](Ck), Dskip) for r in range(G)]
        A = torch.stack([_slice_product(sl[r](pre), b_delta, a_log) for r in range(G)])
        X = torch.stack([c[:, -1] for _, c in loc])
        ys, ckpts = [], []
        for r in range(G):
            if r == 0:
                y, c = loc[0]
            else:
                y, c = ops.s6_scan_fwd(sl[r](u), sl[r](pre), b_delta, a_log, sl[r](Bk), sl[r](Ck), Dskip,
                                       x0=compose_prefix(A, X, r).contiguous())
            ys.append(y)
            ckpts.append(c)
        H = torch.stack([ops.s6_scan_bwd(sl[r](u), sl[r](pre), b_delta, a_log, sl[r](Bk), sl[r](Ck), Dskip, ckpts[r],
                                         sl[r](gy), want_h_out=True)["h_out"] for r in range(G)])
        outs = []
        for r in range(G):
            h_in = compose_suffix(A, H, r) if r < G - 1 else None
            outs.append(ops.s6_scan_bwd(sl[r](u), sl[r](pre), b_delta, a_log, sl[r](Bk), sl[r](Ck), Dskip, ckpts[r],
                                        sl[r](gy), h_in=None if h_in is None else h_in.contiguous()))
        grads = {k: torch.cat([o[k] for o in outs], dim=1) for k in ("gu_local", "gpre", "gBk", "gCk")}
        for k in ("ga_log", "gD", "gb_delta"):
            grads[k] = sum(o[k] for o in outs)
        return torch.cat(ys, dim=1), grads


# ---------------------------------------------------------------------------
# Sequence parallelism for B = 1, long L (config C5), two levels:
#   * inside a GPU the kernels cut the rank's slice into time segments that run
#     concurrently (C5 has B*D = 2048 channels; a GPU needs ~30x more
#     independent lanes), composing the segment maps themselves (lrx_s6v3.cu);
#   * across GPUs each rank computes its slice's map once (lrx_s6_fwd_carry:
#     x_agg, sum delta -- 2 x 131 KB at C5), the maps are all-gathered over
#     NVLink, each rank composes the carry entering its slice, and the main
#     pass reuses the per-segment maps already in the workspace
#     (LRX_S6_REUSE_AGG), so a rank does one aggregate pass + one main pass,
#     the same work as on a single GPU.  The backward mirrors it right to left.

class LongS6:
    """Sequence-parallel selective scan for B = 1, long L (config C5).

    forward/backward operate on this rank's contiguous slice [1, Ls, D]; with
    `group=None` and no initialised process group the slice is the whole
    sequence (single GPU)."""

    def __init__(self, group=None, impl=None):
        """`impl` provides s6_fwd_carry / s6_scan_fwd / s6_bwd_carry / s6_scan_bwd /
        S6_REUSE_AGG (default: the device operators in ops.py); injectable so
        the exchange protocol can be exercised by CPU tests."""
        self.group = group
        self.ops = impl or ops

    def _rank_world(self):
        import torch.distributed as dist
        if not (dist.is_available() and dist.is_initialized()):
            return 0, 1
        return dist.get_rank(self.group), dist.get_world_size(self.group)

    def _gather(self, t):
        return _all_gather(t, self.group)

    @staticmethod
    def _prod(a_log, sd):
        """prod abar over a slice = exp(a * sum delta), [B, D, N]."""
        return torch.exp(-torch.exp(a_log)[None] * sd[..., None])

    def forward(self, u, pre, b_delta, a_log, Bk, Ck, Dskip):
        o = self.ops
        rank, world = self._rank_world()
        if world == 1:
            y, ckpt = o.s6_scan_fwd(u, pre, b_delta, a_log, Bk, Ck, Dskip)
            return y, {"ckpt": ckpt}
        x_agg, sd, ws = o.s6_fwd_carry(u, pre, b_delta, a_log, Bk)
        AX = self._gather(torch.stack((self._prod(a_log, sd), x_agg)))       # [G, 2, B, D, N]
        x_in = compose_prefix(AX[:, 0], AX[:, 1], rank).contiguous()
        y, ckpt = o.s6_scan_fwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, x0=x_in, ws=ws, flags=o.S6_REUSE_AGG)
        return y, {"ckpt": ckpt, "A": AX[:, 0]}

    def backward(self, ctx, u, pre, b_delta, a_log, Bk, Ck, Dskip, gy):
        o = self.ops
        rank, world = self._rank_world()
        if world == 1:
            return o.s6_scan_bwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, ctx["ckpt"], gy)
        h_agg, _, ws = o.s6_bwd_carry(gy, pre, b_delta, a_log, Ck)
        H = self._gather(h_agg)
        h_in = compose_suffix(ctx["A"], H, rank).contiguous()
        # per-rank parameter-gradient contributions: the caller sums them across ranks
        return o.s6_scan_bwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, ctx["ckpt"], gy, h_in=h_in, ws=ws,
                             flags=o.S6_REUSE_AGG)

    @staticmethod
    def simulate(G, u, pre, b_delta, a_log, Bk, Ck, Dskip, gy):
        """Run the two-level protocol with the sequence split into G rank slices
        on one device (the all-gathers become stacks).  Returns (y, grads)
        assembled over slices, parameter grads summed."""
        L = u.shape[1]
        cuts = [shard_range(L, G, r) for r in range(G)]
        sl = [(lambda t, s=s, e=e: t[:, s:e].contiguous()) for s, e in cuts]
        fc = [ops.s6_fwd_carry(sl[r](u), sl[r](pre), b_delta, a_log, sl[r](Bk)) for r in range(G)]
        A = torch.stack([LongS6._prod(a_log, sd) for _, sd, _ in fc])
        X = torch.stack([x for x, _, _ in fc])
        ys, ckpts = [], []
        for r in range(G):
            y, c = ops.s6_scan_fwd(sl[r](u), sl[r](pre), b_delta, a_log, sl[r](Bk), sl[r](Ck), Dskip,
                                   x0=compose_prefix(A, X, r).contiguous(), ws=fc[r][2], flags=ops.S6_REUSE_AGG)
            ys.append(y)
            ckpts.append(c)
        bc = [ops.s6_bwd_carry(sl[r](gy), sl[r](pre), b_delta, a_log, sl[r](Ck)) for r in range(G)]
        H = torch.stack([h for h, _, _ in bc])
        outs = [ops.s6_scan_bwd(sl[r](u), sl[r](pre), b_delta, a_log, sl[r](Bk), sl[r](Ck), Dskip, ckpts[r], sl[r](gy),
                                h_in=compose_suffix(A, H, r).contiguous(), ws=bc[r][2], flags=ops.S6_REUSE_AGG)
                for r in range(G)]
        grads = {k: torch.cat([o[k] for o in outs], dim=1) for k in ("gu_local", "gpre", "gBk", "gCk")}
        for k in ("ga_log", "gD", "gb_delta"):
            grads[k] = sum(o[k] for o in outs)
        return torch.cat(ys, dim=1), grads
