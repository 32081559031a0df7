"""Multi-GPU execution of the scan: batch sharding and sequence parallelism.

One process per GPU (torchrun, NCCL).  Two modes:

* **Batch sharding** (RG-LRU, S6, S5, LRU): lanes are independent, so each rank
  takes a contiguous batch slice and runs the single-GPU operator -- no data-path
  collective.  Parameter gradients are summed by the caller's usual DP
  all-reduce.  `shard_range` is the split.

* **Sequence parallelism** (S6, config C5: B=1, L=2^20; `LongS6`, and the S6
  layer with `seq_group=`): the time axis is split into G contiguous slices,
  one per rank.  The recurrence is affine in its carry, so a slice is
  summarised by (A_r, X_r) with A_r[b,d,n] = exp(a[d,n] * sum_t delta_t) (the
  product of the slice's abar) and X_r = the slice's final state from a zero
  start.  Forward: the (A_r, X_r) pairs are all-gathered (2 x B*D*N fp32 per
  rank, 262 KB for C5), each rank composes its exclusive prefix
  x_in = sum_k<r (prod A) X_k -- the multi-rank analog of the reference's serial
  chunk stitch (scan.py:184-189, layers.py:167-169) -- and scans its slice from
  x_in.  Backward mirrors it right-to-left with the cotangent carry h (the slice
  maps h_in -> h_out = A_r h_in + H_r).  The parameter gradients are sums over
  the whole sequence, so the per-rank partials are reduced inside the backward
  (`reduce_fixed_order`: all-gather, then summed in rank order -- bitwise
  reproducible, and equal to `LongS6.simulate`'s order), giving every rank the
  complete gradients the layer contract returns (autograd.py:222-233).

The carry algebra is in pure functions (`compose_prefix`, `compose_suffix`) so
it is tested on CPU with gloo, and `LongS6.simulate` runs the whole protocol on
one GPU (slices processed in turn) for the parity tests.
"""
from __future__ import annotations

import torch

from . import ops

__all__ = ["shard_range", "compose_prefix", "compose_suffix", "reduce_fixed_order", "LongS6"]


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

def reduce_fixed_order(tensors, group=None):
    """Sum each tensor over the ranks of `group`, in rank order (one all-gather
    of the flattened tensors, then r0 + r1 + ... on every rank): the same bits
    on every rank and on every run, unlike a reduction whose order depends on
    the collective's algorithm.  Returns new tensors of the same shapes."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return [t.clone() for t in tensors]
    dt = tensors[0].dtype
    flat = torch.cat([t.reshape(-1).to(dt) for t in tensors])
    parts = _all_gather(flat[None], group)[:, 0]                          # [G, total]
    tot = parts[0].clone()
    for r in range(1, parts.shape[0]):
        tot += parts[r]
    out, o = [], 0
    for t in tensors:
        out.append(tot[o:o + t.numel()].view(t.shape).to(t.dtype))
        o += t.numel()
    return out


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

    @staticmethod
    def _groups(u, N):
        """d_state 32 / 48 / 64 ...: the protocol runs per 16-state group (the
        recurrence is diagonal, as ops.s6_scan_*'s grouping)."""
        return N > 16 and N % 16 == 0 and u.dtype in (torch.float32, torch.bfloat16)

    def forward(self, u, pre, b_delta, a_log, Bk, Ck, Dskip):
        """This rank's slice of the scan: (y, ctx) for backward."""
        rank, world = self._rank_world()
        N = Bk.shape[-1]
        if world > 1 and self._groups(u, N):
            u32, y, ctxs = u.float(), None, []
            for g in range(N // 16):
                sl = slice(16 * g, 16 * g + 16)
                yg, cg = self._forward16(u32, pre, b_delta, a_log[:, sl].contiguous(), Bk[..., sl].contiguous(),
                                         Ck[..., sl].contiguous(), Dskip if g == 0 else torch.zeros_like(Dskip),
                                         rank, world)
                y = yg if y is None else y.add_(yg)
                ctxs.append(cg)
            return y.to(u.dtype), {"groups": ctxs}
        return self._forward16(u, pre, b_delta, a_log, Bk, Ck, Dskip, rank, world)

    def _forward16(self, u, pre, b_delta, a_log, Bk, Ck, Dskip, rank, world):
        o = self.ops
        if world == 1:
            y, ckpt = o.s6_scan_fwd(u, pre, b_delta, a_log, Bk, Ck, Dskip)
            return y, {"ckpt": ckpt}
        x_agg, sd, ws = o.s6_fwd_carry(u, pre, b_delta, a_log, Bk)
        AX = self._gather(torch.stack((self._prod(a_log, sd), x_agg)))       # [G, 2, B, D, N]
        x_in = compose_prefix(AX[:, 0], AX[:, 1], rank).contiguous()
        y, ckpt = o.s6_scan_fwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, x0=x_in, ws=ws, flags=o.S6_REUSE_AGG)
        return y, {"ckpt": ckpt, "A": AX[:, 0]}

    def backward(self, ctx, u, pre, b_delta, a_log, Bk, Ck, Dskip, gy, reduce=True):
        """Pullback of this rank's slice: gu_local, gpre, gBk, gCk of the slice and
        the parameter gradients ga_log, gD, gb_delta -- summed over all ranks in
        a fixed order when `reduce` (the default; the S6 layer reduces all its
        parameter gradients in one collective and passes reduce=False)."""
        rank, world = self._rank_world()
        if "groups" in ctx:
            u32, gy32, out = u.float(), gy.float(), None
            for g, cg in enumerate(ctx["groups"]):
                sl = slice(16 * g, 16 * g + 16)
                r = self._backward16(cg, u32, pre, b_delta, a_log[:, sl].contiguous(), Bk[..., sl].contiguous(),
                                     Ck[..., sl].contiguous(), Dskip if g == 0 else torch.zeros_like(Dskip),
                                     gy32, rank, world)
                if out is None:
                    out = {k: (v if k in ("gu_local", "gpre", "gD", "gb_delta") else [v]) for k, v in r.items()}
                else:  # fixed group order; gD = sum gy u does not depend on the group
                    for k in ("gu_local", "gpre", "gb_delta"):
                        out[k].add_(r[k])
                    for k in ("gBk", "gCk", "ga_log"):
                        out[k].append(r[k])
            out["gu_local"] = out["gu_local"].to(u.dtype)
            for k in ("gBk", "gCk", "ga_log"):
                out[k] = torch.cat(out[k], dim=-1)
        else:
            out = self._backward16(ctx, u, pre, b_delta, a_log, Bk, Ck, Dskip, gy, rank, world)
        if reduce and world > 1:
            out["ga_log"], out["gD"], out["gb_delta"] = reduce_fixed_order(
                [out["ga_log"], out["gD"], out["gb_delta"]], self.group)
        return out

    def _backward16(self, ctx, u, pre, b_delta, a_log, Bk, Ck, Dskip, gy, rank, world):
        o = self.ops
        if world == 1:
            return o.s6_scan_bwd(u, pre, b_delta, a_log, Bk, Ck, Dskip, ctx["ckpt"], gy)
        h_agg, _, ws = o.s6_bwd_carry(gy, pre, b_delta, a_log, Ck)
        H = self._gather(h_agg)
        h_in = compose_suffix(ctx["A"], H, rank).contiguous()
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
