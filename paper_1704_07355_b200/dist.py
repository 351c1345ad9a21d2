"""Multi-GPU plumbing for the sharded search.

The Quick ADC path shards by database range (exhaustive configs) or by
inverted list (IVF): every rank scans its own codes with the GLOBAL prefix
semantics installed (`DeviceIndex.set_prefix`, only the prefix owner keeps
the saturated first-R lanes), and the only exchange is the per-query top-R
merge below — Q x R x 12 bytes per rank over NCCL (NVLink) or gloo (CPU
tests).

The per-query Index + Tables phases (probe, residual + rotation + LUT,
qmax, quantize, prefix facts) do not depend on which codes a rank holds,
so `sharded_prepare` splits them by query instead of replicating them:
rank r prepares queries [r s, (r + 1) s), the prepared state (uint8
tables, qmin / delta, probe order, bounds, F_sat) is all-gathered — about
0.53 KB per (query, probed cell) at m = 32, 0.34 GB per configs[4] batch —
and every rank then scans its own codes for the whole batch.
"""

from __future__ import annotations

import torch

_BIG = torch.iinfo(torch.int64).max


def merge_sorted_lists(ids: torch.Tensor, dists: torch.Tensor, R: int):
    """Exact top-R by (distance, id) of concatenated per-shard lists:
    ids / dists (Q, S*R), -1 / +inf padding. Two stable sorts (id, then
    distance) give the lexicographic order the reference heap uses."""
    ai = torch.where(ids < 0, torch.full_like(ids, _BIG), ids)
    o = torch.argsort(ai, dim=1, stable=True)
    ai, ad = torch.gather(ai, 1, o), torch.gather(dists, 1, o)
    o = torch.argsort(ad, dim=1, stable=True)
    ai, ad = torch.gather(ai, 1, o)[:, :R], torch.gather(ad, 1, o)[:, :R]
    counts = (ai != _BIG).sum(dim=1).to(torch.int32)
    ai = torch.where(ai == _BIG, torch.full_like(ai, -1), ai)
    return ai, ad, counts


def merge_topr(ids: torch.Tensor, dists: torch.Tensor, R: int, group=None):
    """All-gather every rank's (Q, R) results and merge them exactly; every
    rank returns the global (ids, dists, counts)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:  # a single shard's list is already the exact top-R
        return ids, dists, (ids >= 0).sum(dim=1).to(torch.int32)
    gi = [torch.empty_like(ids) for _ in range(world)]
    gd = [torch.empty_like(dists) for _ in range(world)]
    dist.all_gather(gi, ids.contiguous(), group=group)
    dist.all_gather(gd, dists.contiguous(), group=group)
    return merge_sorted_lists(torch.cat(gi, dim=1), torch.cat(gd, dim=1), R)


def _all_gather_cat(t: torch.Tensor, group=None) -> torch.Tensor:
    """Concatenation (dim 0) of every rank's equally shaped tensor: one
    all_gather_into_tensor over NCCL; gloo stages through host memory."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype,
                          device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        return out
    h = t.detach().cpu().contiguous()
    parts = [torch.empty_like(h) for _ in range(world)]
    dist.all_gather(parts, h, group=group)
    return torch.cat(parts, 0).to(t.device)


def sharded_prepare(index, queries: torch.Tensor, R: int, ma: int, init: int, group=None,
                    fsat_owner: int = 0) -> dict:
    """Query-sharded first half of a distributed search: every rank runs
    index.prepare on its slice of the batch (padded to equal slices), the
    slices are all-gathered, and each rank gets the full batch's prepared
    state — bit-identical to preparing the whole batch locally, since the
    prefix region every rank holds is the GLOBAL one. Only `fsat_owner`
    keeps the saturated first-R lanes (range sharding: the owner of the
    global list heads)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    nq = queries.shape[0]
    if world == 1:
        return index.prepare(queries, R, ma=ma, init=init, with_fsat=True)
    per = -(-nq // world)
    qp = queries
    if per * world != nq:  # pad with copies of the last query
        qp = torch.cat([queries, queries[-1:].expand(per * world - nq, -1)], 0)
    local = index.prepare(qp[rank * per:(rank + 1) * per].contiguous(), R, ma=ma, init=init,
                          with_fsat=True)
    full = {k: _all_gather_cat(v, group)[:nq].contiguous() for k, v in local.items()}
    if rank != fsat_owner:
        full["fsat_n"].zero_()
    return full
