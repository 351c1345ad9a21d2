"""Multi-GPU plumbing for the sharded search.

The Quick ADC path shards by database range (exhaustive configs) or by
inverted list (IVF): every rank scans its own codes with the GLOBAL prefix
semantics installed (`DeviceIndex.set_prefix`, only the prefix owner keeps
the saturated first-R lanes), and the only exchange is the per-query top-R
merge below — Q x R x 12 bytes per rank over NCCL (NVLink) or gloo (CPU
tests).
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
