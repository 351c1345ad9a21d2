"""Sharding plumbing of the batched search, device-agnostic torch.

Two layouts, one prefix rule:

  * range sharding (configs 1 and 4): shard s holds a contiguous id range of
    EVERY list; the global list order is ascending id, i.e. shard order;
  * list sharding (config 2): whole lists are assigned to shards (greedy by
    length, `assign_lists`), the other lists are empty on that shard.

qmax reads the first `init` codes of the first probed cell and the
saturation rule (F_sat) the first R valid lanes of the probe-order stream
(qadc.py:157-194, scan_kernels.c:318-350), both on the GLOBAL list. Every
shard therefore installs the global first P = max(init, R) codes of every
list (`DeviceIndex.set_prefix`). Under range sharding those heads are spread
over the shards: shard s contributes
    need[s, L] = clamp(P - sum_{s' < s} count[s', L], 0, count[s, L])
rows of list L (`prefix_need`), and the heads are concatenated list-major,
shard-minor (`assemble_prefix`). `gather_prefix` does this across ranks with
two all_gathers (counts, then padded heads); it is index-build plumbing, not
part of the timed search.
"""

from __future__ import annotations

import torch


def prefix_need(counts: torch.Tensor, P: int) -> torch.Tensor:
    """counts (S, K) rows per (shard, list) -> rows each shard contributes
    to the global P-row prefix of each list (same shape)."""
    before = torch.cumsum(counts, 0) - counts
    return torch.minimum(torch.clamp(P - before, min=0), counts)


def _ranges(starts: torch.Tensor, lens: torch.Tensor) -> torch.Tensor:
    """Concatenation of arange(starts[i], starts[i] + lens[i])."""
    total = int(lens.sum())
    if total == 0:
        return torch.zeros(0, dtype=torch.int64, device=starts.device)
    excl = torch.cumsum(lens, 0) - lens
    rep = torch.repeat_interleave(torch.arange(lens.shape[0], device=starts.device), lens)
    return starts[rep] + (torch.arange(total, device=starts.device) - excl[rep])


def take_heads(rows: torch.Tensor, ids: torch.Tensor, row_off: torch.Tensor,
               need: torch.Tensor):
    """The first need[L] rows (and ids) of every list L of a row-ordered
    shard (rows (n, w), ids (n,), row_off (K + 1,))."""
    idx = _ranges(row_off[:-1].to(torch.int64), need.to(torch.int64))
    return rows[idx], ids[idx]


def assemble_prefix(parts, need: torch.Tensor):
    """parts[s] = (rows_s, ids_s) heads of shard s (list-major, need[s, L]
    rows of list L); need (S, K). Returns the global prefix (rows, ids,
    row_off (K + 1,)) list-major, shard-minor."""
    S, K = need.shape
    dev = need.device
    per_list = need.sum(0)
    off = torch.zeros(K + 1, dtype=torch.int64, device=dev)
    off[1:] = torch.cumsum(per_list, 0)
    base = off[:-1].unsqueeze(0) + (torch.cumsum(need, 0) - need)  # (S, K) start of shard s in L
    width = parts[0][0].shape[1]
    rows = torch.empty((int(off[-1]), width), dtype=parts[0][0].dtype, device=dev)
    ids = torch.empty(int(off[-1]), dtype=torch.int64, device=dev)
    for s, (r, i) in enumerate(parts):
        dst = _ranges(base[s], need[s])
        rows[dst] = r.to(dev)
        ids[dst] = i.to(dev)
    return rows, ids, off


def gather_prefix(rows: torch.Tensor, ids: torch.Tensor, row_off: torch.Tensor, P: int,
                  group=None):
    """Range-sharded global prefix across ranks (torch.distributed, NCCL on
    GPUs, gloo in the CPU tests). Returns (rows, ids, row_off, global_count)
    identical on every rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    cnt = (row_off[1:] - row_off[:-1]).to(torch.int64).contiguous()
    allc = [torch.empty_like(cnt) for _ in range(world)]
    dist.all_gather(allc, cnt, group=group)
    counts = torch.stack(allc)
    need = prefix_need(counts, P)
    hr, hi = take_heads(rows, ids, row_off, need[rank])
    tot = need.sum(1)
    mx = int(tot.max())
    pr = torch.zeros((mx, rows.shape[1]), dtype=rows.dtype, device=rows.device)
    pi = torch.zeros(mx, dtype=torch.int64, device=rows.device)
    pr[: hr.shape[0]] = hr
    pi[: hi.shape[0]] = hi
    gr = [torch.empty_like(pr) for _ in range(world)]
    gi = [torch.empty_like(pi) for _ in range(world)]
    dist.all_gather(gr, pr, group=group)
    dist.all_gather(gi, pi, group=group)
    parts = [(gr[s][: int(tot[s])], gi[s][: int(tot[s])]) for s in range(world)]
    prow, pid, poff = assemble_prefix(parts, need)
    return prow, pid, poff, counts.sum(0)


def assign_lists(sizes, world: int):
    """List sharding: greedy longest-first assignment of lists to shards
    (SURVEY 8e "greedy by length for balance"); returns owner (K,) int64."""
    import numpy as np

    sizes = np.asarray(sizes, dtype=np.int64)
    owner = np.zeros(sizes.shape[0], dtype=np.int64)
    load = np.zeros(world, dtype=np.int64)
    for L in np.argsort(-sizes, kind="stable"):
        s = int(np.argmin(load))
        owner[L] = s
        load[s] += sizes[L]
    return owner


def keep_lists(rows: torch.Tensor, ids: torch.Tensor, row_off: torch.Tensor,
               keep: torch.Tensor):
    """Row-ordered shard that keeps only the lists with keep[L] (the others
    become empty); returns (rows, ids, row_off)."""
    cnt = (row_off[1:] - row_off[:-1]).to(torch.int64)
    new_cnt = torch.where(keep.to(torch.bool), cnt, torch.zeros_like(cnt))
    idx = _ranges(row_off[:-1].to(torch.int64), new_cnt)
    off = torch.zeros_like(row_off, dtype=torch.int64)
    off[1:] = torch.cumsum(new_cnt, 0)
    return rows[idx].contiguous(), ids[idx].contiguous(), off
