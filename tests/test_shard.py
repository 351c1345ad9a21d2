"""CPU: sharding plumbing (paper_1704_07355_b200/shard.py) and the sharded
oracle (order-free restatement, oracle/qadc_oracle.c
orc_search_batch_sharded) against the heap restatement on the unsharded
index — range shards (configs 1, 4) and list shards (config 2), with
saturated first-R lanes and short first cells. The gloo world-2 test runs
the multi-rank prefix exchange the bench uses over NCCL."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_1704_07355_b200 import shard
from paper_1704_07355_b200.dist import merge_sorted_lists
from paper_1704_07355_b200.qadc import transpose_list


def _row_lists(rng, K, mean, width):
    sizes = rng.integers(0, 2 * mean, K)
    sizes[rng.random(K) < 0.2] = 0
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    rows = rng.integers(0, 256, (int(off[-1]), width), dtype=np.uint8)
    ids = np.arange(int(off[-1]), dtype=np.int64)
    return rows, ids, off


def _direct_prefix(rows, ids, off, P):
    r, i, o = [], [], [0]
    for L in range(off.shape[0] - 1):
        k = min(P, int(off[L + 1] - off[L]))
        r.append(rows[off[L]:off[L] + k])
        i.append(ids[off[L]:off[L] + k])
        o.append(o[-1] + k)
    return np.concatenate(r), np.concatenate(i), np.asarray(o, np.int64)


def _range_split(rows, ids, off, S, rng):
    """Shard s keeps a contiguous piece of every list (cut points random)."""
    out = []
    K = off.shape[0] - 1
    cuts = [np.sort(rng.integers(0, int(off[L + 1] - off[L]) + 1, S - 1)) for L in range(K)]
    for s in range(S):
        r, i, o = [], [], [0]
        for L in range(K):
            n = int(off[L + 1] - off[L])
            c = np.concatenate([[0], cuts[L], [n]])
            a, b = off[L] + c[s], off[L] + c[s + 1]
            r.append(rows[a:b])
            i.append(ids[a:b])
            o.append(o[-1] + (b - a))
        out.append((np.concatenate(r), np.concatenate(i), np.asarray(o, np.int64)))
    return out


def test_prefix_need_and_assembly_equal_global_prefix(rng):
    for trial in range(20):
        K, S, P = int(rng.integers(1, 40)), int(rng.integers(1, 6)), int(rng.integers(1, 50))
        rows, ids, off = _row_lists(rng, K, 30, 3)
        parts = _range_split(rows, ids, off, S, rng)
        counts = torch.stack([torch.from_numpy(np.diff(o)) for _, _, o in parts])
        need = shard.prefix_need(counts, P)
        heads = [shard.take_heads(torch.from_numpy(r), torch.from_numpy(i), torch.from_numpy(o),
                                  need[s]) for s, (r, i, o) in enumerate(parts)]
        pr, pi, po = shard.assemble_prefix(heads, need)
        wr, wi, wo = _direct_prefix(rows, ids, off, P)
        assert np.array_equal(po.numpy(), wo)
        assert np.array_equal(pr.numpy(), wr)
        assert np.array_equal(pi.numpy(), wi)
        assert np.array_equal(counts.sum(0).numpy(), np.diff(off))


def test_assign_lists_balances_and_keep_lists(rng):
    sizes = rng.integers(0, 1000, 257)
    owner = shard.assign_lists(sizes, 4)
    loads = np.bincount(owner, weights=sizes, minlength=4)
    assert loads.max() - loads.min() <= sizes.max()
    rows, ids, off = _row_lists(rng, 30, 20, 2)
    keep = torch.from_numpy(np.arange(30) % 3 == 1)
    r, i, o = shard.keep_lists(torch.from_numpy(rows), torch.from_numpy(ids),
                               torch.from_numpy(off), keep)
    for L in range(30):
        a, b = int(o[L]), int(o[L + 1])
        if L % 3 == 1:
            assert np.array_equal(i[a:b].numpy(), ids[off[L]:off[L + 1]])
            assert np.array_equal(r[a:b].numpy(), rows[off[L]:off[L + 1]])
        else:
            assert a == b


def _gather_worker(rank, world, port, seed, P, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(seed)
    rows, ids, off = _row_lists(rng, 23, 15, 4)
    parts = _range_split(rows, ids, off, world, rng)
    r, i, o = parts[rank]
    pr, pi, po, gc = shard.gather_prefix(torch.from_numpy(r), torch.from_numpy(i),
                                         torch.from_numpy(o), P)
    q.put((rank, pr.numpy(), pi.numpy(), po.numpy(), gc.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gather_prefix_equals_global_prefix():
    world, seed, P = 2, 5, 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + os.getpid() % 2000
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, seed, P, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(seed)
    rows, ids, off = _row_lists(rng, 23, 15, 4)
    wr, wi, wo = _direct_prefix(rows, ids, off, P)
    for _, pr, pi, po, gc in got:
        assert np.array_equal(pr, wr) and np.array_equal(pi, wi) and np.array_equal(po, wo)
        assert np.array_equal(gc, np.diff(off))


# ------------------------------------------------------------ sharded oracle

def _flat(rows, ids, off):
    blocks, bids, boff, count = [], [], [0], []
    for L in range(off.shape[0] - 1):
        tl = transpose_list(rows[off[L]:off[L + 1]], ids[off[L]:off[L + 1]])
        blocks.append(tl.blocks.reshape(-1))
        bids.append(tl.ids)
        boff.append(boff[-1] + tl.blocks.shape[0])
        count.append(tl.count)
    return (np.concatenate(blocks), np.asarray(boff, np.int64), np.concatenate(bids),
            np.asarray(count, np.int64))


def _ivf_case(seed, K=12, n=6000, m=8, d=32):
    rng = np.random.default_rng(seed)
    X = (rng.random((n, d)) * 50).astype(np.float32)
    coarse = X[rng.choice(n, K, replace=False)].copy()
    lab = np.argmin(((X[:, None, :] - coarse[None]) ** 2).sum(-1), 1)
    order = np.argsort(lab, kind="stable")
    sizes = np.bincount(lab, minlength=K)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    rows = rng.integers(0, 256, (n, m // 2), dtype=np.uint8)  # any codes: parity is per index
    cb = (rng.random((m, 16, d // m)) * 10).astype(np.float32)
    rot = np.linalg.qr(rng.standard_normal((d, d)))[0].astype(np.float32)
    qs = (rng.random((24, d)) * 50).astype(np.float32)
    return rows, order.astype(np.int64), off, coarse, cb, rot, qs


def _short_first_case(seed, sizes=(3, 2000, 50, 1500, 0, 2445), m=8, d=32):
    """The queries' nearest cell holds 3 codes: qmax is the max of those 3,
    most other lanes saturate, and the saturated lanes among the first R
    valid lanes (F_sat) fill the result."""
    rng = np.random.default_rng(seed)
    K = len(sizes)
    coarse = (rng.random((K, d)) * 50).astype(np.float32)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(off[-1])
    rows = rng.integers(0, 256, (n, m // 2), dtype=np.uint8)
    ids = rng.permutation(n).astype(np.int64)
    for L in range(K):
        ids[off[L]:off[L + 1]].sort()
    cb = (rng.random((m, 16, d // m)) * 10).astype(np.float32)
    rot = np.linalg.qr(rng.standard_normal((d, d)))[0].astype(np.float32)
    qs = (coarse[0] + rng.standard_normal((24, d))).astype(np.float32)
    return rows, ids, off, coarse, cb, rot, qs


@pytest.mark.parametrize("R,init,ma,short", [(40, 1000, 3, False), (30, 25, 4, False),
                                              (200, 10, 5, False), (100, 1000, 3, True),
                                              (300, 1000, 6, True)])
def test_sharded_oracle_equals_heap_oracle(R, init, ma, short):
    """Unsharded (prefix = the lists themselves), 3 range shards and 2 list
    shards, merged by (dist, id), all equal the heap restatement. The
    `short` cases start every query in a 3-code cell, so saturated first-R
    lanes (F_sat, only shard 0 contributes them) are part of the answer."""
    rows, ids, off, coarse, cb, rot, qs = (_short_first_case(R) if short else _ivf_case(7 + R))
    full = _flat(rows, ids, off)
    want_i, want_d, want_n, _ = orc.search_batch(qs, cb, rot, coarse, ma, full, R, init)
    if short:  # F_sat really matters here
        nof = orc.search_batch_sharded(qs, cb, rot, coarse, ma, full,
                                       _flat(*_direct_prefix(rows, ids, off, max(init, R)))[:3]
                                       + (np.diff(off),), R, init, with_fsat=False)
        assert (nof[2] < want_n).all()
    P = max(init, R)
    prefix = _flat(*_direct_prefix(rows, ids, off, P))[:3] + (np.diff(off),)
    one = orc.search_batch_sharded(qs, cb, rot, coarse, ma, full, prefix, R, init)
    assert np.array_equal(one[0], want_i)
    assert np.array_equal(one[1].view(np.uint32), want_d.view(np.uint32))
    rng = np.random.default_rng(R)
    splits = {"range": _range_split(rows, ids, off, 3, rng)}
    owner = shard.assign_lists(np.diff(off), 2)
    splits["list"] = []
    for s in range(2):
        r, i, o = shard.keep_lists(torch.from_numpy(rows), torch.from_numpy(ids),
                                   torch.from_numpy(off), torch.from_numpy(owner == s))
        splits["list"].append((r.numpy(), i.numpy(), o.numpy()))
    for kind, parts in splits.items():
        outs = [orc.search_batch_sharded(qs, cb, rot, coarse, ma, _flat(*p), prefix, R, init,
                                         with_fsat=(s == 0)) for s, p in enumerate(parts)]
        gi, gd, gc = merge_sorted_lists(torch.from_numpy(np.concatenate([o[0] for o in outs], 1)),
                                        torch.from_numpy(np.concatenate([o[1] for o in outs], 1)),
                                        R)
        assert np.array_equal(gi.numpy(), want_i), kind
        assert np.array_equal(gd.numpy().view(np.uint32), want_d.view(np.uint32)), kind
        assert np.array_equal(gc.numpy(), want_n), kind
