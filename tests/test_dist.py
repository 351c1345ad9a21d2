"""Multi-process merge of per-shard top-R lists (world_size 2, gloo, CPU)
and the sharded-search semantics on one GPU (two shards of one list)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1704_07355_b200.dist import merge_sorted_lists, merge_topr


def _oracle_topr(ids, d, R):
    out_i = np.full((ids.shape[0], R), -1, np.int64)
    out_d = np.full((ids.shape[0], R), np.inf, np.float32)
    for q in range(ids.shape[0]):
        ok = ids[q] >= 0
        o = np.lexsort((ids[q][ok], d[q][ok]))[:R]
        out_i[q, :len(o)] = ids[q][ok][o]
        out_d[q, :len(o)] = d[q][ok][o]
    return out_i, out_d


def _shard_lists(seed, Q, R, world):
    """Per-rank (Q, R) ascending lists with heavy distance ties and padding."""
    rng = np.random.default_rng(seed)
    ids, ds = [], []
    for r in range(world):
        d = np.sort(rng.integers(0, 30, (Q, R)).astype(np.float32), axis=1)
        i = rng.integers(0, 10**6, (Q, R)).astype(np.int64) * world + r  # disjoint per rank
        pad = rng.random((Q, R)) < 0.1
        d = np.where(pad, np.inf, d).astype(np.float32)
        i = np.where(pad, -1, i)
        o = np.argsort(d, axis=1, kind="stable")
        ids.append(np.take_along_axis(i, o, 1))
        ds.append(np.take_along_axis(d, o, 1))
    return ids, ds


def _worker(rank, world, port, seed, Q, R, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids, ds = _shard_lists(seed, Q, R, world)
    gi, gd, gc = merge_topr(torch.from_numpy(ids[rank]), torch.from_numpy(ds[rank]), R)
    q.put((rank, gi.numpy(), gd.numpy(), gc.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_merge_sorted_lists_matches_lexsort():
    ids, ds = _shard_lists(3, 16, 50, 3)
    ai, ad = np.concatenate(ids, 1), np.concatenate(ds, 1)
    gi, gd, gc = merge_sorted_lists(torch.from_numpy(ai), torch.from_numpy(ad), 50)
    wi, wd = _oracle_topr(ai, ad, 50)
    assert np.array_equal(gi.numpy(), wi)
    assert np.array_equal(gd.numpy(), wd)
    assert np.array_equal(gc.numpy(), (wi >= 0).sum(1))


def test_gloo_world2_merge_equals_global_topr():
    world, Q, R, seed = 2, 8, 40, 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 2000
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, Q, R, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids, ds = _shard_lists(seed, Q, R, world)
    wi, wd = _oracle_topr(np.concatenate(ids, 1), np.concatenate(ds, 1), R)
    for _, gi, gd, gc in got:  # every rank holds the same global result
        assert np.array_equal(gi, wi)
        assert np.array_equal(gd, wd)


@pytest.mark.gpu
def test_two_shards_with_global_prefix_equal_unsharded(gpu):
    """Shard a flat list in two ranges on one GPU (sequentially, no waits
    between ranks): each shard installs the global prefix, only shard 0
    keeps F_sat; the merged result equals the unsharded search bit for bit,
    including saturated first-R lanes and qmax from the global prefix."""
    from paper_1704_07355_b200.device import DeviceIndex
    from paper_1704_07355_b200.ivf import encode_device
    from paper_1704_07355_b200.workload import _PQ
    rng = np.random.default_rng(21)
    n, m, d, R, init = 120_000, 16, 64, 100, 1000
    cb = (rng.random((m, 16, d // m)) * 40).astype(np.float32)
    pq = _PQ(cb)
    X = torch.from_numpy((rng.random((n, d)) * 40).astype(np.float32)).cuda()
    codes = encode_device(pq, X)
    cbt = torch.from_numpy(cb).cuda()
    full = DeviceIndex.from_device_rows(d, m, codes, torch.tensor([0, n], device="cuda"), cbt)
    qs = (rng.random((32, d)) * 40).astype(np.float32)
    want = full.search(qs, R, init=init)
    cut = 70_001
    parts = []
    for k, (lo, hi) in enumerate([(0, cut), (cut, n)]):
        sh = DeviceIndex.from_device_rows(
            d, m, codes[lo:hi].contiguous(), torch.tensor([0, hi - lo], device="cuda"), cbt,
            ids=torch.arange(lo, hi, dtype=torch.int64, device="cuda"))
        p = max(init, R)
        sh.set_prefix(codes[:p].contiguous(), torch.tensor([0, p], device="cuda"), [n],
                      ids=torch.arange(p, dtype=torch.int64, device="cuda"))
        parts.append(sh.search(qs, R, init=init, with_fsat=(k == 0)))
    gi, gd, gc = merge_sorted_lists(torch.from_numpy(np.concatenate([p.ids for p in parts], 1)),
                                    torch.from_numpy(np.concatenate([p.distances for p in parts],
                                                                    1)), R)
    assert np.array_equal(gi.numpy(), want.ids)
    assert np.array_equal(gd.numpy().view(np.uint32), want.distances.view(np.uint32))
    assert np.array_equal(gc.numpy(), want.counts)


@pytest.mark.gpu
def test_ivf_list_shards_with_global_prefix_equal_unsharded(gpu):
    """IVF list sharding (BASELINE config 2 "lists sharded across GPUs"),
    emulated on one GPU: shard k keeps the lists L with L % 2 == k, installs
    the global prefix of EVERY list (qmax and the saturation rule read the
    first probed cell's global prefix, whichever shard owns it), only shard
    0 keeps F_sat; the merged shard results equal the unsharded search."""
    from paper_1704_07355_b200 import datagen
    from paper_1704_07355_b200.device import DeviceIndex
    from paper_1704_07355_b200.ivf import assign_device, encode_device
    from paper_1704_07355_b200.workload import _PQ
    rng = np.random.default_rng(8)
    K, n, m, d, R, ma, init = 64, 60_000, 16, 64, 50, 6, 300
    mix = datagen.Mixture(d=d, components=40, centre_high=100.0, sigma=10.0)
    X = datagen.mixture_numpy(mix, n, seed=2, stream=2)
    coarse = X[rng.choice(n, K, replace=False)].copy()
    Rm = np.linalg.qr(rng.standard_normal((d, d)))[0].astype(np.float32)
    cb = (rng.standard_normal((m, 16, d // m)) * 6).astype(np.float32)
    pq = _PQ(cb, Rm)
    Xd, C = torch.from_numpy(X).cuda(), torch.from_numpy(coarse).cuda()
    lab = assign_device(coarse, Xd)
    codes = encode_device(pq, Xd - C[lab])
    order = torch.argsort(lab, stable=True)
    sizes = torch.bincount(lab, minlength=K)
    off = torch.zeros(K + 1, dtype=torch.int64, device="cuda")
    off[1:] = torch.cumsum(sizes, 0)
    sc = codes[order].contiguous()
    cbt, Rt = torch.from_numpy(cb).cuda(), torch.from_numpy(Rm).cuda()
    full = DeviceIndex.from_device_rows(d, m, sc, off, cbt, rotation=Rt, coarse=C, ids=order)
    qs = datagen.mixture_numpy(mix, 32, seed=2, stream=3)
    want = full.search(qs, R, ma=ma, init=init)
    # global prefixes of every list
    p = max(init, R)
    offn, szn = off.cpu().numpy(), sizes.cpu().numpy()
    pre_rows, pre_ids, pre_off = [], [], [0]
    for L in range(K):
        k = min(p, int(szn[L]))
        pre_rows.append(sc[offn[L]:offn[L] + k])
        pre_ids.append(order[offn[L]:offn[L] + k])
        pre_off.append(pre_off[-1] + k)
    pre_rows = torch.cat(pre_rows).contiguous()
    pre_ids = torch.cat(pre_ids).contiguous()
    pre_off = torch.tensor(pre_off, dtype=torch.int64, device="cuda")
    parts = []
    for shard in range(2):
        rows, ids, soff = [], [], [0]
        for L in range(K):
            a, b = int(offn[L]), int(offn[L + 1])
            if L % 2 != shard:
                b = a  # list owned by the other shard: empty here
            rows.append(sc[a:b])
            ids.append(order[a:b])
            soff.append(soff[-1] + (b - a))
        sh = DeviceIndex.from_device_rows(
            d, m, torch.cat(rows).contiguous(), torch.tensor(soff, device="cuda"), cbt,
            rotation=Rt, coarse=C, ids=torch.cat(ids).contiguous())
        sh.set_prefix(pre_rows, pre_off, szn, ids=pre_ids)
        parts.append(sh.search(qs, R, ma=ma, init=init, with_fsat=(shard == 0)))
        # query-sharded Tables phase (dist.sharded_prepare's exchange, the
        # all_gather emulated by concatenation): two halves of the batch
        # prepared separately give the same state as the whole batch, and
        # scanning it gives this shard's search result bit for bit
        qd = torch.from_numpy(qs).cuda()
        halves = [sh.prepare(qd[:13], R, ma=ma, init=init), sh.prepare(qd[13:], R, ma=ma, init=init)]
        prep = {k: torch.cat([h[k] for h in halves]).contiguous() for k in halves[0]}
        whole = sh.prepare(qd, R, ma=ma, init=init)
        for k in prep:
            assert torch.equal(prep[k], whole[k]), k
        if shard != 0:
            prep["fsat_n"].zero_()
        res2 = sh.scan(prep, R, ma=ma, init=init)
        assert np.array_equal(res2.ids.cpu().numpy(), parts[-1].ids)
        assert np.array_equal(res2.distances.cpu().numpy().view(np.uint32),
                              parts[-1].distances.view(np.uint32))
    gi, gd, gc = merge_sorted_lists(torch.from_numpy(np.concatenate([x.ids for x in parts], 1)),
                                    torch.from_numpy(np.concatenate([x.distances for x in parts],
                                                                    1)), R)
    assert np.array_equal(gi.numpy(), want.ids)
    assert np.array_equal(gd.numpy().view(np.uint32), want.distances.view(np.uint32))
    assert np.array_equal(gc.numpy(), want.counts)


class _FakePrepIndex:
    """CPU stand-in for DeviceIndex.prepare: a deterministic per-query
    function with the same output names, shapes and dtypes (the exchange
    under test only moves rows)."""

    K, m = 64, 32

    def prepare(self, queries, R, ma=1, init=1000, with_fsat=True):
        nq = queries.shape[0]
        s = (queries.double().sum(1) * 1000).long()
        ar = torch.arange(ma)
        p = {"cells": (s[:, None] * 7 + ar) % self.K,
             "qt": ((s[:, None, None] + torch.arange(self.m * 4)) % 127).int().expand(
                 nq, ma, self.m * 4).contiguous(),
             "qmin_f": queries[:, :ma].float().contiguous(),
             "delta_f": queries[:, -ma:].float().contiguous(),
             "depth": (s[:, None] % 5 + ar).to(torch.uint8),
             "qmax": queries.max(1).values.float(),
             "M_bits": (s % 1000).int(),
             "fsat_n": (s % 3).int() if with_fsat else torch.zeros(nq, dtype=torch.int32),
             "fsat_mid": queries[:, :1].expand(nq, R).float().contiguous(),
             "fsat_id": (s[:, None] + torch.arange(R)).long()}
        return p


def _prep_worker(rank, world, port, nq, q):
    from paper_1704_07355_b200.dist import sharded_prepare
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    qs = torch.from_numpy(np.random.default_rng(5).random((nq, 16)).astype(np.float32))
    got = sharded_prepare(_FakePrepIndex(), qs, 10, 4, 1000)
    q.put((rank, {k: v.numpy() for k, v in got.items()}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("nq", [9, 16])
def test_gloo_world2_sharded_prepare_equals_local(nq):
    """Query-sharded Index + Tables phases (dist.sharded_prepare): each of
    two ranks prepares half the batch (odd sizes padded), the halves are
    all-gathered, and every rank's state equals preparing the whole batch
    locally — except F_sat, which only the prefix owner (rank 0) keeps."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + (os.getpid() + nq) % 2000
    procs = [ctx.Process(target=_prep_worker, args=(r, world, port, nq, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    qs = torch.from_numpy(np.random.default_rng(5).random((nq, 16)).astype(np.float32))
    want = {k: v.numpy() for k, v in _FakePrepIndex().prepare(qs, 10, 4, 1000).items()}
    for rank, g in got.items():
        for k, v in want.items():
            if k == "fsat_n" and rank != 0:
                assert not g[k].any()
            else:
                assert np.array_equal(g[k], v), (rank, k)
