"""BASELINE.json workloads built on the GPU (index-build side, not the
search hot path): synthetic mixture base vectors drawn on the device,
encoded by the GPU encoder with reference-trained codebooks
(bench_data/*_codebooks.npy), and repacked into a DeviceIndex without a
host round trip.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import os

import numpy as np

from . import datagen
from .device import DeviceIndex

BENCH_DATA = Path(__file__).resolve().parent.parent / "bench_data"

_TIMING = os.environ.get("QADC_BUILD_TIMING") == "1"
BUILD_TIMES: dict = {}


class _phase:
    """Accumulates device-synchronised wall time of an index-build phase
    into BUILD_TIMES when QADC_BUILD_TIMING=1 (developer diagnostics)."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        if _TIMING:
            import time

            import torch
            torch.cuda.synchronize()
            self.t = time.perf_counter()
        return self

    def __exit__(self, *a):
        if _TIMING:
            import time

            import torch
            torch.cuda.synchronize()
            BUILD_TIMES[self.name] = BUILD_TIMES.get(self.name, 0.0) + time.perf_counter() - self.t


@dataclass(frozen=True)
class FlatConfig:
    name: str
    mix: datagen.Mixture
    m: int
    n: int
    q: int
    R: int
    init: int
    codebooks_file: str


CONFIGS = {
    "cfg0": FlatConfig("cfg0_exhaustive_m16_N1e6_Q100", datagen.SIFT_LIKE, 16, 1_000_000, 100,
                       100, 1000, "cfg0_m16_codebooks.npy"),
    "cfg1": FlatConfig("cfg1_exhaustive_m32_N1e7_Q1000", datagen.SIFT_LIKE, 32, 10_000_000,
                       1000, 100, 1000, "cfg1_m32_codebooks.npy"),
    "cfg3": FlatConfig("cfg3_exhaustive_d960_m32_N1e6_Q1000", datagen.GIST_LIKE, 32, 1_000_000,
                       1000, 100, 1000, "cfg3_m32_d960_codebooks.npy"),
}

SEED = 1
# every split (learn: bench_data/make_*.py, base, queries) draws around the
# centres of corpus 0, so queries come from the base's distribution
CORPUS = 0


class _PQ:
    """Minimal ProductQuantizer-shaped holder (codebooks trained by the
    reference, loaded from bench_data)."""

    def __init__(self, codebooks: np.ndarray, rotation=None):
        self.codebooks = np.ascontiguousarray(codebooks, dtype=np.float32)
        self.m = self.codebooks.shape[0]
        self.b = 4
        self.rotation = rotation

    @property
    def d(self) -> int:
        return self.m * self.codebooks.shape[2]


def load_pq(cfg: FlatConfig) -> _PQ:
    return _PQ(np.load(BENCH_DATA / cfg.codebooks_file))


def shard_codes(cfg: FlatConfig, pq: _PQ, n: int, shard: int, device="cuda"):
    """Packed codes (n, m/2) of base shard `shard` (drawn + encoded on GPU)."""
    import torch

    from .ivf import encode_device

    out = torch.empty((n, pq.m // 2), dtype=torch.uint8, device=device)
    step = datagen.CHUNK
    for c0 in range(0, n, 4 * step):
        k = min(4 * step, n - c0)
        X = datagen.mixture_torch(cfg.mix, k, seed=SEED * 1000 + shard, centre_seed=CORPUS,
                                  stream=datagen.STREAM_BASE * 100 + c0 // (4 * step),
                                  device=device)
        out[c0:c0 + k] = encode_device(pq, X)
        del X
    return out


def queries(cfg: FlatConfig, q: int | None = None) -> np.ndarray:
    return datagen.mixture_numpy(cfg.mix, q or cfg.q, seed=SEED, stream=datagen.STREAM_QUERY,
                                 centre_seed=CORPUS)


def build_shard_index(cfg: FlatConfig, pq: _PQ, n: int, rank: int, world: int, prefix: int):
    """DeviceIndex over shard `rank` of a flat list of world * n codes
    (global ids rank * n + i). For world > 1 every shard also installs the
    GLOBAL prefix (the first `prefix` codes = the start of shard 0) so
    qmax and the saturation rule match the unsharded search."""
    import torch

    codes = shard_codes(cfg, pq, n, rank)
    dev = torch.device("cuda")
    row_off = torch.tensor([0, n], dtype=torch.int64, device=dev)
    ids = torch.arange(rank * n, (rank + 1) * n, dtype=torch.int64, device=dev)
    cb = torch.from_numpy(pq.codebooks).to(dev)
    index = DeviceIndex.from_device_rows(pq.d, pq.m, codes, row_off, cb, ids=ids)
    if world > 1:
        p = min(prefix, n)
        head = codes[:p] if rank == 0 else shard_codes(cfg, pq, min(n, datagen.CHUNK), 0)[:p]
        index.set_prefix(head.contiguous(), torch.tensor([0, p], dtype=torch.int64, device=dev),
                         [world * n], ids=torch.arange(p, dtype=torch.int64, device=dev))
    return index, codes


# ------------------------------------------------------------------ IVF


@dataclass(frozen=True)
class IvfConfig:
    name: str
    mix: datagen.Mixture
    m: int
    n: int  # total codes (list-sharded and range-sharded configs alike)
    q: int
    R: int
    init: int
    K: int
    nprobe: int
    coarse_file: str  # bench_data/: GPU Lloyd (tools/train_coarse.py)
    codebooks_file: str
    rotation_file: str
    sharding: str  # "lists" (config 2) or "range" (config 4)


IVF_CONFIGS = {
    "cfg2": IvfConfig("cfg2_ivf_opq_K4096_m32_N1e8_Q1e4", datagen.SIFT_LIKE, 32, 100_000_000,
                      10_000, 100, 1000, 4096, 16, "cfg2_coarse_K4096.npy",
                      "cfg2_m32_codebooks.npy", "cfg2_rotation.npy", "lists"),
    "cfg4": IvfConfig("cfg4_ivf_opq_K65536_m32_N1e9_Q1e4", datagen.SIFT_LIKE, 32, 1_000_000_000,
                      10_000, 100, 1000, 65536, 64, "cfg4_coarse_K65536.npy",
                      "cfg4_m32_codebooks.npy", "cfg2_rotation.npy", "range"),
}

# config 4 base: a global grid of 10^6-vector chunks (chunk g = ids
# g*10^6 ..), so every range shard of 1, 2, 4 or 8 GPUs draws exactly its
# own chunks and the dataset does not depend on the GPU count
CFG4_CHUNK = 1_000_000


def load_ivf_model(cfg: IvfConfig):
    pq = _PQ(np.load(BENCH_DATA / cfg.codebooks_file), np.load(BENCH_DATA / cfg.rotation_file))
    return pq, np.load(BENCH_DATA / cfg.coarse_file)


def assign_tensor_core(X, C, cn=None, chunk: int = 16384):
    """Index-build coarse assignment on the tensor cores: argmin over
    ||c||^2 - 2 x.c with TF32 cuBLAS GEMMs (cuBLAS for a plain library GEMM;
    not the search path). Near-ties may resolve differently from the exact
    einsum order of qadc_b200_assign; the index is whatever this produces
    and parity is defined given the index."""
    import torch

    if cn is None:
        cn = (C.double() ** 2).sum(1).float()
    out = torch.empty(X.shape[0], dtype=torch.int64, device=X.device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        Ct = C.t().contiguous()
        for i in range(0, X.shape[0], chunk):
            S = torch.addmm(cn, X[i:i + chunk], Ct, beta=1.0, alpha=-2.0)
            out[i:i + chunk] = S.argmin(1)
            del S
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out


def _sorted_rows(codes, labels, ids, K):
    """Row-ordered lists: stable sort by cell (ids stay ascending in every
    list, ivf.py:109-151), row offsets."""
    import torch

    order = torch.argsort(labels, stable=True)
    sizes = torch.bincount(labels, minlength=K)
    row_off = torch.zeros(K + 1, dtype=torch.int64, device=codes.device)
    row_off[1:] = torch.cumsum(sizes, 0)
    return codes[order].contiguous(), ids[order].contiguous(), row_off


def ivf_rows(cfg: IvfConfig, pq: _PQ, coarse: np.ndarray, n: int, device="cuda",
             chunk: int = 1 << 22, rank: int = 0, world: int = 1):
    """Base vectors drawn on the GPU, coarse-assigned, residual + OPQ + PQ
    encoded (GPU encoder), grouped into row-ordered lists.

    Config 2 (list sharding): the whole base of n codes (every rank builds
    it; `shard_ivf_lists` keeps the rank's lists). Config 4 (range
    sharding): rank r draws the chunks of its id range of the global
    CFG4_CHUNK grid. Both assign with qadc_b200_assign (exact einsum-order
    nearest centroid, ties to the lower index, on the fused tensor-core
    kernel); the index is an input of the search path and parity is
    defined given the index.
    Returns (codes (n_r, m/2), ids (n_r,), row_off (K + 1,))."""
    import torch

    from .ivf import assign_device, encode_device

    C = torch.from_numpy(np.ascontiguousarray(coarse, dtype=np.float32)).to(device)
    cn = (C.double() ** 2).sum(1).float()
    if cfg.sharding == "range":
        nch = -(-n // CFG4_CHUNK)
        per = -(-nch // world)
        gs = range(rank * per, min(nch, (rank + 1) * per))
        spans = [(g * CFG4_CHUNK, min(n, (g + 1) * CFG4_CHUNK), g) for g in gs]
    else:
        spans = [(c0, min(n, c0 + chunk), c0 // chunk) for c0 in range(0, n, chunk)]
    tot = sum(b - a for a, b, _ in spans)
    codes = torch.empty((tot, pq.m // 2), dtype=torch.uint8, device=device)
    labels = torch.empty(tot, dtype=torch.int64, device=device)
    ids = torch.empty(tot, dtype=torch.int64, device=device)
    o = 0
    for a, b, g in spans:
        k = b - a
        with _phase("generate"):
            if cfg.sharding == "range":
                X = datagen.mixture_torch(cfg.mix, k, seed=SEED * 1000 + 4, centre_seed=CORPUS,
                                          stream=datagen.STREAM_BASE * 100_000 + g, device=device)
            else:
                X = datagen.mixture_torch(cfg.mix, k, seed=SEED * 1000, centre_seed=CORPUS,
                                          stream=datagen.STREAM_BASE * 100 + g, device=device)
        with _phase("assign"):
            # nearest coarse centroid, exact einsum order (qadc_b200_assign:
            # the fused tcgen05 nearest-centroid kernel + exact re-rank)
            lab = assign_device(C, X)
        labels[o:o + k] = lab
        with _phase("encode"):
            codes[o:o + k] = encode_device(pq, X - C[lab])
        ids[o:o + k] = torch.arange(a, b, dtype=torch.int64, device=device)
        o += k
        del X, lab
    with _phase("sort"):
        rows, rid, row_off = _sorted_rows(codes, labels, ids, C.shape[0])
    del codes, labels, ids
    return rows, rid, row_off


def base_chunks(cfg, n: int, device="cuda"):
    """(offset, vectors) chunks of the base exactly as the index build draws
    it (same seeds and chunk grid; shard 0 of an exhaustive config), for
    the recall harness's ground truth."""
    if isinstance(cfg, IvfConfig) and cfg.sharding == "range":
        for g in range(-(-n // CFG4_CHUNK)):
            a, b = g * CFG4_CHUNK, min(n, (g + 1) * CFG4_CHUNK)
            yield a, datagen.mixture_torch(cfg.mix, b - a, seed=SEED * 1000 + 4,
                                           centre_seed=CORPUS,
                                           stream=datagen.STREAM_BASE * 100_000 + g, device=device)
        return
    step = 4 * datagen.CHUNK  # == ivf_rows' list-sharded chunk (1 << 22)
    for c0 in range(0, n, step):
        yield c0, datagen.mixture_torch(cfg.mix, min(step, n - c0), seed=SEED * 1000,
                                        centre_seed=CORPUS,
                                        stream=datagen.STREAM_BASE * 100 + c0 // step,
                                        device=device)


def encode_torch(pq: _PQ, resid):
    """pq.encode_batch (pq.py:210-217) restated in plain torch for the
    REFERENCE arm's index setup (no product kernels in that process):
    rotation x @ R^T in fp32 (TF32 off), per sub-space argmin of
    ||c||^2 - 2 y.c (ties to the lowest index), two sub-codes per byte,
    low nibble first (pq.py:90-105). Near-tie codes may differ from the
    GPU encoder's exact einsum form; the index is an input of the timed
    path."""
    import torch

    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        y = resid
        if pq.rotation is not None:
            y = resid @ torch.from_numpy(np.ascontiguousarray(pq.rotation, np.float32)).to(
                resid.device).t()
        cb = torch.from_numpy(pq.codebooks).to(resid.device)  # (m, 16, dsub)
        m, dsub = cb.shape[0], cb.shape[2]
        sc = (cb * cb).sum(-1)[None] - 2.0 * torch.einsum("njd,jkd->njk",
                                                         y.view(-1, m, dsub), cb)
        c = sc.argmin(-1).to(torch.uint8)  # (n, m)
        return (c[:, 0::2] | (c[:, 1::2] << 4)).contiguous()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def ivf_rows_torch(cfg: IvfConfig, pq: _PQ, coarse: np.ndarray, n: int, keep, device="cuda"):
    """Reference-arm index setup in plain torch (no product library): the
    same seeded base as ivf_rows (configs 4 / 2 chunk grids), the same
    TF32 coarse assignment, and encode_torch for the members of the lists
    flagged in `keep` (bool, K) only — the CPU sample scans nothing else.
    Returns (codes, ids, row_off) row-ordered, other lists empty."""
    import torch

    C = torch.from_numpy(np.ascontiguousarray(coarse, dtype=np.float32)).to(device)
    cn = (C.double() ** 2).sum(1).float()
    keep_d = torch.as_tensor(keep, dtype=torch.bool, device=device)
    if cfg.sharding == "range":
        spans = [(g * CFG4_CHUNK, min(n, (g + 1) * CFG4_CHUNK), g)
                 for g in range(-(-n // CFG4_CHUNK))]
    else:
        chunk = 1 << 22
        spans = [(c0, min(n, c0 + chunk), c0 // chunk) for c0 in range(0, n, chunk)]
    codes, labels, ids = [], [], []
    for a, b, g in spans:
        k = b - a
        if cfg.sharding == "range":
            X = datagen.mixture_torch(cfg.mix, k, seed=SEED * 1000 + 4, centre_seed=CORPUS,
                                      stream=datagen.STREAM_BASE * 100_000 + g, device=device)
        else:
            X = datagen.mixture_torch(cfg.mix, k, seed=SEED * 1000, centre_seed=CORPUS,
                                      stream=datagen.STREAM_BASE * 100 + g, device=device)
        lab = assign_tensor_core(X, C, cn)
        sel = keep_d[lab].nonzero().flatten()
        if sel.numel():
            codes.append(encode_torch(pq, X[sel] - C[lab[sel]]))
            labels.append(lab[sel])
            ids.append(sel + a)
        del X, lab
    if not codes:
        z = torch.zeros(0, dtype=torch.int64, device=device)
        return (torch.zeros((0, pq.m // 2), dtype=torch.uint8, device=device), z,
                torch.zeros(C.shape[0] + 1, dtype=torch.int64, device=device))
    return _sorted_rows(torch.cat(codes), torch.cat(labels), torch.cat(ids), C.shape[0])


def make_ivf_index(pq: _PQ, coarse: np.ndarray, rows, ids, row_off, device="cuda"):
    import torch

    return DeviceIndex.from_device_rows(
        pq.d, pq.m, rows, row_off, torch.from_numpy(pq.codebooks).to(device),
        rotation=torch.from_numpy(np.ascontiguousarray(pq.rotation, np.float32)).to(device),
        coarse=torch.from_numpy(np.ascontiguousarray(coarse, np.float32)).to(device), ids=ids)


def build_ivf_index(cfg: IvfConfig, pq: _PQ, coarse: np.ndarray, n: int, shard: int = 0,
                    device="cuda", chunk: int = 1 << 22):
    """Unsharded IVF index of n base vectors (configs 2 and 4 on one GPU).
    Returns the DeviceIndex, list sizes, and the row-ordered (codes, ids,
    row_off) it was built from."""
    rows, ids, row_off = ivf_rows(cfg, pq, coarse, n, device=device, chunk=chunk)
    with _phase("index_create"):
        index = make_ivf_index(pq, coarse, rows, ids, row_off, device)
    sizes = (row_off[1:] - row_off[:-1]).cpu().numpy()
    return index, sizes, rows, ids, row_off


def build_sharded_ivf_index(cfg: IvfConfig, pq: _PQ, coarse: np.ndarray, n: int, rank: int,
                            world: int, prefix: int, device="cuda"):
    """This rank's shard of an IVF index plus the GLOBAL prefix of every
    list. Config 2: greedy list sharding, every rank draws the
    whole base and keeps its lists. Config 4: range sharding, each rank
    draws only its id range; the prefix heads move over NCCL
    (shard.gather_prefix). Returns (index, rows, ids, row_off) of the
    rank's part."""
    import torch

    from . import shard

    if cfg.sharding == "lists":
        rows, ids, row_off = ivf_rows(cfg, pq, coarse, n, device=device)
        cnt = row_off[1:] - row_off[:-1]
        need = torch.clamp(cnt, max=prefix)
        prow, pid = shard.take_heads(rows, ids, row_off, need)
        poff = torch.zeros_like(row_off)
        poff[1:] = torch.cumsum(need, 0)
        owner = torch.from_numpy(shard.assign_lists(cnt.cpu().numpy(), world)).to(device)
        full_count = cnt
        rows, ids, row_off = shard.keep_lists(rows, ids, row_off, owner == rank)
    else:
        rows, ids, row_off = ivf_rows(cfg, pq, coarse, n, device=device, rank=rank, world=world)
        prow, pid, poff, full_count = shard.gather_prefix(rows, ids, row_off, prefix)
    index = make_ivf_index(pq, coarse, rows, ids, row_off, device)
    index.set_prefix(prow.contiguous(), poff, full_count.cpu().numpy(), ids=pid.contiguous())
    return index, rows, ids, row_off
