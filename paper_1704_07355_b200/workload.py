"""BASELINE.json workloads built on the GPU (index-build side, not the
search hot path): synthetic mixture base vectors drawn on the device,
encoded by the GPU encoder with reference-trained codebooks
(bench_data/*_codebooks.npy), and repacked into a DeviceIndex without a
host round trip.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import datagen
from .device import DeviceIndex

BENCH_DATA = Path(__file__).resolve().parent.parent / "bench_data"


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
    n: int
    q: int
    R: int
    init: int
    K: int
    nprobe: int
    coarse_file: str
    codebooks_file: str
    rotation_file: str


IVF_CONFIGS = {
    "cfg2": IvfConfig("cfg2_ivf_opq_K4096_m32_N1e8_Q1e4", datagen.SIFT_LIKE, 32, 100_000_000,
                      10_000, 100, 1000, 4096, 16, "cfg2_coarse_K4096.npy",
                      "cfg2_m32_codebooks.npy", "cfg2_rotation.npy"),
}


def load_ivf_model(cfg: IvfConfig):
    pq = _PQ(np.load(BENCH_DATA / cfg.codebooks_file), np.load(BENCH_DATA / cfg.rotation_file))
    return pq, np.load(BENCH_DATA / cfg.coarse_file)


def build_ivf_index(cfg: IvfConfig, pq: _PQ, coarse: np.ndarray, n: int, shard: int = 0,
                    device="cuda", chunk: int = 1 << 22):
    """IVF index of n base vectors drawn on the GPU: coarse assignment,
    residual, OPQ rotation + PQ encoding (GPU encoder), lists with ids
    ascending (ivf.py:109-151). Returns the DeviceIndex and the list sizes."""
    import torch

    from .ivf import assign_device, encode_device

    C = torch.from_numpy(np.ascontiguousarray(coarse, dtype=np.float32)).to(device)
    codes = torch.empty((n, pq.m // 2), dtype=torch.uint8, device=device)
    labels = torch.empty(n, dtype=torch.int64, device=device)
    for c0 in range(0, n, chunk):
        k = min(chunk, n - c0)
        X = datagen.mixture_torch(cfg.mix, k, seed=SEED * 1000 + shard, centre_seed=CORPUS,
                                  stream=datagen.STREAM_BASE * 100 + c0 // chunk, device=device)
        lab = assign_device(coarse, X)
        labels[c0:c0 + k] = lab
        codes[c0:c0 + k] = encode_device(pq, X - C[lab])
        del X
    order = torch.argsort(labels, stable=True)
    sizes = torch.bincount(labels, minlength=C.shape[0])
    row_off = torch.zeros(C.shape[0] + 1, dtype=torch.int64, device=device)
    row_off[1:] = torch.cumsum(sizes, 0)
    sorted_codes = codes[order].contiguous()
    del codes, labels
    index = DeviceIndex.from_device_rows(
        pq.d, pq.m, sorted_codes, row_off, torch.from_numpy(pq.codebooks).to(device),
        rotation=torch.from_numpy(np.ascontiguousarray(pq.rotation, np.float32)).to(device),
        coarse=C, ids=order + shard * n)
    return index, sizes.cpu().numpy(), sorted_codes, order, row_off
