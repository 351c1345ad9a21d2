"""Offline index-build helper: coarse quantizer for the IVF configs
(BASELINE configs 2 and 4) trained on the GPU.

The reference's k-means (kmeans.py:130-151, NumPy Lloyd with k-means++
seeding) is infeasible at K=4096 on 10^6 samples (hours) and at K=65536
(SURVEY 7 "Config-4 index build"), so this tool runs Lloyd iterations with
the reference's assignment semantics on the GPU: einsum-order squared
distances with ties to the lowest centroid (qadc_b200_assign), mean update,
empty clusters re-seeded from the farthest points (kmeans.py:110-127
restated). Seeding is a seeded random sample (not k-means++). The result is
an input of the index, not part of the search path; parity is defined
given the same index.

    python tools/train_coarse.py --K 4096 --n 1000000 --iters 12 \
        --out bench_data/cfg2_coarse_K4096.npy
"""

import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_1704_07355_b200 import datagen
    from paper_1704_07355_b200.ivf import assign_device

    p = argparse.ArgumentParser()
    p.add_argument("--K", type=int, default=4096)
    p.add_argument("--n", type=int, default=1_000_000)
    p.add_argument("--iters", type=int, default=12)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", required=True)
    a = p.parse_args()
    X = torch.from_numpy(datagen.mixture_numpy(datagen.SIFT_LIKE, a.n, seed=0,
                                               stream=datagen.STREAM_LEARN)).cuda()
    g = torch.Generator(device="cpu").manual_seed(a.seed)
    C = X[torch.randperm(a.n, generator=g)[: a.K].cuda()].clone()
    for it in range(a.iters):
        lab = assign_device(C.cpu().numpy(), X)
        cnt = torch.bincount(lab, minlength=a.K)
        S = torch.zeros_like(C).index_add_(0, lab, X)
        newC = S / cnt.clamp(min=1).unsqueeze(1).to(S.dtype)
        empty = (cnt == 0).nonzero().flatten()
        if empty.numel():
            d = ((X - C[lab]) ** 2).sum(1)
            far = torch.argsort(d, descending=True)[: empty.numel()]
            newC[empty] = X[far]
        shift = float(((newC - C) ** 2).sum(1).max())
        C = newC
        print(f"iter {it}: empty {empty.numel()} max shift {shift:.4g}", flush=True)
    np.save(a.out, C.cpu().numpy().astype(np.float32))
    print("saved", a.out, tuple(C.shape))


if __name__ == "__main__":
    main()
