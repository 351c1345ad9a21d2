"""BASELINE config 4 model (IVF K=65536 + OPQ, m=32 x 4-bit): the coarse
centroids of bench_data/cfg4_coarse_K65536.npy (GPU Lloyd on 2^21 learn
vectors, tools/train_coarse.py — the reference's NumPy k-means cannot train
K=65536), config 2's seeded orthogonal rotation, and residual PQ
codebooks trained by the REFERENCE's train_pq (pq.py:130-141) on the rotated
residuals of 10^5 learn vectors (assignment by the reference's
kmeans.assign_batch).

    python bench_data/make_cfg4.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent / "tests" / "golden"))
from make_golden import load_reference  # noqa: E402

from paper_1704_07355_b200 import datagen  # noqa: E402

if __name__ == "__main__":
    load_reference()
    from qadc import kmeans
    from qadc import pq as rpq
    coarse = np.load(HERE / "cfg4_coarse_K65536.npy")
    R = np.load(HERE / "cfg2_rotation.npy")
    learn = datagen.mixture_numpy(datagen.SIFT_LIKE, 100_000, seed=0, stream=datagen.STREAM_LEARN)
    labels, _ = kmeans.assign_batch(coarse, learn)
    resid = learn - coarse[labels]
    pq = rpq.train_pq((resid @ R.T).astype(np.float32), m=32, b=4, iters=25, seed=0)
    np.save(HERE / "cfg4_m32_codebooks.npy", pq.codebooks.astype(np.float32))
    print("cfg4 model written", pq.codebooks.shape)
