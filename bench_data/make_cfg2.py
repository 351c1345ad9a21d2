"""BASELINE config 2 model (IVF + OPQ, m=32 x 4-bit): seeded random
orthogonal rotation (np.linalg.qr of a seeded Gaussian, as BASELINE states),
PQ codebooks trained by the REFERENCE's train_pq (pq.py:130-141) on the
rotated residuals of 10^5 learn vectors, with the coarse centroids of
bench_data/cfg2_coarse_K4096.npy (GPU Lloyd, tools/train_coarse.py;
assignment by the reference's kmeans.assign_batch).

    python bench_data/make_cfg2.py
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
    coarse = np.load(HERE / "cfg2_coarse_K4096.npy")
    rng = np.random.default_rng(2)
    R = np.linalg.qr(rng.standard_normal((128, 128)))[0].astype(np.float32)
    np.save(HERE / "cfg2_rotation.npy", R)
    learn = datagen.mixture_numpy(datagen.SIFT_LIKE, 100_000, seed=0, stream=datagen.STREAM_LEARN)
    labels, _ = kmeans.assign_batch(coarse, learn)
    resid = learn - coarse[labels]
    pq = rpq.train_pq((resid @ R.T).astype(np.float32), m=32, b=4, iters=25, seed=0)
    np.save(HERE / "cfg2_m32_codebooks.npy", pq.codebooks.astype(np.float32))
    print("cfg2 model written", pq.codebooks.shape)
