"""Train the PQ codebooks of BASELINE.json configs 0, 1 and 3 with the
REFERENCE's own trainer (qadc.pq.train_pq, pq.py:130-141) on 10^5 learn
vectors from the configs' mixture generator, and store them here as .npy
(8 KiB / 60 KiB). Codebook training stays in the reference (north_star);
bench.py only loads the result. Run in the build container:

    python bench_data/make_codebooks.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent / "tests" / "golden"))
from make_golden import load_reference  # noqa: E402

from paper_1704_07355_b200 import datagen  # noqa: E402

CONFIGS = {
    "cfg0_m16": (datagen.SIFT_LIKE, 16),
    "cfg1_m32": (datagen.SIFT_LIKE, 32),
    "cfg3_m32_d960": (datagen.GIST_LIKE, 32),
}

if __name__ == "__main__":
    load_reference()
    from qadc import pq as rpq
    for name, (mix, m) in CONFIGS.items():
        out = HERE / f"{name}_codebooks.npy"
        if out.exists():
            continue
        learn = datagen.mixture_numpy(mix, 100_000, seed=0, stream=datagen.STREAM_LEARN)
        pq = rpq.train_pq(learn, m=m, b=4, iters=25, seed=0)
        np.save(out, pq.codebooks.astype(np.float32))
        print(name, pq.codebooks.shape, flush=True)
