"""(query, list) pairs per probed list at an IVF config, weighted by the
codes they scan (developer tool: how much of the scan sits in lists with
few / many queries — the PRMT vs tensor-core split).

    python tools/list_stats.py cfg4
"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1704_07355_b200.workload import IVF_CONFIGS, build_ivf_index, load_ivf_model, queries

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
cfg = IVF_CONFIGS[name]
pq, coarse = load_ivf_model(cfg)
index, sizes, rows, ids, row_off = build_ivf_index(cfg, pq, coarse, cfg.n)
qs = torch.from_numpy(queries(cfg)).cuda()
t = index.tables(qs, cfg.R, ma=cfg.nprobe, init=cfg.init)
cells = t["cells"].cpu().numpy().ravel()
pairs = np.bincount(cells, minlength=cfg.K)
work = pairs * sizes  # codes scanned per list
tot = work.sum()
print(f"{name}: pairs {cells.size}, lists probed {np.count_nonzero(pairs)} of {cfg.K}, "
      f"codes scanned {tot:.4g}")
for lo, hi in [(1, 4), (5, 8), (9, 16), (17, 32), (33, 64), (65, 128), (129, 256), (257, 10**9)]:
    m = (pairs >= lo) & (pairs <= hi)
    print(f"  pairs/list {lo:4d}-{hi:<10d}: lists {m.sum():6d}  share of scanned codes "
          f"{work[m].sum() / tot:6.3f}  mean list {sizes[m].mean() if m.any() else 0:9.0f}")
