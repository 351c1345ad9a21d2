"""Developer tool: scan time vs R at configs[1] (hit-path cost scales with
the candidate count, ~R ln(N / prefix)).  python tools/r_sweep.py"""
import sys

sys.path.insert(0, ".")
import torch

from paper_1704_07355_b200.workload import CONFIGS, build_shard_index, load_pq, queries

cfg = CONFIGS["cfg1"]
pq = load_pq(cfg)
index, _ = build_shard_index(cfg, pq, cfg.n, 0, 1, prefix=1000)
q = torch.from_numpy(queries(cfg, cfg.q)).cuda()
for R in (1, 10, 100, 1000):
    for _ in range(3):
        res = index.search(q, R, init=1000)
    us = []
    for _ in range(5):
        res = index.search(q, R, init=1000)
        us.append(res.stats["scan_us"])
    print(f"R={R} scan_ms={sum(us) / len(us) / 1e3:.3f} cands/query={res.stats['candidates'] / cfg.q:.0f}",
          flush=True)
