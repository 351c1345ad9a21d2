"""Developer tool: host-side overhead of one batched search (wall time per
call vs device time of its kernels).  python tools/host_overhead.py"""
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_1704_07355_b200.workload import CONFIGS, build_shard_index, load_pq, queries

cfg = CONFIGS["cfg1"]
pq = load_pq(cfg)
index, _ = build_shard_index(cfg, pq, cfg.n, 0, 1, prefix=1000)
qa = torch.from_numpy(queries(cfg, cfg.q)).cuda()
for nq in (1, 16, 1000):
    q = qa[:nq].contiguous()
    for _ in range(3):
        index.search(q, 100, init=1000)
    torch.cuda.synchronize()
    n = 20
    t0 = time.perf_counter()
    scan = 0
    for _ in range(n):
        r = index.search(q, 100, init=1000)
        scan += r.stats["scan_us"]
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n * 1e3
    print(f"nq={nq}: wall {wall:.3f} ms/search, scan {scan / n / 1e3:.3f} ms, launches {r.stats['launches']}",
          flush=True)
