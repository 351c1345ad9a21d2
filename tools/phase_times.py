"""Per-kernel device time of one batched search (developer tool).

    python tools/phase_times.py cfg2 30000000 10000
    python tools/phase_times.py cfg1 10000000 1000

Runs the bench workload, warms up, then records 3 searches under the
CUPTI-based torch profiler and prints the per-kernel mean time per search.
Not a bench number (the profiler serialises nothing, but adds overhead
around launches); use it to see which phase dominates.
"""
import sys

sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile

from paper_1704_07355_b200.workload import (CONFIGS, IVF_CONFIGS, build_ivf_index,
                                            build_shard_index, load_ivf_model, load_pq, queries)

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else None
nq = int(float(sys.argv[3])) if len(sys.argv) > 3 else None
import time
t0 = time.perf_counter()
ivf = IVF_CONFIGS.get(name)
cfg = ivf or CONFIGS[name]
n = n or cfg.n
if ivf:
    pq, coarse = load_ivf_model(ivf)
    index = build_ivf_index(ivf, pq, coarse, n)[0]
    ma = ivf.nprobe
else:
    pq = load_pq(cfg)
    index = build_shard_index(cfg, pq, n, 0, 1, prefix=max(cfg.init, cfg.R))[0]
    ma = 1
torch.cuda.synchronize()
print(f"model+index build {time.perf_counter() - t0:.1f} s", flush=True)
from paper_1704_07355_b200.workload import BUILD_TIMES
print("build phases (QADC_BUILD_TIMING=1):", {k: round(v, 2) for k, v in BUILD_TIMES.items()}, flush=True)
qs = torch.from_numpy(queries(cfg, nq or cfg.q)).cuda()
for _ in range(3):
    index.search(qs, cfg.R, ma=ma, init=cfg.init)
torch.cuda.synchronize()
reps = 3
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        index.search(qs, cfg.R, ma=ma, init=cfg.init)
    torch.cuda.synchronize()
rows = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        t = rows.setdefault(e.name, [0.0, 0])
        t[0] += e.device_time
        t[1] += 1
tot = sum(v[0] for v in rows.values()) / reps
print(f"{name} n={n} q={qs.shape[0]}: device total {tot / 1e3:.3f} ms / search")
for k, (us, c) in sorted(rows.items(), key=lambda kv: -kv[1][0]):
    print(f"  {us / reps / 1e3:8.3f} ms  x{c // reps:<3d} {k[:90]}")
