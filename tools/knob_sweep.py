"""Developer tool: time the batched search of an IVF config under several
environment-knob settings without rebuilding the index each time (the
row-ordered index is cached under /dev/shm or /tmp once; each setting runs
in a fresh process because the knobs are read once per process).

    python tools/knob_sweep.py cfg4 "" "QADC_B200_RANK_BUCKETS=1" "QADC_B200_NO_HALF=1"
"""
import json
import os
import shutil
import subprocess
import sys
import time

sys.path.insert(0, ".")

name = sys.argv[1]
settings = sys.argv[2:] or [""]
cache_dir = "/dev/shm" if shutil.disk_usage("/dev/shm").free > 40e9 else "/tmp"
cache = os.path.join(cache_dir, f"qadc_{name}_rows.pt")

if os.environ.get("KNOB_CHILD") != "1":
    if not os.path.exists(cache):
        import torch

        from paper_1704_07355_b200.workload import IVF_CONFIGS, ivf_rows, load_ivf_model
        cfg = IVF_CONFIGS[name]
        pq, coarse = load_ivf_model(cfg)
        t0 = time.perf_counter()
        rows, ids, row_off = ivf_rows(cfg, pq, coarse, cfg.n)
        torch.save({"rows": rows.cpu(), "ids": ids.cpu(), "row_off": row_off.cpu()}, cache)
        print(f"built + cached in {time.perf_counter() - t0:.0f} s -> {cache}", flush=True)
        del rows, ids, row_off
    for st in settings:
        env = dict(os.environ, KNOB_CHILD="1")
        for kv in filter(None, st.split(";")):
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, __file__, name, st], env=env, capture_output=True,
                             text=True)
        print(f"[{st or 'default'}] {out.stdout.strip()} {out.stderr.strip()[-1500:]}", flush=True)
    sys.exit(0)

import torch

from paper_1704_07355_b200.workload import IVF_CONFIGS, load_ivf_model, make_ivf_index, queries
cfg = IVF_CONFIGS[name]
pq, coarse = load_ivf_model(cfg)
d = torch.load(cache)
index = make_ivf_index(pq, coarse, d["rows"].cuda(), d["ids"].cuda(), d["row_off"].cuda())
del d
qs = torch.from_numpy(queries(cfg)).cuda()
if os.environ.get("KNOB_Q"):  # a smaller batch (the scan-kernel heuristic depends on queries per list)
    qs = qs[:int(os.environ["KNOB_Q"])].contiguous()
if os.environ.get("KNOB_LIST_STATS") == "1":  # (query, list) pairs per list, weighted by scanned codes
    import numpy as np
    ro = torch.load(cache)["row_off"].numpy()
    sizes = np.diff(ro)
    cells = index.tables(qs, cfg.R, ma=cfg.nprobe, init=cfg.init)["cells"].cpu().numpy().ravel()
    pairs = np.bincount(cells, minlength=cfg.K)
    work = pairs * sizes
    tot = work.sum()
    print(f"pairs {cells.size} lists probed {np.count_nonzero(pairs)} codes scanned {tot:.4g} "
          f"codes in probed lists {sizes[pairs > 0].sum():.4g}", file=sys.stderr)
    for lo, hi in [(1, 4), (5, 8), (9, 12), (13, 16), (17, 24), (25, 32), (33, 48), (49, 64), (65, 128), (129, 10**9)]:
        mk = (pairs >= lo) & (pairs <= hi)
        print(f" {lo}-{hi}: lists {mk.sum()} work {work[mk].sum() / tot:.3f} codes {sizes[mk].sum():.3g} "
              f"mean {sizes[mk].mean() if mk.any() else 0:.0f};", file=sys.stderr)
for _ in range(3):
    index.search(qs, cfg.R, ma=cfg.nprobe, init=cfg.init)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
scan, cand = 0, 0
e0.record()
for _ in range(5):
    r = index.search(qs, cfg.R, ma=cfg.nprobe, init=cfg.init)
    scan += r.stats["scan_us"]
    cand += r.stats["candidates"]
e1.record()
torch.cuda.synchronize()
if os.environ.get("KNOB_COMPARE") == "1":  # tensor-core vs PRMT scan on the same index: ids and distance bits
    out = {}
    for mode in ("prmt", os.environ.get("KNOB_COMPARE_MODE", "auto")):
        for _ in range(2):
            r = index.search(qs, cfg.R, ma=cfg.nprobe, init=cfg.init, scan=mode)
        out[mode] = (r.ids.clone(), r.distances.clone().view(torch.int32), r.counts.clone(), r.stats["scan_us"] / 1e3,
                     r.stats["candidates"] / qs.shape[0])
    a, b = out["prmt"], out[os.environ.get("KNOB_COMPARE_MODE", "auto")]
    ok_i = (a[0] == b[0]).all(dim=1)
    ok_d = (a[1] == b[1]).all(dim=1)
    print(f"compare: prmt scan {a[3]:.2f} ms ({a[4]:.0f} cand/q), {os.environ.get("KNOB_COMPARE_MODE", "auto")} scan {b[3]:.2f} ms ({b[4]:.0f} cand/q); "
          f"ids exact {int(ok_i.sum())}/{qs.shape[0]}, dist bits exact {int(ok_d.sum())}/{qs.shape[0]}, "
          f"counts equal {bool((a[2] == b[2]).all())}", file=sys.stderr)
if os.environ.get("KNOB_PROFILE") == "1":  # per-kernel device time of one search (torch profiler)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            index.search(qs, cfg.R, ma=cfg.nprobe, init=cfg.init)
        torch.cuda.synchronize()
    rows = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            t = rows.setdefault(ev.name, [0.0, 0])
            t[0] += ev.device_time
            t[1] += 1
    for k, (us, c) in sorted(rows.items(), key=lambda kv: -kv[1][0])[:14]:
        k = k.replace("qadc::(anonymous namespace)::", "").replace("void ", "")
        print(f"  {us / 3 / 1e3:8.3f} ms x{c // 3:<2d} {k[:40]}", file=sys.stderr)
print(json.dumps({"step_ms": round(e0.elapsed_time(e1) / 5, 3), "scan_ms": round(scan / 5e3, 3),
                  "cand_per_query": round(cand / 5 / qs.shape[0], 1)}))
