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
        print(f"[{st or 'default'}] {out.stdout.strip()} {out.stderr.strip()[-300:]}", flush=True)
    sys.exit(0)

import torch

from paper_1704_07355_b200.workload import IVF_CONFIGS, load_ivf_model, make_ivf_index, queries
cfg = IVF_CONFIGS[name]
pq, coarse = load_ivf_model(cfg)
d = torch.load(cache)
index = make_ivf_index(pq, coarse, d["rows"].cuda(), d["ids"].cuda(), d["row_off"].cuda())
del d
qs = torch.from_numpy(queries(cfg)).cuda()
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
print(json.dumps({"step_ms": round(e0.elapsed_time(e1) / 5, 3), "scan_ms": round(scan / 5e3, 3),
                  "cand_per_query": round(cand / 5 / qs.shape[0], 1)}))
