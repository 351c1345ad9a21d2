"""Diagnostic: quantized-LUT statistics of the bench workload (how large
are table entries and the q-thresholds? decides the byte-sum depth)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_1704_07355_b200.workload import CONFIGS, load_pq, shard_codes, queries
from paper_1704_07355_b200.adc import compute_tables
from paper_1704_07355_b200.qadc import quantize_tables, find_qmax, transpose_list
from paper_1704_07355_b200.pq_util import unpack_codes
from paper_1704_07355_b200.device import DeviceIndex

for name in sys.argv[1:] or ["cfg1"]:
    cfg = CONFIGS[name]
    pq = load_pq(cfg)
    n = min(cfg.n, 2_000_000)
    codes = shard_codes(cfg, pq, n, 0)
    idx = DeviceIndex.from_device_rows(pq.d, pq.m, codes, torch.tensor([0, n], device='cuda'),
                                       torch.from_numpy(pq.codebooks).cuda())
    qs = queries(cfg, 16)
    res = idx.search(qs, cfg.R, init=cfg.init)
    cn = codes[:16384].cpu().numpy()
    un = unpack_codes(cn, pq.m).astype(np.int64)
    tl = transpose_list(codes[:1000].cpu().numpy(), np.arange(1000))
    rows = []
    for i, q in enumerate(qs):
        t = compute_tables(pq, q).tables
        qmax = find_qmax([(t, tl)], cfg.R, cfg.init)
        qmin = min(float(t.min()), qmax)
        qt = quantize_tables(t, qmin, qmax)
        lane = qt.tables[np.arange(pq.m)[None, :], un].astype(np.int64).sum(1)
        thr0 = np.sort(lane)[cfg.R - 1]
        dR = res.distances[i, cfg.R - 1]
        qR = (dR - np.float32(qt.qmin)) / np.float32(qt.delta) - 0.5
        g4 = max(qt.tables[j:j + 4].max(1).sum() for j in range(0, pq.m, 4))
        rows.append((int(qt.tables.max()), float(np.mean(qt.tables.max(1))), int(thr0), float(qR), int(g4)))
    a = np.array(rows)
    print(name, "n", n, "max entry", a[:, 0].min(), a[:, 0].max(), "mean row max %.1f" % a[:, 1].mean(),
          "thr0(16K prefix) %d..%d" % (a[:, 2].min(), a[:, 2].max()),
          "final qR %.1f..%.1f" % (a[:, 3].min(), a[:, 3].max()), "G4 max", a[:, 4].max())
