"""Ad-hoc GPU parity sweep vs the C oracle (developer tool)."""
import sys, time, faulthandler
faulthandler.enable()
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_1704_07355_b200 import kernels, qadc as Q, adc, ivf
from paper_1704_07355_b200.device import DeviceIndex
from oracle import oracle as orc

rng = np.random.default_rng(1)
print("level", kernels.simd_level())
# block dists
for mrows in (1, 3, 8, 16):
    blocks = rng.integers(0, 256, (50, mrows, 16), dtype=np.uint8)
    qt = rng.integers(0, 256, (2 * mrows, 16), dtype=np.uint8)
    print("block_dists", mrows, np.array_equal(kernels.block_distances(blocks, qt), orc.block_dists(blocks, qt)))
# quantize
t = (rng.random((32, 16)) * 100).astype(np.float32)
qt = Q.quantize_tables(t, 3.0, 90.0)
ot, od = orc.quantize_tables(t, 3.0, 90.0)
print("quantize", np.array_equal(qt.tables, ot), qt.delta == od)
# scan_blocks vs oracle heap
for trial in range(20):
    nb = int(rng.integers(0, 10)); mrows = int(rng.integers(1, 9)); cap = int(rng.integers(1, 25))
    blocks = rng.integers(0, 256, (nb, mrows, 16), dtype=np.uint8)
    qt = rng.integers(0, 90, (2 * mrows, 16), dtype=np.uint8)
    ids = np.arange(16 * nb, dtype=np.int64); ids[rng.random(ids.shape[0]) < 0.15] = -1
    h = Q.NeighborHeap(cap)
    pre = trial % 3 == 0
    if pre: h.push_batch(np.array([10**7, 10**7+1]), np.array([0.9, 1.8], np.float32))
    hd0, hi0, s0 = h.dists.copy(), h.ids.copy(), h.size
    kernels.scan_blocks(blocks, ids, qt, 0.25, 0.03, h)
    gi, gd = h.extract()
    oi, od = orc.qadc_scan(blocks, ids, qt, 0.25, 0.03, hd0, hi0, s0, cap)
    if not (np.array_equal(gi, oi) and np.array_equal(gd.view(np.uint32), od.view(np.uint32))):
        print("scan_blocks MISMATCH", trial, gi, oi)
print("scan_blocks done")
# batched search flat
m, d, N = 16, 128, 200000
cb = (rng.random((m, 16, d // m)) * 50).astype(np.float32)
X = (rng.random((N, d)) * 50).astype(np.float32)
idx = ivf.build_flat(Q.__class__ and type("P", (), {})(), X) if False else None
class PQ: pass
pq = PQ(); pq.m = m; pq.b = 4; pq.codebooks = cb; pq.rotation = None
codes = ivf.encode_device(pq, torch.from_numpy(X).cuda()).cpu().numpy()
tl = Q.transpose_list(codes, np.arange(N, dtype=np.int64))
index = ivf.IvfIndex(d=d, m=m, b=4, coarse=None, lists=[tl], layout="transposed16")
queries = (rng.random((64, d)) * 50).astype(np.float32)
flat = orc.flatten_index(index)
dev = DeviceIndex.from_ivf(index, pq)
for R in (1, 10, 100, 1000):
    t0 = time.time()
    res = dev.search(queries, R, init=1000)
    t1 = time.time()
    oi, od, on, diag = orc.search_batch(queries, cb, None, None, 1, flat, R, 1000)
    ok = np.array_equal(res.ids, oi) and np.array_equal(res.distances.view(np.uint32), od.view(np.uint32)) and np.array_equal(res.counts, on)
    print("flat R", R, "match", ok, "stats", res.stats, f"{(t1-t0)*1e3:.1f}ms")
    if not ok:
        bad = [q for q in range(len(queries)) if not np.array_equal(res.ids[q], oi[q])]
        print(" bad queries", bad[:10], res.ids[bad[0]][:10], oi[bad[0]][:10])
