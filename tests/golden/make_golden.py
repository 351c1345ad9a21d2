"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory, builds the reference's
Cython extension there (`setup.py build_ext --inplace`, the survey-verified
recipe), imports it, and records inputs + outputs of the reference's own
functions on small seeded cases. The GPU box never runs this script; it only
reads the committed .npz files.

Fixtures (all small):
  quantize.npz     qadc.quantize_tables (incl. the test_qadc.py:89-109 KATs)
  block_dists.npz  kernels.block_distances (shared + per-block, bytes 0..255)
  scan_blocks.npz  kernels.scan_blocks with padding lanes and pre-filled heaps
  tables.npz       adc.compute_tables bit patterns (dsub 4, 8, 30)
  probe.npz        ivf.probe (K=300, d=128)
  find_qmax.npz    qadc.find_qmax (single cell, prefix, degenerate)
  search_*.npz     adc.search(method="qadc") end to end on seeded corpora
  search_cfg2_k4096.npz  configs[2]'s K=4096 + OPQ model at N=1e5 (nprobe 16, 64)

`python tests/golden/make_golden.py cfg2` regenerates only the last one.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
SCRATCH = Path(os.environ.get("QADC_REF_BUILD", "/tmp/qadc_ref_golden"))


def load_reference():
    src = SCRATCH / "src"
    if not (src / "qadc").exists() or not list((src / "qadc").glob("_kernels*.so")):
        if SCRATCH.exists():
            shutil.rmtree(SCRATCH)
        shutil.copytree("/root/reference/pkg", SCRATCH)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                       check=True, stdout=subprocess.DEVNULL)
    sys.path.insert(0, str(src))
    import qadc  # noqa: F401  (the reference package)
    return qadc


def main(only=None):
    load_reference()
    sys.path.insert(0, str(REPO))
    if only == "cfg2":
        make_search_cfg2(HERE / "search_cfg2_k4096.npz", n=100_000, nq=16, mas=(16, 64))
        return
    if only == "gt":
        make_ground_truth(HERE / "ground_truth.npz")
        return
    if only == "qivf":
        make_qivf(HERE / "ref_index.qivf", HERE / "ref_index.npz")
        return
    from qadc import adc, ivf, kernels, qadc as rq
    from qadc import pq as rpq
    from qadc.heap import NeighborHeap

    sys.path.insert(0, str(REPO))
    from paper_1704_07355_b200 import datagen

    assert kernels.have_extension()
    out = {}

    # ---- quantize_tables: KATs of tests/test_qadc.py:89-109 + random ----
    rng = np.random.default_rng(2024)
    qcases = [
        (np.array([[3.0, 300.0, 0.0, -5.0] + [10.0] * 12], np.float32), 0.0, 254.0),
        (np.full((2, 16), 7.0, np.float32), 7.0, 7.0),
    ]
    t = np.full((2, 16), 7.0, np.float32)
    t[0, 3] = 7.5
    qcases.append((t, 7.0, 7.0))
    for _ in range(40):
        m = int(rng.choice([2, 8, 16, 32, 64]))
        tab = (rng.random((m, 16)) * rng.uniform(1, 1e5)).astype(np.float32)
        lo = float(tab.min()) * float(rng.uniform(0.5, 1.0))
        hi = lo + float(rng.uniform(0, 1) * (tab.max() - lo + 1))
        qcases.append((tab, lo, hi))
    for i, (tab, lo, hi) in enumerate(qcases):
        qt = rq.quantize_tables(tab, lo, hi)
        out[f"c{i}_tables"] = tab
        out[f"c{i}_qmin"] = np.float64(lo)
        out[f"c{i}_qmax"] = np.float64(hi)
        out[f"c{i}_q"] = qt.tables
        out[f"c{i}_delta"] = np.float64(qt.delta)
    out["n"] = np.int64(len(qcases))
    np.savez_compressed(HERE / "quantize.npz", **out)

    # ---- block_distances (acceptance criterion 1 style) ----
    out = {}
    rng = np.random.default_rng(7)
    for i, mrows in enumerate([1, 4, 8, 16, 64]):
        nb = 200
        blocks = rng.integers(0, 256, (nb, mrows, 16), dtype=np.uint8)
        shared = rng.integers(0, 128, (2 * mrows, 16), dtype=np.uint8)
        per = rng.integers(0, 256, (nb, 2 * mrows, 16), dtype=np.uint8)
        out[f"c{i}_blocks"] = blocks
        out[f"c{i}_shared"] = shared
        out[f"c{i}_per"] = per
        out[f"c{i}_out_shared"] = kernels.block_distances(blocks, shared, variant="scalar")
        out[f"c{i}_out_per"] = kernels.block_distances(blocks, per, variant="scalar")
    out["n"] = np.int64(5)
    np.savez_compressed(HERE / "block_dists.npz", **out)

    # ---- scan_blocks with padding + pre-filled heaps (test_kernels.py:145-168) ----
    out = {}
    rng = np.random.default_rng(11)
    n = 0
    for trial in range(60):
        nb = int(rng.integers(0, 12))
        mrows = int(rng.integers(1, 9))
        cap = int(rng.integers(1, 40))
        blocks = rng.integers(0, 256, (nb, mrows, 16), dtype=np.uint8)
        top = int(rng.choice([40, 90, 127]))
        qt = rng.integers(0, top + 1, (2 * mrows, 16), dtype=np.uint8)
        ids = np.arange(16 * nb, dtype=np.int64) * 3
        ids[rng.random(ids.shape[0]) < 0.15] = -1
        qmin, delta = float(rng.uniform(0, 2)), float(rng.uniform(0.001, 0.2))
        heap = NeighborHeap(cap)
        pre = trial % 3 == 0
        if pre:
            heap.push_batch(np.array([10**7, 10**7 + 1], np.int64),
                            np.array([0.9, 1.8], np.float32))
        pre_i, pre_d = heap.ids[: heap.size].copy(), heap.dists[: heap.size].copy()
        kernels.scan_blocks(blocks, ids, qt, qmin, delta, heap, variant="simd256")
        gi, gd = heap.extract()
        for k, v in dict(blocks=blocks, qt=qt, ids=ids, qmin=np.float64(qmin),
                         delta=np.float64(delta), cap=np.int64(cap), pre_i=pre_i, pre_d=pre_d,
                         out_i=gi, out_d=gd).items():
            out[f"c{n}_{k}"] = v
        n += 1
    out["n"] = np.int64(n)
    np.savez_compressed(HERE / "scan_blocks.npz", **out)

    # ---- compute_tables bit patterns ----
    out = {}
    rng = np.random.default_rng(5)
    for i, (m, dsub) in enumerate([(16, 8), (32, 4), (32, 30), (8, 16), (4, 33)]):
        cb = (rng.standard_normal((m, 16, dsub)) * rng.uniform(0.1, 50)).astype(np.float32)
        pq = rpq.ProductQuantizer(m=m, b=4, codebooks=cb)
        ys = (rng.standard_normal((8, m * dsub)) * 20).astype(np.float32)
        out[f"c{i}_codebooks"] = cb
        out[f"c{i}_y"] = ys
        out[f"c{i}_tables"] = np.stack([adc.compute_tables(pq, y).tables for y in ys])
    out["n"] = np.int64(5)
    np.savez_compressed(HERE / "tables.npz", **out)

    # ---- probe ----
    cen = datagen.mixture_numpy(datagen.SIFT_LIKE, 300, seed=3, stream=1)
    qs = datagen.mixture_numpy(datagen.SIFT_LIKE, 20, seed=3, stream=3)
    from qadc.kmeans import Codebook
    fake = ivf.IvfIndex(d=128, m=16, b=4, coarse=Codebook(cen),
                        lists=[ivf.StandardList(np.zeros(0, np.int64), np.zeros((0, 8), np.uint8))
                               for _ in range(300)], layout=ivf.LAYOUT_STANDARD)
    cells, res = [], []
    for q in qs:
        ps = ivf.probe(fake, q, 16)
        cells.append(ps.cells)
        res.append(ps.residual_queries)
    np.savez_compressed(HERE / "probe.npz", centroids=cen, queries=qs, ma=np.int64(16),
                        cells=np.stack(cells), residuals=np.stack(res))

    # ---- find_qmax ----
    out = {}
    rng = np.random.default_rng(9)
    n = 0
    for (m, cnt, R, init) in [(8, 1000, 100, 200), (8, 1000, 1, 50), (8, 1000, 10, 10000),
                              (16, 37, 100, 1000), (32, 5000, 100, 1000), (4, 0, 10, 100),
                              (16, 3, 5, 2), (64, 700, 256, 1000)]:
        tab = (rng.random((m, 16)) * 100).astype(np.float32)
        codes = rng.integers(0, 256, (cnt, m // 2), dtype=np.uint8)
        tl = rq.transpose_list(codes, np.arange(cnt, dtype=np.int64))
        out[f"c{n}_tables"] = tab
        out[f"c{n}_codes"] = codes
        out[f"c{n}_R"] = np.int64(R)
        out[f"c{n}_init"] = np.int64(init)
        out[f"c{n}_qmax"] = np.float64(rq.find_qmax([(tab, tl)], R=R, init=init))
        n += 1
    out["n"] = np.int64(n)
    np.savez_compressed(HERE / "find_qmax.npz", **out)

    # ---- end-to-end searches ----
    make_search(HERE / "search_flat16.npz", datagen.SIFT_LIKE, m=16, n=20000, nq=40,
                Rs=(1, 10, 100), init=1000, opq=False, K=0, mas=(1,))
    make_search(HERE / "search_flat_hd.npz", datagen.GIST_LIKE, m=32, n=6000, nq=20,
                Rs=(100,), init=1000, opq=False, K=0, mas=(1,))
    make_search(HERE / "search_ivf_opq.npz", datagen.SIFT_LIKE, m=32, n=20000, nq=30,
                Rs=(100,), init=1000, opq=True, K=64, mas=(4, 16))
    make_search_cfg2(HERE / "search_cfg2_k4096.npz", n=100_000, nq=16, mas=(16, 64))
    print("golden fixtures written to", HERE)


def make_search(path, mix, m, n, nq, Rs, init, opq, K, mas):
    """Reference-built index + reference search results (ids, distance bits)
    and, for injected-LUT parity, the reference's per-(query, cell) tables."""
    from qadc import adc, ivf, kmeans
    from qadc import pq as rpq

    from paper_1704_07355_b200 import datagen

    learn = datagen.mixture_numpy(mix, 20000, seed=1, stream=datagen.STREAM_LEARN)
    base = datagen.mixture_numpy(mix, n, seed=1, stream=datagen.STREAM_BASE)
    queries = datagen.mixture_numpy(mix, nq, seed=1, stream=datagen.STREAM_QUERY)
    out = {"queries": queries}
    if K:
        coarse = kmeans.train(learn, K, iters=8, seed=0)
        labels, _ = kmeans.assign_batch(coarse.centroids, learn)
        resid = learn - coarse.centroids[labels]
        if opq:
            rng = np.random.default_rng(4)
            R_ = np.linalg.qr(rng.standard_normal((mix.d, mix.d)))[0].astype(np.float32)
            base_pq = rpq.train_pq(resid @ R_.T, m=m, b=4, iters=8, seed=0)
            pq = rpq.ProductQuantizer(m=m, b=4, codebooks=base_pq.codebooks, rotation=R_)
        else:
            pq = rpq.train_pq(resid, m=m, b=4, iters=8, seed=0)
        index = ivf.build(pq, coarse_k=K, base=base, iters=8, seed=0,
                          layout=ivf.LAYOUT_TRANSPOSED, learn=learn)
        out["coarse"] = index.coarse.centroids
    else:
        pq = rpq.train_pq(learn, m=m, b=4, iters=8, seed=0)
        index = ivf.build_flat(pq, base, layout=ivf.LAYOUT_TRANSPOSED)
    out["codebooks"] = pq.codebooks
    if pq.rotation is not None:
        out["rotation"] = pq.rotation
    codes, ids, nlist = [], [], []
    for lst in index.lists:
        c, i = ivf._canonical(lst)
        codes.append(c)
        ids.append(i)
        nlist.append(c.shape[0])
    out["codes"] = np.concatenate(codes)
    out["ids"] = np.concatenate(ids)
    out["list_sizes"] = np.asarray(nlist, np.int64)
    out["init"] = np.int64(init)
    for ma in mas:
        for R in Rs:
            res_i = np.full((nq, R), -1, np.int64)
            res_d = np.full((nq, R), np.inf, np.float32)
            res_n = np.zeros(nq, np.int64)
            for qi, q in enumerate(queries):
                r = adc.search(index, pq, q, R=R, ma=ma, method="qadc", init=init)
                res_n[qi] = r.ids.shape[0]
                res_i[qi, : r.ids.shape[0]] = r.ids
                res_d[qi, : r.ids.shape[0]] = r.distances
            out[f"ma{ma}_R{R}_ids"] = res_i
            out[f"ma{ma}_R{R}_d"] = res_d
            out[f"ma{ma}_R{R}_n"] = res_n
        if K:
            luts = np.zeros((nq, ma, m, 16), np.float32)
            cells = np.zeros((nq, ma), np.int64)
            for qi, q in enumerate(queries):
                ps = ivf.probe(index, q, ma)
                cells[qi] = ps.cells
                for s, r in enumerate(ps.residual_queries):
                    luts[qi, s] = adc.compute_tables(pq, adc._rotate(pq, r)).tables
            out[f"ma{ma}_luts"] = luts
            out[f"ma{ma}_cells"] = cells
    np.savez_compressed(path, **out)


def make_qivf(path, expect_path):
    """A QIVF v1 file written by the reference's own ivf.save_index
    (ivf.py:185-244): IVF K=5 with empty and padded lists, transposed
    layout; plus the lists it holds, for the reader test."""
    from qadc import ivf, kmeans
    from qadc import qadc as rq

    rng = np.random.default_rng(9)
    sizes = [0, 17, 32, 1, 40]
    lists, codes, ids = [], [], []
    nid = 0
    for s in sizes:
        c = rng.integers(0, 256, (s, 4), dtype=np.uint8)
        i = np.arange(nid, nid + s, dtype=np.int64) * 3
        nid += s
        lists.append(rq.transpose_list(c, i))
        codes.append(c)
        ids.append(i)
    cen = rng.random((5, 8)).astype(np.float32)
    idx = ivf.IvfIndex(d=8, m=8, b=4, coarse=kmeans.Codebook(cen), lists=lists,
                       layout=ivf.LAYOUT_TRANSPOSED)
    ivf.save_index(idx, path)
    np.savez_compressed(expect_path, centroids=cen, sizes=np.asarray(sizes),
                        codes=np.concatenate(codes), ids=np.concatenate(ids))


def make_ground_truth(path):
    """synth.ground_truth (synth.py:45-70): exact nearest neighbours, ties
    to the lower id, on a seeded mixture base with duplicated rows (forced
    distance ties) and a query equal to a base row."""
    from qadc import synth
    from qadc.vecio import Dataset

    from paper_1704_07355_b200 import datagen

    mix = datagen.Mixture(d=32, components=16, centre_high=10.0, sigma=1.0)
    base = datagen.mixture_numpy(mix, 5000, seed=3, stream=datagen.STREAM_BASE)
    base[4000:4100] = base[100:200]  # duplicates: ties resolve to the lower id
    queries = datagen.mixture_numpy(mix, 24, seed=3, stream=datagen.STREAM_QUERY)
    queries[0] = base[150]
    gt = synth.ground_truth(Dataset.from_array(base), Dataset.from_array(queries), depth=10)
    np.savez_compressed(path, base=base, queries=queries, ids=gt.ids)


def make_search_cfg2(path, n, nq, mas, R=100, init=1000):
    """configs[2]'s model at reduced N: the committed K=4096 coarse
    quantizer, OPQ rotation and residual codebooks (bench_data/), a seeded
    mixture base assigned and encoded by the REFERENCE (kmeans.assign_batch,
    pq.encode_batch, ivf._split_lists), and the reference's adc.search
    (method="qadc") outputs at nprobe 16 and 64 plus its probe order and
    (nprobe 16) fp32 tables."""
    from qadc import adc, ivf, kmeans
    from qadc import pq as rpq

    from paper_1704_07355_b200 import datagen

    bd = REPO / "bench_data"
    coarse = np.load(bd / "cfg2_coarse_K4096.npy")
    rot = np.load(bd / "cfg2_rotation.npy")
    cbk = np.load(bd / "cfg2_m32_codebooks.npy")
    K = coarse.shape[0]
    pq = rpq.ProductQuantizer(m=cbk.shape[0], b=4, codebooks=cbk, rotation=rot)
    base = datagen.mixture_numpy(datagen.SIFT_LIKE, n, seed=11, stream=datagen.STREAM_BASE)
    queries = datagen.mixture_numpy(datagen.SIFT_LIKE, nq, seed=11, stream=datagen.STREAM_QUERY)
    labels, _ = kmeans.assign_batch(coarse, base)
    packed = rpq.encode_batch(pq, base - coarse[labels])
    index = ivf.IvfIndex(d=pq.d, m=pq.m, b=pq.b, coarse=kmeans.Codebook(coarse),
                         lists=ivf._split_lists(packed, labels, K, ivf.LAYOUT_TRANSPOSED),
                         layout=ivf.LAYOUT_TRANSPOSED)
    out = {"queries": queries, "labels": labels.astype(np.uint16), "codes": packed,
           "init": np.int64(init)}
    for ma in mas:
        res_i = np.full((nq, R), -1, np.int64)
        res_d = np.full((nq, R), np.inf, np.float32)
        cells = np.zeros((nq, ma), np.int64)
        for qi, q in enumerate(queries):
            r = adc.search(index, pq, q, R=R, ma=ma, method="qadc", init=init)
            res_i[qi, : r.ids.shape[0]] = r.ids
            res_d[qi, : r.ids.shape[0]] = r.distances
            ps = ivf.probe(index, q, ma)
            cells[qi] = ps.cells
            if ma == mas[0]:
                if qi == 0:
                    out["luts"] = np.zeros((nq, ma, pq.m, 16), np.float32)
                for s_, rq_ in enumerate(ps.residual_queries):
                    out["luts"][qi, s_] = adc.compute_tables(pq, adc._rotate(pq, rq_)).tables
        out[f"ma{ma}_ids"] = res_i
        out[f"ma{ma}_d"] = res_d
        out[f"ma{ma}_cells"] = cells
    np.savez_compressed(path, **out)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
