"""GPU parity: the sm_100a path (through the C ABI of libqadc_b200.so)
against the reference's golden outputs and the CPU oracle on the same
seeded inputs. Integer / byte / id results must be bit-exact; reported
distances are compared by fp32 bit pattern."""

import numpy as np
import pytest
from conftest import cases, golden

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ------------------------------------------------------------ kernels

def test_block_distances_match_golden(gpu):
    from paper_1704_07355_b200 import kernels
    for c in cases(golden("block_dists.npz")):
        assert np.array_equal(kernels.block_distances(c["blocks"], c["shared"]), c["out_shared"])
        assert np.array_equal(kernels.block_distances(c["blocks"], c["per"]), c["out_per"])


def test_acceptance_criterion_1_fuzz(gpu):
    """tests/test_acceptance.py:118-142: >=10^5 block/table pairs, m in
    (8, 16, 32), half with full-range table bytes, byte-exact."""
    from paper_1704_07355_b200 import kernels
    rng = np.random.default_rng(7)
    pairs = 0
    for m in (8, 16, 32):
        nb = 34000
        blocks = rng.integers(0, 256, (nb, m // 2, 16), dtype=np.uint8)
        tables = rng.integers(0, 128, (nb, m, 16), dtype=np.uint8)
        tables[nb // 2:] = rng.integers(0, 256, (nb - nb // 2, m, 16), dtype=np.uint8)
        assert np.array_equal(kernels.block_distances(blocks, tables),
                              orc.block_dists(blocks, tables))
        pairs += nb
    assert pairs >= 100_000


def test_saturation_kat(gpu):
    from paper_1704_07355_b200.qadc import scan_block_scalar
    qt = np.zeros((2, 16), np.uint8)
    qt[0, 2], qt[1, 3] = 200, 100
    block = np.full((1, 16), 0x32, np.uint8)
    assert (scan_block_scalar(block, qt) == 255).all()
    qt[1, 3] = 50
    assert (scan_block_scalar(block, qt) == 250).all()


def test_quantize_tables_match_golden(gpu):
    from paper_1704_07355_b200.qadc import quantize_tables
    for c in cases(golden("quantize.npz")):
        qt = quantize_tables(c["tables"], float(c["qmin"]), float(c["qmax"]))
        assert np.array_equal(qt.tables, c["q"])
        assert qt.delta == float(c["delta"])


def test_scan_blocks_match_golden(gpu):
    """Padding lanes, pre-filled heaps, saturation rule (test_kernels.py:145-168)."""
    from paper_1704_07355_b200 import kernels
    from paper_1704_07355_b200.heap import NeighborHeap
    for c in cases(golden("scan_blocks.npz")):
        h = NeighborHeap(int(c["cap"]))
        if c["pre_i"].shape[0]:
            h.push_batch(c["pre_i"], c["pre_d"])
        kernels.scan_blocks(c["blocks"], c["ids"], c["qt"], float(c["qmin"]), float(c["delta"]), h)
        gi, gd = h.extract()
        assert np.array_equal(gi, c["out_i"])
        assert np.array_equal(_bits(gd), _bits(c["out_d"]))


def test_scan_blocks_saturated_only_below_capacity(gpu):
    """test_qadc.py:255-274: every lane saturates -> first `capacity` ids;
    a full heap never admits a saturated lane."""
    from paper_1704_07355_b200 import qadc as Q
    from paper_1704_07355_b200.heap import NeighborHeap
    from paper_1704_07355_b200.pq_util import pack_codes
    codes = np.full((64, 4), 3, np.uint8)
    tl = Q.transpose_list(pack_codes(codes), np.arange(64, dtype=np.int64))
    qt = np.full((4, 16), 127, np.uint8)
    h = NeighborHeap(10)
    Q.qadc_scan(tl, qt, h, qmin=0.0, delta=0.1)
    assert np.array_equal(h.extract()[0], np.arange(10))
    h2 = NeighborHeap(10)
    h2.push_batch(np.arange(100, 110, dtype=np.int64), np.full(10, 500.0, np.float32))
    Q.qadc_scan(tl, qt, h2, qmin=0.0, delta=0.1)
    assert np.array_equal(h2.extract()[0], np.arange(100, 110))


def test_scan_codes_float_matches_oracle(gpu, rng):
    from paper_1704_07355_b200 import kernels
    from paper_1704_07355_b200.heap import NeighborHeap
    lib = orc.lib()
    import ctypes
    for trial in range(30):
        b = int(rng.choice([4, 8, 16]))
        m = int(rng.integers(1, 7)) * (2 if b == 4 else 1)
        n = int(rng.integers(0, 300))
        cap = int(rng.integers(1, 30))
        tables = (rng.random((m, 1 << b), dtype=np.float32) * 10).astype(np.float32)
        width = {4: m // 2, 8: m, 16: 2 * m}[b]
        codes = rng.integers(0, 256, (n, width), dtype=np.uint8)
        ids = rng.permutation(n).astype(np.int64) * 3
        h = NeighborHeap(cap)
        kernels.scan_codes(codes, ids, tables, b, h)
        hd, hi = np.zeros(cap, np.float32), np.zeros(cap, np.int64)
        p = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))  # noqa: E731
        k = lib.orc_adc_scan_f32(p(codes, ctypes.c_uint8), n, p(ids, ctypes.c_int64), m, b,
                                 p(tables, ctypes.c_float), p(hd, ctypes.c_float),
                                 p(hi, ctypes.c_int64), 0, cap)
        lib.orc_heap_extract(p(hd, ctypes.c_float), p(hi, ctypes.c_int64), k)
        gi, gd = h.extract()
        assert np.array_equal(gi, hi[:k]) and np.array_equal(_bits(gd), _bits(hd[:k]))


def test_find_qmax_matches_golden(gpu):
    from paper_1704_07355_b200.qadc import find_qmax, transpose_list
    for c in cases(golden("find_qmax.npz")):
        tl = transpose_list(c["codes"], np.arange(c["codes"].shape[0], dtype=np.int64))
        got = find_qmax([(c["tables"], tl)], R=int(c["R"]), init=int(c["init"]))
        assert np.float32(got) == np.float32(c["qmax"])


def test_compute_tables_bit_exact(gpu):
    """einsum-order LUT (adc.py:61-75) is bit-exact, not just within 1e-5."""
    from paper_1704_07355_b200.adc import compute_tables
    from paper_1704_07355_b200.workload import _PQ
    for c in cases(golden("tables.npz")):
        pq = _PQ(c["codebooks"])
        for y, want in zip(c["y"], c["tables"]):
            assert np.array_equal(_bits(compute_tables(pq, y).tables), _bits(want))


def test_probe_matches_golden(gpu):
    from paper_1704_07355_b200 import ivf
    g = golden("probe.npz")
    index = ivf.IvfIndex(d=128, m=16, b=4, coarse=ivf.Codebook(g["centroids"]),
                         lists=[None] * g["centroids"].shape[0], layout=ivf.LAYOUT_STANDARD)
    for q, cells, res in zip(g["queries"], g["cells"], g["residuals"]):
        ps = ivf.probe(index, q, int(g["ma"]))
        assert np.array_equal(ps.cells, cells)
        assert np.array_equal(_bits(ps.residual_queries), _bits(res))


# ------------------------------------------------------------ batched search

def _index_from_golden(g):
    from paper_1704_07355_b200 import ivf
    from paper_1704_07355_b200.qadc import transpose_list
    sizes = g["list_sizes"]
    off = np.concatenate([[0], np.cumsum(sizes)])
    lists = [transpose_list(g["codes"][off[L]:off[L + 1]], g["ids"][off[L]:off[L + 1]])
             for L in range(sizes.shape[0])]
    coarse = ivf.Codebook(g["coarse"]) if "coarse" in g.files else None
    return ivf.IvfIndex(d=g["queries"].shape[1], m=g["codebooks"].shape[0], b=4, coarse=coarse,
                        lists=lists, layout=ivf.LAYOUT_TRANSPOSED)


def _pq_from_golden(g):
    from paper_1704_07355_b200.workload import _PQ
    return _PQ(g["codebooks"], g["rotation"] if "rotation" in g.files else None)


@pytest.mark.parametrize("name", ["search_flat16.npz", "search_flat_hd.npz"])
def test_flat_search_batch_matches_reference(gpu, name):
    from paper_1704_07355_b200.adc import search_batch
    g = golden(name)
    index, pq = _index_from_golden(g), _pq_from_golden(g)
    for key in [k for k in g.files if k.endswith("_ids")]:
        R = int(key.split("_R")[1].split("_")[0])
        res = search_batch(index, pq, g["queries"], R, init=int(g["init"]))
        assert np.array_equal(res.ids, g[key]), key
        assert np.array_equal(_bits(res.distances), _bits(g[key.replace("_ids", "_d")])), key
        assert np.array_equal(res.counts, g[key.replace("_ids", "_n")]), key


def test_single_query_search_matches_reference(gpu):
    from paper_1704_07355_b200.adc import search
    g = golden("search_flat16.npz")
    index, pq = _index_from_golden(g), _pq_from_golden(g)
    for qi in range(5):
        r = search(index, pq, g["queries"][qi], R=10, method="qadc")
        n = int(g["ma1_R10_n"][qi])
        assert np.array_equal(r.ids, g["ma1_R10_ids"][qi, :n])
        assert np.array_equal(_bits(r.distances), _bits(g["ma1_R10_d"][qi, :n]))
        t = r.timings
        assert t.total_ms == pytest.approx(t.index_ms + t.tables_ms + t.scan_ms, abs=1e-9)


@pytest.mark.parametrize("ma", [4, 16])
def test_ivf_opq_injected_lut_bit_exact(gpu, ma):
    """Reference-LUT-injected mode: with the reference's fp32
    tables and probe order, ids and distances are bit-exact."""
    from paper_1704_07355_b200.adc import search_batch
    g = golden("search_ivf_opq.npz")
    index, pq = _index_from_golden(g), _pq_from_golden(g)
    res = search_batch(index, pq, g["queries"], 100, ma=ma, init=int(g["init"]),
                       lut=g[f"ma{ma}_luts"], cells=g[f"ma{ma}_cells"])
    assert np.array_equal(res.ids, g[f"ma{ma}_R100_ids"])
    assert np.array_equal(_bits(res.distances), _bits(g[f"ma{ma}_R100_d"]))


@pytest.mark.parametrize("ma", [4, 16])
def test_ivf_opq_native_bit_exact(gpu, ma):
    """Native OPQ mode (the GPU probes, rotates, builds and quantizes the
    tables itself) against the reference's own adc.search outputs: the
    rotation follows OpenBLAS sgemv's order (adc.py:108-111), so probe
    order, fp32 tables, ids and distances are all bit-exact."""
    import torch

    from paper_1704_07355_b200.adc import search_batch
    from paper_1704_07355_b200.device import DeviceIndex
    g = golden("search_ivf_opq.npz")
    index, pq = _index_from_golden(g), _pq_from_golden(g)
    res = search_batch(index, pq, g["queries"], 100, ma=ma, init=int(g["init"]))
    assert np.array_equal(res.ids, g[f"ma{ma}_R100_ids"])
    assert np.array_equal(_bits(res.distances), _bits(g[f"ma{ma}_R100_d"]))
    t = DeviceIndex.from_ivf(index, pq).tables(torch.from_numpy(g["queries"]).cuda(), 100, ma=ma,
                                               init=int(g["init"]))
    assert np.array_equal(t["cells"].cpu().numpy(), g[f"ma{ma}_cells"])
    assert np.array_equal(_bits(t["lut"].cpu().numpy()), _bits(g[f"ma{ma}_luts"]))


def _cfg2_device_index(g, model, order, bounds):
    import torch

    from paper_1704_07355_b200.device import DeviceIndex
    cb, rot, coarse = model
    rows = torch.from_numpy(g["codes"][order]).cuda()
    row_off = torch.from_numpy(bounds.astype(np.int64)).cuda()
    return DeviceIndex.from_device_rows(
        128, 32, rows, row_off, torch.from_numpy(cb).cuda(), rotation=torch.from_numpy(rot).cuda(),
        coarse=torch.from_numpy(coarse).cuda(), ids=torch.from_numpy(order.astype(np.int64)).cuda())


@pytest.mark.parametrize("ma", [16, 64])
def test_cfg2_scale_native_bit_exact_vs_reference(gpu, ma):
    """configs[2]'s K = 4096 coarse quantizer + OPQ rotation (N = 1e5):
    native GPU search == the reference's adc.search (committed outputs),
    ids and fp32 distance bits, every query; probe order and (nprobe 16)
    fp32 tables bit-exact too; and in reference-LUT-injected mode."""
    import torch

    from test_oracle import cfg2_golden
    g, model, flat, order, bounds = cfg2_golden()
    idx = _cfg2_device_index(g, model, order, bounds)
    q = torch.from_numpy(g["queries"]).cuda()
    for scan in ("auto", "prmt", "tc"):
        res = idx.search(q, 100, ma=ma, init=int(g["init"]), scan=scan)
        assert np.array_equal(res.ids.cpu().numpy(), g[f"ma{ma}_ids"]), scan
        assert np.array_equal(_bits(res.distances.cpu().numpy()), _bits(g[f"ma{ma}_d"])), scan
    t = idx.tables(q, 100, ma=ma, init=int(g["init"]))
    assert np.array_equal(t["cells"].cpu().numpy(), g[f"ma{ma}_cells"])
    if ma == 16:
        assert np.array_equal(_bits(t["lut"].cpu().numpy()), _bits(g["luts"]))
        inj = idx.search(q, 100, ma=ma, init=int(g["init"]), lut=torch.from_numpy(g["luts"]).cuda(),
                         cells=torch.from_numpy(g["ma16_cells"]).cuda())
        assert np.array_equal(inj.ids.cpu().numpy(), g["ma16_ids"])
        assert np.array_equal(_bits(inj.distances.cpu().numpy()), _bits(g["ma16_d"]))


@pytest.mark.parametrize("ma", [16, 64])
def test_cfg2_scale_native_vs_this_hosts_blas(gpu, ma):
    """The same index against the reference's Index + Tables phases re-run
    on THIS host (numpy / OpenBLAS rotation, adc.py:108-111, plus the
    pinned oracle): counts fp32 LUT bit mismatches, uint8 flips, qmax
    mismatches (SURVEY 8c native mode). LUT relative error must be
    <= 1e-5, probe order exact, and top-R ids + distance bits exact on
    every query whose tables did not diverge. On hosts whose OpenBLAS
    dispatches to the SkylakeX/Haswell sgemv kernels every count is 0."""
    import torch

    from oracle import parity
    from test_oracle import cfg2_golden
    g, (cb, rot, coarse), flat, order, bounds = cfg2_golden()
    idx = _cfg2_device_index(g, (cb, rot, coarse), order, bounds)
    q = torch.from_numpy(g["queries"]).cuda()
    t = {k: v.cpu().numpy() for k, v in idx.tables(q, 100, ma=ma, init=1000).items()}
    ref = parity.reference_tables(g["queries"], cb, rot, coarse, ma, flat, 100, 1000)
    acc = parity.account(t, ref)
    print("native-mode accounting vs this host's BLAS:",
          {k: v for k, v in acc.items() if not k.startswith("_")})
    assert acc["cells_mismatch_queries"] == 0
    assert acc["lut_max_rel_err"] <= 1e-5
    oi, od, _, _ = orc.search_batch(g["queries"], cb, rot, coarse, ma, flat, 100, 1000,
                                    lut_in=ref["lut"], cells_in=ref["cells"])
    res = idx.search(q, 100, ma=ma, init=1000)
    cmp = parity.compare_results(res.ids.cpu().numpy(), res.distances.cpu().numpy(), oi, od,
                                 acc["_diverged"])
    print("results:", cmp)
    assert cmp["clean_exact"] == cmp["clean_queries"]


# ------------------------------------------------------------ oracle, larger sizes

def _random_flat(rng, n, m, d, nq, cb_scale=50.0):
    import torch

    from paper_1704_07355_b200.device import DeviceIndex
    from paper_1704_07355_b200.ivf import encode_device
    from paper_1704_07355_b200.qadc import transpose_list
    from paper_1704_07355_b200.workload import _PQ
    cb = (rng.random((m, 16, d // m)) * cb_scale).astype(np.float32)
    pq = _PQ(cb)
    X = torch.from_numpy((rng.random((n, d)) * cb_scale).astype(np.float32)).cuda()
    codes = encode_device(pq, X)
    idx = DeviceIndex.from_device_rows(d, m, codes, torch.tensor([0, n], device="cuda"),
                                       torch.from_numpy(cb).cuda())
    tl = transpose_list(codes.cpu().numpy(), np.arange(n, dtype=np.int64))
    flat = (tl.blocks.reshape(-1), np.array([0, tl.blocks.shape[0]], np.int64), tl.ids,
            np.array([n], np.int64))
    qs = (rng.random((nq, d)) * cb_scale).astype(np.float32)
    return idx, flat, qs, cb


@pytest.mark.parametrize("m,R,init", [(16, 1, 1000), (16, 100, 1000), (32, 100, 1000),
                                      (32, 1000, 1000), (8, 37, 50), (64, 100, 1000),
                                      (32, 100, 20)])
def test_search_batch_vs_oracle(gpu, m, R, init):
    rng = np.random.default_rng(m * 1000 + R)
    idx, flat, qs, cb = _random_flat(rng, 150_000, m, 128, 48)
    tc = m in (16, 32)  # the int8 tensor-core scan applies
    res = idx.search(qs, R, init=init, scan="tc" if tc else "auto")
    oi, od, on, _ = orc.search_batch(qs, cb, None, None, 1, flat, R, init)
    assert res.stats["scan_tc"] == (1 if tc else 0)
    assert np.array_equal(res.ids, oi)
    assert np.array_equal(_bits(res.distances), _bits(od))
    assert np.array_equal(res.counts, on)
    if tc:  # the one-SM tensor-core scan (not CTA pairs) on the same inputs
        t1 = idx.search(qs, R, init=init, scan="tc1")
        assert t1.stats["scan_tc"] == 1
        assert np.array_equal(t1.ids, oi)
        assert np.array_equal(_bits(t1.distances), _bits(od))
    if tc:  # the CUDA-core PRMT scan on the same inputs
        pr = idx.search(qs, R, init=init, scan="prmt")
        assert pr.stats["scan_tc"] == 0
        assert np.array_equal(pr.ids, oi)
        assert np.array_equal(_bits(pr.distances), _bits(od))
        assert np.array_equal(pr.counts, on)


def test_edge_cases_vs_oracle(gpu):
    rng = np.random.default_rng(3)
    # tiny lists (R > N), odd sizes, exactly one chunk, chunk + 1
    for n in (1, 7, 16, 255, 256, 257, 1000):
        idx, flat, qs, cb = _random_flat(rng, n, 16, 64, 8)
        for R in (1, 5, 300):
            res = idx.search(qs, R, init=1000)
            oi, od, on, _ = orc.search_batch(qs, cb, None, None, 1, flat, R, 1000)
            assert np.array_equal(res.ids, oi), (n, R)
            assert np.array_equal(_bits(res.distances), _bits(od)), (n, R)
            assert np.array_equal(res.counts, on), (n, R)


def test_tensor_core_scan_edge_cases_vs_oracle(gpu):
    """The CTA-pair (cta_group::2) and one-SM tensor-core scans on partial
    chunks, one query (MMA N = 16: 8 B rows per CTA of the pair), a query
    count that is not a multiple of 16, and more queries than one MMA's N
    (two items per code range)."""
    rng = np.random.default_rng(11)
    for n in (1, 255, 257, 5000):
        for nq in (1, 17, 300):
            idx, flat, qs, cb = _random_flat(rng, n, 32, 128, nq)
            for R in (1, 100):
                oi, od, on, _ = orc.search_batch(qs, cb, None, None, 1, flat, R, 1000)
                for scan in ("tc", "tc1"):
                    res = idx.search(qs, R, init=1000, scan=scan)
                    assert res.stats["scan_tc"] == 1
                    assert np.array_equal(res.ids, oi), (n, nq, R, scan)
                    assert np.array_equal(_bits(res.distances), _bits(od)), (n, nq, R, scan)
                    assert np.array_equal(res.counts, on), (n, nq, R, scan)


@pytest.mark.parametrize("m", [16, 32])
def test_tensor_core_scan_long_list_vs_oracle(gpu, m):
    """A list long enough (>= 8192 chunks) for the CTA-pair scan's flusher
    rings, bit-exact against the oracle (two query items per code range)."""
    rng = np.random.default_rng(12 + m)
    idx, flat, qs, cb = _random_flat(rng, 2_200_000, m, 128, 264)
    oi, od, on, _ = orc.search_batch(qs, cb, None, None, 1, flat, 100, 1000)
    res = idx.search(qs, 100, init=1000, scan="tc")
    assert res.stats["scan_tc"] == 1
    assert np.array_equal(res.ids, oi)
    assert np.array_equal(_bits(res.distances), _bits(od))
    assert np.array_equal(res.counts, on)


@pytest.mark.parametrize("n", [60_000, 200_000])
def test_massive_ties_vs_oracle(gpu, n):
    """Three code patterns only (about n, n/7 and n/40 copies): every lane
    ties with thousands of others; the exact (distance, id) order must
    still pick the lowest ids. Covers the select kernel's radix path (ties
    sorted in shared memory, and the id-radix passes beyond that) and, at
    n = 200000, the candidate-capacity rerun."""
    import torch

    from paper_1704_07355_b200.device import DeviceIndex
    from paper_1704_07355_b200.qadc import transpose_list
    m, d = 16, 64
    rng = np.random.default_rng(5)
    cb = (rng.random((m, 16, d // m)) * 10).astype(np.float32)
    codes = np.full((n, m // 2), 0x21, np.uint8)
    codes[::7] = 0x43
    codes[::40] = 0x65
    idx = DeviceIndex.from_device_rows(d, m, torch.from_numpy(codes).cuda(),
                                       torch.tensor([0, n], device="cuda"),
                                       torch.from_numpy(cb).cuda())
    tl = transpose_list(codes, np.arange(n, dtype=np.int64))
    flat = (tl.blocks.reshape(-1), np.array([0, tl.blocks.shape[0]], np.int64), tl.ids,
            np.array([n], np.int64))
    qs = (rng.random((6, d)) * 10).astype(np.float32)
    for R in (10, 100, 1500):
        res = idx.search(qs, R, init=1000)
        oi, od, on, _ = orc.search_batch(qs, cb, None, None, 1, flat, R, 1000)
        assert np.array_equal(res.ids, oi)
        assert np.array_equal(_bits(res.distances), _bits(od))


def test_property_large_index_sorted_and_self_consistent(gpu):
    """At 4*10^6 codes (oracle too slow for every query): results are sorted
    by (distance, id), distances are bin midpoints, and a sampled query
    matches the oracle bit-exactly."""
    rng = np.random.default_rng(11)
    idx, flat, qs, cb = _random_flat(rng, 4_000_000, 32, 128, 64)
    res = idx.search(qs, 100, init=1000)
    ids, d = res.ids, res.distances
    for i in range(ids.shape[0]):
        o = np.lexsort((ids[i], d[i]))
        assert np.array_equal(o, np.arange(100))
        assert len(set(ids[i].tolist())) == 100
    oi, od, on, _ = orc.search_batch(qs[:3], cb, None, None, 1, flat, 100, 1000)
    assert np.array_equal(ids[:3], oi) and np.array_equal(_bits(d[:3]), _bits(od))


def test_encoder_matches_reference_assignment(gpu):
    """GPU encoder == reference pq.encode_batch codes (golden corpus)."""
    import torch

    from paper_1704_07355_b200 import datagen
    from paper_1704_07355_b200.ivf import encode_device
    g = golden("search_flat16.npz")
    pq = _pq_from_golden(g)
    base = datagen.mixture_numpy(datagen.SIFT_LIKE, 20000, seed=1, stream=datagen.STREAM_BASE)
    codes = encode_device(pq, torch.from_numpy(base).cuda()).cpu().numpy()
    assert np.array_equal(codes, g["codes"][np.argsort(g["ids"])])


@pytest.mark.parametrize("K,n", [(300, 3000), (4096, 20000), (65536, 2000)])
def test_tensor_core_assign_matches_exact_einsum(gpu, K, n):
    """qadc_b200_assign on the fused tcgen05 nearest-centroid kernel
    (probe_tc.cu, ma = 1): every label equals the exact einsum-order argmin
    with ties to the lower index (the oracle's probe at ma = 1), including
    duplicated centroids (forced ties) and points on centroids."""
    import torch

    from paper_1704_07355_b200 import datagen
    from paper_1704_07355_b200.ivf import assign_device
    rng = np.random.default_rng(K)
    X = datagen.mixture_numpy(datagen.SIFT_LIKE, n, seed=K, stream=2)
    C = X[rng.choice(n, min(K, n), replace=False)].copy()
    if C.shape[0] < K:
        C = np.concatenate([C, datagen.mixture_numpy(datagen.SIFT_LIKE, K - C.shape[0], seed=K,
                                                     stream=5)])
    C[K // 2] = C[K // 3]  # exact duplicate: ties resolve to the lower index
    X[:5] = C[K // 3]      # points sitting on the duplicated centroid
    lab = assign_device(C, torch.from_numpy(X).cuda()).cpu().numpy()
    want = np.array([orc.probe(C, x, 1)[0][0] for x in X])
    assert np.array_equal(lab, want)


@pytest.mark.parametrize("ma", [1, 8, 32])
def test_ivf_search_vs_oracle_at_scale(gpu, ma):
    """IVF + OPQ, K=256 lists, 2*10^5 codes: with the oracle's float LUTs
    and probe order injected, ids and distances are bit-exact; natively the
    probe order is exact and results agree except for rotation flips."""
    import torch

    from paper_1704_07355_b200 import datagen
    from paper_1704_07355_b200.device import DeviceIndex
    from paper_1704_07355_b200.ivf import assign_device, encode_device
    from paper_1704_07355_b200.qadc import transpose_list
    from paper_1704_07355_b200.workload import _PQ
    rng = np.random.default_rng(ma)
    K, n, m, d, R = 256, 200_000, 32, 128, 100
    X = datagen.mixture_numpy(datagen.SIFT_LIKE, n, seed=5, stream=2)
    coarse = X[rng.choice(n, K, replace=False)].copy()
    Rm = np.linalg.qr(rng.standard_normal((d, d)))[0].astype(np.float32)
    cb = (rng.standard_normal((m, 16, d // m)) * 8).astype(np.float32)
    pq = _PQ(cb, Rm)
    Xd = torch.from_numpy(X).cuda()
    C = torch.from_numpy(coarse).cuda()
    lab = assign_device(coarse, Xd)
    codes = encode_device(pq, Xd - C[lab])
    order = torch.argsort(lab, stable=True)
    sizes = torch.bincount(lab, minlength=K)
    row_off = torch.zeros(K + 1, dtype=torch.int64, device="cuda")
    row_off[1:] = torch.cumsum(sizes, 0)
    sc = codes[order].contiguous()
    idx = DeviceIndex.from_device_rows(d, m, sc, row_off, torch.from_numpy(cb).cuda(),
                                       rotation=torch.from_numpy(Rm).cuda(), coarse=C, ids=order)
    # reference-layout copy for the oracle
    sc_np, ord_np, off = sc.cpu().numpy(), order.cpu().numpy(), row_off.cpu().numpy()
    blocks, ids, boff, count = [], [], [0], []
    for L in range(K):
        tl = transpose_list(sc_np[off[L]:off[L + 1]], ord_np[off[L]:off[L + 1]])
        blocks.append(tl.blocks.reshape(-1))
        ids.append(tl.ids)
        boff.append(boff[-1] + tl.blocks.shape[0])
        count.append(tl.count)
    flat = (np.concatenate(blocks), np.asarray(boff, np.int64), np.concatenate(ids),
            np.asarray(count, np.int64))
    qs = datagen.mixture_numpy(datagen.SIFT_LIKE, 24, seed=5, stream=3)
    # oracle LUTs injected into both sides
    luts = np.zeros((qs.shape[0], ma, m, 16), np.float32)
    cells = np.zeros((qs.shape[0], ma), np.int64)
    for i, q in enumerate(qs):
        c, res = orc.probe(coarse, q, ma)
        cells[i] = c
        for s_, r in enumerate(res):
            luts[i, s_] = orc.compute_tables(cb, orc.rotate(Rm, r))
    oi, od, on, _ = orc.search_batch(qs, cb, Rm, coarse, ma, flat, R, 1000, lut_in=luts,
                                     cells_in=cells)
    # int8 tensor-core scans (all warps on one tile / warpgroup-pipelined), PRMT scan, heuristic
    for scan in ("tc", "tcw", "prmt", "auto"):
        got = idx.search(qs, R, ma=ma, init=1000, lut=luts, cells=cells, scan=scan)
        if scan != "auto":
            assert got.stats["scan_tc"] == {"tc": 1, "tcw": 2, "prmt": 0}[scan]
        assert np.array_equal(got.ids, oi), scan
        assert np.array_equal(_bits(got.distances), _bits(od)), scan
        assert np.array_equal(got.counts, on), scan
    # native: the GPU rotates, probes and builds the tables itself in the
    # reference's arithmetic (OpenBLAS sgemv order for the rotation), so the
    # whole native path is bit-exact against the oracle too
    nat = idx.search(qs, R, ma=ma, init=1000)
    ni, nd, nn, _ = orc.search_batch(qs, cb, Rm, coarse, ma, flat, R, 1000)
    assert np.array_equal(nat.ids, ni)
    assert np.array_equal(_bits(nat.distances), _bits(nd))

@pytest.mark.parametrize("m,K,n,nq,ma,R", [(32, 48, 60_000, 150, 12, 50), (16, 20, 30_000, 64, 5, 100),
                                           (32, 300, 40_000, 400, 20, 10), (16, 24, 30_000, 200, 8, 100),
                                           (32, 16, 50_000, 300, 10, 100)])
def test_warpgroup_tensor_core_scan_vs_oracle(gpu, m, K, n, nq, ma, R):
    """k_scan_tcw (IVF lists probed by a few queries each: code-major one-hot
    expansion, one issuing warp per warpgroup, survivors through per-warp
    rings): ids, fp32 distance bits and counts equal the oracle's and the PRMT
    scan's on lists of 0..~3000 codes with 1..~200 pairs each (<= 32 queries
    per pass: lists with more pairs take several passes, MMA N = 16 and
    32)."""
    import torch

    from paper_1704_07355_b200 import datagen
    from paper_1704_07355_b200.device import DeviceIndex
    from paper_1704_07355_b200.ivf import assign_device, encode_device
    from paper_1704_07355_b200.qadc import transpose_list
    from paper_1704_07355_b200.workload import _PQ
    rng = np.random.default_rng(m + K)
    d = 128
    X = datagen.mixture_numpy(datagen.SIFT_LIKE, n, seed=7, stream=2)
    coarse = X[rng.choice(n, K, replace=False)].copy()
    Rm = np.linalg.qr(rng.standard_normal((d, d)))[0].astype(np.float32)
    cb = (rng.standard_normal((m, 16, d // m)) * 8).astype(np.float32)
    pq = _PQ(cb, Rm)
    Xd = torch.from_numpy(X).cuda()
    C = torch.from_numpy(coarse).cuda()
    lab = assign_device(coarse, Xd)
    codes = encode_device(pq, Xd - C[lab])
    order = torch.argsort(lab, stable=True)
    sizes = torch.bincount(lab, minlength=K)
    row_off = torch.zeros(K + 1, dtype=torch.int64, device="cuda")
    row_off[1:] = torch.cumsum(sizes, 0)
    sc = codes[order].contiguous()
    idx = DeviceIndex.from_device_rows(d, m, sc, row_off, torch.from_numpy(cb).cuda(),
                                       rotation=torch.from_numpy(Rm).cuda(), coarse=C, ids=order)
    sc_np, ord_np, off = sc.cpu().numpy(), order.cpu().numpy(), row_off.cpu().numpy()
    blocks, ids, boff, count = [], [], [0], []
    for L in range(K):
        tl = transpose_list(sc_np[off[L]:off[L + 1]], ord_np[off[L]:off[L + 1]])
        blocks.append(tl.blocks.reshape(-1))
        ids.append(tl.ids)
        boff.append(boff[-1] + tl.blocks.shape[0])
        count.append(tl.count)
    flat = (np.concatenate(blocks), np.asarray(boff, np.int64), np.concatenate(ids),
            np.asarray(count, np.int64))
    qs = datagen.mixture_numpy(datagen.SIFT_LIKE, nq, seed=7, stream=3)
    oi, od, on, _ = orc.search_batch(qs, cb, Rm, coarse, ma, flat, R, 1000)
    qd = torch.from_numpy(qs).cuda()
    ref = idx.search(qd, R, ma=ma, init=1000, scan="prmt")
    got = idx.search(qd, R, ma=ma, init=1000, scan="tcw")
    assert got.stats["scan_tc"] == 2
    for r in (ref, got):
        assert np.array_equal(r.ids.cpu().numpy(), oi)
        assert np.array_equal(_bits(r.distances.cpu().numpy()), _bits(od))
        assert np.array_equal(r.counts.cpu().numpy(), on)


@pytest.mark.parametrize("K,ma", [(300, 1), (300, 64), (300, 300), (5000, 16), (5000, 130),
                                  (9000, 64)])
def test_probe_vs_oracle_many_sizes(gpu, K, ma):
    """Probe order (einsum d2, ties -> lower cell) for multi-tile K and
    ma beyond one selection buffer, including forced distance ties."""
    from paper_1704_07355_b200 import datagen, ivf
    cen = datagen.mixture_numpy(datagen.SIFT_LIKE, K, seed=K, stream=1)
    cen[K // 3] = cen[K // 2]  # duplicate centroid -> exact d2 tie
    index = ivf.IvfIndex(d=128, m=16, b=4, coarse=ivf.Codebook(cen), lists=[None] * K,
                         layout=ivf.LAYOUT_STANDARD)
    qs = datagen.mixture_numpy(datagen.SIFT_LIKE, 6, seed=K, stream=3)
    qs[0] = cen[K // 2]
    for q in qs:
        want, _ = orc.probe(cen, q, ma)
        assert np.array_equal(ivf.probe(index, q, ma).cells, want)


@pytest.mark.parametrize("K,ma,distinct", [(4096, 16, 4096), (4096, 64, 20), (1003, 8, 3),
                                           (70000, 32, 70000), (65536, 64, 65536)])
def test_probe_batch_bounds_and_tie_fallback(gpu, K, ma, distinct):
    """Batched native probe (nq not a multiple of the 8-query CTA) against
    the oracle. `distinct` < K repeats centroids so that hundreds of cells
    share the exact same d2: the FFMA pre-selection then keeps more
    candidates than its buffer and the exact all-cells fallback runs."""
    import torch
    from paper_1704_07355_b200 import _native, datagen
    base = datagen.mixture_numpy(datagen.SIFT_LIKE, distinct, seed=K + distinct, stream=1)
    cen = np.ascontiguousarray(base[np.arange(K) % distinct])
    qs = datagen.mixture_numpy(datagen.SIFT_LIKE, 13, seed=K, stream=4)
    qs[1] = cen[5]
    qs[2] = 0.0
    dev = torch.device("cuda")
    cd, qd = torch.from_numpy(cen).to(dev), torch.from_numpy(qs).to(dev)
    cells = torch.empty((13, ma), dtype=torch.int64, device=dev)
    res = torch.empty((13, ma, 128), dtype=torch.float32, device=dev)
    lib = _native.load_library()
    _native.check(lib.qadc_b200_probe(_native.dptr(cd), K, 128, _native.dptr(qd), 13, ma,
                                      _native.dptr(cells), _native.dptr(res),
                                      torch.cuda.current_stream().cuda_stream), "probe")
    got = cells.cpu().numpy()
    for i in range(13):
        want, wres = orc.probe(cen, qs[i], ma)
        assert np.array_equal(got[i], want), i
        assert np.array_equal(_bits(res[i].cpu().numpy()), _bits(wres))


@pytest.mark.parametrize("K,ma,nq", [(8192, 64, 1000), (65536, 16, 300), (1024, 1, 777)])
def test_probe_many_query_tiles_vs_oracle(gpu, K, ma, nq):
    """The fused tensor-core probe over several 128-query tiles and
    centroid-range slices (the configs' batch shapes) equals the oracle's
    probe order for every query."""
    import torch

    from paper_1704_07355_b200 import _native, datagen
    cen = datagen.mixture_numpy(datagen.SIFT_LIKE, K, seed=K + nq, stream=1)
    qs = datagen.mixture_numpy(datagen.SIFT_LIKE, nq, seed=K, stream=4)
    dev = torch.device("cuda")
    cells = torch.empty((nq, ma), dtype=torch.int64, device=dev)
    cd, qd = torch.from_numpy(cen).to(dev), torch.from_numpy(qs).to(dev)  # alive during the call
    _native.check(_native.load_library().qadc_b200_probe(
        _native.dptr(cd), K, 128, _native.dptr(qd), nq, ma, _native.dptr(cells), None,
        torch.cuda.current_stream().cuda_stream), "probe")
    got = cells.cpu().numpy()
    for i in range(nq):
        assert np.array_equal(got[i], orc.probe(cen, qs[i], ma)[0]), i
