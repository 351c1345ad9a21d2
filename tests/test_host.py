"""CPU: host-side logic of the package and the C-ABI boundary (no GPU
compute): heap contract, layout helpers, variant registry, QIVF I/O,
workload generator, and that libqadc_b200.so loads and exports every
symbol include/qadc_b200.h declares."""

import ctypes
import re
from pathlib import Path

from conftest import golden

import numpy as np
import pytest

from paper_1704_07355_b200 import _native, datagen, ivf, kernels
from paper_1704_07355_b200.heap import NeighborHeap
from paper_1704_07355_b200.qadc import (PAD_BYTE, PAD_ID, QuantizedTables, TransposedList,
                                        dequantize, transpose_block, transpose_list,
                                        untranspose_block, untranspose_list)

ROOT = Path(__file__).resolve().parent.parent


# ---------------------------------------------------------------- C ABI

def _declared_symbols():
    hdr = (ROOT / "include" / "qadc_b200.h").read_text()
    decls = re.findall(r"^QADC_API\s+[\w\s\*]*?\b(\w+)\s*\(", hdr, re.M)
    assert len(decls) >= 15
    return decls


def test_header_declares_reference_abi():
    names = set(_declared_symbols())
    # scan_kernels.h:15-46
    assert {"qadc_simd_level", "adc_scan_f32", "qadc_scan_u8", "qadc_block_dists"} <= names
    assert "qadc_b200_search_batch" in names


def test_library_loads_and_exports_every_declared_symbol():
    if not _native.library_available():
        pytest.fail("libqadc_b200.so is not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in _declared_symbols():
        assert hasattr(lib, name), name


def test_search_flags_match_header():
    """The ctypes flag constants are the header's #defines (the C ABI a
    maintainer binds)."""
    hdr = (ROOT / "include" / "qadc_b200.h").read_text()
    defs = {k: int(v) for k, v in re.findall(r"#define QADC_B200_(\w+) (\d+)u", hdr)}
    for name in ("HOST_IO", "LUT_IN", "NO_FSAT", "SCAN_PRMT", "SCAN_TC", "SCAN_TC1", "SCAN_TCW"):
        assert defs[name] == getattr(_native, name), name
    flags = [defs[n] for n in ("HOST_IO", "LUT_IN", "NO_FSAT", "SCAN_PRMT", "SCAN_TC", "SCAN_TC1", "SCAN_TCW")]
    assert len(set(flags)) == len(flags) and all(f & (f - 1) == 0 for f in flags)


def test_reference_abi_signatures_match_reference_header():
    """Argument lists of the four replaced functions equal the reference's
    (scan_kernels.h), parameter for parameter."""
    ref = Path("/root/reference/pkg/src/qadc/src/scan_kernels.h")
    if not ref.exists():
        pytest.skip("reference sources not present on this host")
    norm = lambda s: re.sub(r"\s+", " ", s).strip()  # noqa: E731
    ours = (ROOT / "include" / "qadc_b200.h").read_text()
    for fn in ("adc_scan_f32", "qadc_scan_u8", "qadc_block_dists"):
        pat = re.compile(r"\b" + fn + r"\(([^;]*?)\);", re.S)
        a = norm(pat.search(ref.read_text()).group(1))
        b = norm(pat.search(ours).group(1))
        assert a == b, fn


# ---------------------------------------------------------------- registry

def test_registry_names_and_resolution(monkeypatch):
    monkeypatch.delenv(kernels.ENV_VAR, raising=False)
    assert kernels.available_variants() == ("b200",)
    assert kernels.resolve_variant(None) == "b200"
    assert kernels.resolve_variant("auto") == "b200"
    monkeypatch.setenv(kernels.ENV_VAR, "b200")
    assert kernels.resolve_variant(None) == "b200"


def test_registry_errors_match_reference(monkeypatch):
    monkeypatch.delenv(kernels.ENV_VAR, raising=False)
    with pytest.raises(ValueError):
        kernels.resolve_variant("turbo")
    monkeypatch.setenv(kernels.ENV_VAR, "turbo")
    with pytest.raises(ValueError):
        kernels.resolve_variant(None)
    monkeypatch.delenv(kernels.ENV_VAR)
    # the reference's CPU variants are known names but unavailable here
    for v in ("python", "scalar", "simd128", "simd256"):
        with pytest.raises(RuntimeError):
            kernels.resolve_variant(v)


def test_no_cpu_fallback_when_library_missing(monkeypatch):
    monkeypatch.setattr(_native, "LIB_PATH", Path("/nonexistent/libqadc_b200.so"))
    monkeypatch.setattr(_native, "_lib", None)
    assert kernels.available_variants() == ()
    with pytest.raises(RuntimeError):
        kernels.resolve_variant(None)
    with pytest.raises(RuntimeError):
        _native.load_library()


def test_shape_validation_before_any_device_work():
    heap = NeighborHeap(3)
    with pytest.raises(ValueError):
        kernels.scan_codes(np.zeros((5, 3), np.uint8), np.arange(5), np.zeros((4, 16), np.float32),
                           4, heap)
    with pytest.raises(ValueError):
        kernels.scan_blocks(np.zeros((2, 3, 8), np.uint8), np.arange(32), np.zeros((6, 16),
                            np.uint8), 0.0, 1.0, heap)
    with pytest.raises(ValueError):
        kernels.scan_blocks(np.zeros((2, 3, 16), np.uint8), np.arange(31),
                            np.zeros((6, 16), np.uint8), 0.0, 1.0, heap)
    with pytest.raises(ValueError):
        kernels.block_distances(np.zeros((2, 3, 16), np.uint8), np.zeros((5, 16), np.uint8))
    with pytest.raises(ValueError):
        kernels.block_distances(np.zeros((2, 70, 16), np.uint8), np.zeros((140, 16), np.uint8))


def test_empty_inputs_never_touch_the_device():
    heap = NeighborHeap(4)
    heap.push(3, 1.0)
    kernels.scan_codes(np.zeros((0, 2), np.uint8), np.zeros(0, np.int64),
                       np.zeros((4, 16), np.float32), 4, heap)
    kernels.scan_blocks(np.zeros((0, 2, 16), np.uint8), np.zeros(0, np.int64),
                        np.zeros((4, 16), np.uint8), 0.0, 1.0, heap)
    assert heap.size == 1 and heap.worst() == (1.0, 3)
    assert kernels.block_distances(np.zeros((0, 2, 16), np.uint8),
                                   np.zeros((4, 16), np.uint8)).shape == (0, 16)


# ---------------------------------------------------------------- heap

def test_heap_keeps_r_best_with_id_ties(rng):
    for _ in range(30):
        n = int(rng.integers(0, 200))
        cap = int(rng.integers(1, 40))
        d = rng.integers(0, 20, n).astype(np.float32)  # forced ties
        ids = rng.permutation(n).astype(np.int64)
        h1, h2 = NeighborHeap(cap), NeighborHeap(cap)
        for i, x in zip(ids, d):
            h1.push(int(i), float(x))
        h2.push_batch(ids, d)
        o = np.lexsort((ids, d))[:cap]
        for h in (h1, h2):
            gi, gd = h.extract()
            assert np.array_equal(gi, ids[o]) and np.array_equal(gd, d[o])


def test_heap_pop_order_and_validation():
    with pytest.raises(ValueError):
        NeighborHeap(0)
    h = NeighborHeap(5)
    for i, x in enumerate([3.0, 1.0, 2.0, 2.0, 5.0, 0.5]):
        h.push(i, x)
    out = [h.pop() for _ in range(5)]
    assert [d for _, d in out] == sorted([d for _, d in out], reverse=True)
    with pytest.raises(IndexError):
        h.pop()


# ---------------------------------------------------------------- layout

def test_transpose_block_kat():
    codes = np.zeros((16, 1), np.uint8)
    codes[0, 0] = 0x95
    block = transpose_block(codes)
    assert block.shape == (1, 16) and block[0, 0] == 0x95 and (block[0, 1:] == 0).all()
    assert np.array_equal(untranspose_block(block), codes)
    with pytest.raises(ValueError):
        transpose_block(np.zeros((15, 2), np.uint8))


def test_transpose_list_pads_and_round_trips(rng):
    packed = rng.integers(0, 256, (21, 4), dtype=np.uint8)
    ids = np.arange(21, dtype=np.int64) * 7
    tl = transpose_list(packed, ids)
    assert tl.nblocks == 2 and tl.count == 21 and tl.m == 8
    assert (tl.ids[21:] == PAD_ID).all() and (tl.blocks[1, :, 5:] == PAD_BYTE).all()
    c, i = untranspose_list(tl)
    assert np.array_equal(c, packed) and np.array_equal(i, ids)
    c, i = untranspose_list(tl, limit=5)
    assert np.array_equal(c, packed[:5])
    empty = transpose_list(np.zeros((0, 3), np.uint8), np.zeros(0, np.int64))
    assert empty.nblocks == 0 and empty.m == 6


def test_quantized_tables_validation():
    with pytest.raises(ValueError):
        QuantizedTables(np.full((1, 16), 128, np.uint8), 0.0, 1.0, np.zeros(1, np.float32))
    with pytest.raises(ValueError):
        QuantizedTables(np.zeros((1, 16), np.uint8), 0.0, -1.0, np.zeros(1, np.float32))
    with pytest.raises(ValueError):
        TransposedList(np.zeros((1, 2, 16), np.uint8), np.zeros(15, np.int64), 3)


def test_dequantize_is_two_rounding_midpoint():
    qt = QuantizedTables(np.zeros((1, 16), np.uint8), 1000.5, 0.37, np.zeros(1, np.float32))
    q = np.arange(256)
    want = np.float32(1000.5) + (q.astype(np.float32) + np.float32(0.5)) * np.float32(0.37)
    assert np.array_equal(dequantize(q, qt), want)


# ---------------------------------------------------------------- QIVF I/O

def test_qivf_round_trip(tmp_path, rng):
    cen = rng.standard_normal((3, 8)).astype(np.float32)
    lists = []
    for c in range(3):
        n = int(rng.integers(0, 40))
        lists.append(transpose_list(rng.integers(0, 256, (n, 2), dtype=np.uint8),
                                    np.sort(rng.choice(10**6, n, replace=False)).astype(np.int64)))
    idx = ivf.IvfIndex(d=8, m=4, b=4, coarse=ivf.Codebook(cen), lists=lists,
                       layout=ivf.LAYOUT_TRANSPOSED)
    p = tmp_path / "i.qivf"
    ivf.save_index(idx, p)
    back = ivf.load_index(p)
    assert back.layout == ivf.LAYOUT_TRANSPOSED and back.K == 3
    assert np.array_equal(back.coarse.centroids, cen)
    for a, b in zip(idx.lists, back.lists):
        assert np.array_equal(a.blocks, b.blocks) and np.array_equal(a.ids, b.ids)
    raw = p.read_bytes()
    (tmp_path / "t.qivf").write_bytes(raw[:-1])
    with pytest.raises(ivf.FormatError):
        ivf.load_index(tmp_path / "t.qivf")
    (tmp_path / "x.qivf").write_bytes(raw + b"\0")
    with pytest.raises(ivf.FormatError):
        ivf.load_index(tmp_path / "x.qivf")


def test_qivf_reads_reference_written_file():
    """A QIVF v1 file written by the reference's own save_index
    (tests/golden/ref_index.qivf, made by make_golden.py qivf: IVF K=5 with
    empty, partial and padded lists) loads here with identical lists."""
    from paper_1704_07355_b200.qadc import untranspose_list
    from conftest import GOLDEN
    want = golden("ref_index.npz")
    back = ivf.load_index(GOLDEN / "ref_index.qivf")
    assert np.array_equal(back.coarse.centroids, want["centroids"])
    off = np.concatenate([[0], np.cumsum(want["sizes"])])
    assert len(back.lists) == want["sizes"].shape[0]
    for L, lst in enumerate(back.lists):
        codes, ids = untranspose_list(lst)
        assert np.array_equal(codes, want["codes"][off[L]:off[L + 1]])
        assert np.array_equal(ids, want["ids"][off[L]:off[L + 1]])


# ---------------------------------------------------------------- workload

def test_mixture_generator_shapes_and_determinism():
    a = datagen.mixture_numpy(datagen.SIFT_LIKE, 1000, seed=3, stream=2)
    b = datagen.mixture_numpy(datagen.SIFT_LIKE, 1000, seed=3, stream=2)
    assert a.shape == (1000, 128) and a.dtype == np.float32 and (a >= 0).all()
    assert np.array_equal(a, b)
    g = datagen.mixture_numpy(datagen.GIST_LIKE, 10, seed=3, stream=2)
    assert g.shape == (10, 960) and g.max() < 2.0


def test_recall_ground_truth_matches_reference_synth():
    """recall.ground_truth (the GPU recall harness's exact k-NN, here on the
    CPU device) equals the reference's synth.ground_truth (synth.py:45-70,
    committed output): ids in exact fp64 order, ties to the lower id, over
    a base split into several chunks; recall_at follows bench.py:110-122."""
    import torch

    from paper_1704_07355_b200.recall import ground_truth, recall_at
    g = golden("ground_truth.npz")
    base = torch.from_numpy(g["base"])

    def chunks():
        for c0 in range(0, base.shape[0], 1700):
            yield c0, base[c0:c0 + 1700]
    got = ground_truth(chunks(), g["queries"], depth=10, device="cpu")
    assert np.array_equal(got, g["ids"])
    res = np.stack([np.roll(g["ids"][i], i % 3) for i in range(g["ids"].shape[0])])
    gt1 = g["ids"][:, 0]
    assert recall_at(res, gt1, 1) == np.mean([i % 3 == 0 for i in range(24)])
    assert recall_at(res, gt1, 3) == 1.0
