"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the CPU oracle.

Two libraries, both CPU:
  * oracle/_build/libqadc_oracle.so — C restatement of the reference's
    Quick ADC search path (qadc_oracle.c, every function cites the
    reference file:line it restates);
  * oracle/_ref/libqadc_ref.so — the reference's OWN scan kernels
    (/root/reference/pkg/src/qadc/src/scan_kernels.c) compiled in place by
    oracle/Makefile (`make ref`), when that source was available at build
    time.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this module; the product package never does.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_int64, c_uint8, c_void_p
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "_build" / "libqadc_oracle.so"
REF_LIB = HERE / "_ref" / "libqadc_ref.so"

_u8p, _i64p, _f32p, _i32p, _f64p = (POINTER(c_uint8), POINTER(c_int64), POINTER(c_float),
                                     POINTER(ctypes.c_int32), POINTER(c_double))
SCAN_FN = ctypes.CFUNCTYPE(c_int, _u8p, c_int64, _i64p, c_int, _u8p, c_float, c_float, _f32p,
                           _i64p, c_int, c_int, c_int)

_orc = None
_ref = None


def _p(a, t):
    return None if a is None else a.ctypes.data_as(POINTER(t))


def lib():
    global _orc
    if _orc is None:
        if not ORACLE_LIB.exists():
            import subprocess
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        L = ctypes.CDLL(str(ORACLE_LIB))
        L.orc_einsum_sqdist.restype = c_float
        L.orc_einsum_sqdist.argtypes = [_f32p, _f32p, c_int]
        L.orc_sum_f32.restype = c_float
        L.orc_sum_f32.argtypes = [_f32p, c_int]
        L.orc_compute_tables.argtypes = [_f32p, c_int, c_int, _f32p, _f32p]
        L.orc_probe.argtypes = [_f32p, c_int, c_int, _f32p, c_int, _i64p, _f32p]
        L.orc_rotate.argtypes = [_f32p, c_int, _f32p, _f32p]
        L.orc_find_qmax.restype = c_float
        L.orc_find_qmax.argtypes = [_f32p, c_int, _u8p, c_int64, c_int, c_int]
        L.orc_quantize_tables.restype = c_double
        L.orc_quantize_tables.argtypes = [_f32p, c_int, c_double, c_double, _u8p]
        L.orc_block_dists.argtypes = [_u8p, c_int64, c_int, _u8p, c_int, _u8p]
        L.orc_qadc_scan.restype = c_int
        L.orc_qadc_scan.argtypes = [_u8p, c_int64, _i64p, c_int, _u8p, c_float, c_float, _f32p,
                                    _i64p, c_int, c_int]
        L.orc_adc_scan_f32.restype = c_int
        L.orc_adc_scan_f32.argtypes = [_u8p, c_int64, _i64p, c_int, c_int, _f32p, _f32p, _i64p,
                                       c_int, c_int]
        L.orc_heap_extract.argtypes = [_f32p, _i64p, c_int]
        L.orc_search_batch.argtypes = [_f32p, c_int, c_int, c_int, _f32p, _f32p, _f32p, c_int,
                                       c_int, _u8p, _i64p, _i64p, _i64p, c_int, c_int, _f32p,
                                       _i64p, c_void_p, c_int, c_int, _i64p, _f32p, _i32p, _f64p]
        L.orc_search_batch_sharded.argtypes = [
            _f32p, c_int, c_int, c_int, _f32p, _f32p, _f32p, c_int, c_int, _u8p, _i64p, _i64p,
            _u8p, _i64p, _i64p, _i64p, c_int, c_int, c_int, c_int, _i64p, _f32p, _i32p]
        _orc = L
    return _orc


def ref_lib():
    """The reference's own compiled scan kernels, or None if not built."""
    global _ref
    if _ref is None and REF_LIB.exists():
        R = ctypes.CDLL(str(REF_LIB))
        R.qadc_simd_level.restype = c_int
        R.qadc_scan_u8.restype = c_int
        R.qadc_scan_u8.argtypes = [_u8p, c_int64, _i64p, c_int, _u8p, c_float, c_float, _f32p,
                                   _i64p, c_int, c_int, c_int]
        R.qadc_block_dists.argtypes = [_u8p, c_int64, c_int, _u8p, c_int, _u8p, c_int]
        R.adc_scan_f32.restype = c_int
        R.adc_scan_f32.argtypes = [_u8p, c_int64, _i64p, c_int, c_int, _f32p, _f32p, _i64p, c_int,
                                   c_int]
        _ref = R
    return _ref


# ------------------------------------------------------------------ helpers

def einsum_sqdist(a, b) -> np.float32:
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return np.float32(lib().orc_einsum_sqdist(_p(a, c_float), _p(b, c_float), a.shape[0]))


def sum_f32(x) -> np.float32:
    x = np.ascontiguousarray(x, np.float32)
    return np.float32(lib().orc_sum_f32(_p(x, c_float), x.shape[0]))


def compute_tables(codebooks, y) -> np.ndarray:
    cb = np.ascontiguousarray(codebooks, np.float32)
    y = np.ascontiguousarray(y, np.float32).ravel()
    m, _, dsub = cb.shape
    out = np.empty((m, 16), np.float32)
    lib().orc_compute_tables(_p(cb, c_float), m, dsub, _p(y, c_float), _p(out, c_float))
    return out


def probe(cent, q, ma):
    cent = np.ascontiguousarray(cent, np.float32)
    q = np.ascontiguousarray(q, np.float32).ravel()
    K, d = cent.shape
    cells = np.empty(ma, np.int64)
    res = np.empty((ma, d), np.float32)
    lib().orc_probe(_p(cent, c_float), K, d, _p(q, c_float), ma, _p(cells, c_int64),
                    _p(res, c_float))
    return cells, res


def rotate(R, v):
    R = np.ascontiguousarray(R, np.float32)
    v = np.ascontiguousarray(v, np.float32).ravel()
    out = np.empty_like(v)
    lib().orc_rotate(_p(R, c_float), v.shape[0], _p(v, c_float), _p(out, c_float))
    return out


def find_qmax(tables, blocks, count, R, init) -> float:
    t = np.ascontiguousarray(tables, np.float32)
    b = np.ascontiguousarray(blocks, np.uint8)
    return float(lib().orc_find_qmax(_p(t, c_float), t.shape[0], _p(b, c_uint8), count, R, init))


def quantize_tables(tables, qmin, qmax):
    t = np.ascontiguousarray(tables, np.float32)
    out = np.empty(t.shape, np.uint8)
    delta = lib().orc_quantize_tables(_p(t, c_float), t.shape[0], float(qmin), float(qmax),
                                      _p(out, c_uint8))
    return out, float(delta)


def block_dists(blocks, qt) -> np.ndarray:
    b = np.ascontiguousarray(blocks, np.uint8)
    q = np.ascontiguousarray(qt, np.uint8)
    out = np.empty((b.shape[0], 16), np.uint8)
    lib().orc_block_dists(_p(b, c_uint8), b.shape[0], b.shape[1], _p(q, c_uint8),
                          int(q.ndim == 3), _p(out, c_uint8))
    return out


def qadc_scan(blocks, ids, qt, qmin, delta, heap_d, heap_i, size, R):
    """Sequential reference heap semantics; returns (ids, dists) sorted."""
    b = np.ascontiguousarray(blocks, np.uint8)
    i = np.ascontiguousarray(ids, np.int64)
    q = np.ascontiguousarray(qt, np.uint8)
    hd = np.zeros(R, np.float32)
    hi = np.zeros(R, np.int64)
    hd[:size] = heap_d[:size]
    hi[:size] = heap_i[:size]
    n = lib().orc_qadc_scan(_p(b, c_uint8), b.shape[0], _p(i, c_int64), b.shape[1],
                            _p(q, c_uint8), float(qmin), float(delta), _p(hd, c_float),
                            _p(hi, c_int64), size, R)
    lib().orc_heap_extract(_p(hd, c_float), _p(hi, c_int64), n)
    return hi[:n].copy(), hd[:n].copy()


def flatten_index(index):
    """(blocks, blk_off, ids, count) of a reference-layout index."""
    blocks, ids, off, count = [], [], [0], []
    for lst in index.lists:
        blocks.append(np.ascontiguousarray(lst.blocks, np.uint8).reshape(-1))
        ids.append(np.ascontiguousarray(lst.ids, np.int64))
        off.append(off[-1] + lst.blocks.shape[0])
        count.append(lst.count)
    return (np.concatenate(blocks), np.asarray(off, np.int64), np.concatenate(ids),
            np.asarray(count, np.int64))


def search_batch(queries, codebooks, rotation, coarse, ma, flat, R, init, lut_in=None,
                 cells_in=None, use_ref_scan=False, nthreads=None):
    """adc.search(method='qadc') for every query (C restatement); with
    use_ref_scan the block scan is the reference's own qadc_scan_u8."""
    blocks, blk_off, ids, count = flat
    q = np.ascontiguousarray(queries, np.float32)
    nq, d = q.shape
    cb = np.ascontiguousarray(codebooks, np.float32)
    m = cb.shape[0]
    rot = None if rotation is None else np.ascontiguousarray(rotation, np.float32)
    cent = None if coarse is None else np.ascontiguousarray(coarse, np.float32)
    K = 0 if cent is None else cent.shape[0]
    out_i = np.empty((nq, R), np.int64)
    out_d = np.empty((nq, R), np.float32)
    out_n = np.empty(nq, np.int32)
    diag = np.empty((nq, 2), np.float64)
    lut = None if lut_in is None else np.ascontiguousarray(lut_in, np.float32)
    cin = None if cells_in is None else np.ascontiguousarray(cells_in, np.int64)
    fn, variant = None, 0
    if use_ref_scan:
        R_ = ref_lib()
        if R_ is None:
            raise RuntimeError("oracle/_ref/libqadc_ref.so is not built")
        fn = ctypes.cast(R_.qadc_scan_u8, c_void_p)
        variant = int(R_.qadc_simd_level())
    lib().orc_search_batch(_p(q, c_float), nq, d, m, _p(cb, c_float), _p(rot, c_float),
                           _p(cent, c_float), K, ma, _p(blocks, c_uint8), _p(blk_off, c_int64),
                           _p(ids, c_int64), _p(count, c_int64), R, init, _p(lut, c_float),
                           _p(cin, c_int64), fn, variant, nthreads or (os.cpu_count() or 1),
                           _p(out_i, c_int64), _p(out_d, c_float), out_n.ctypes.data_as(_i32p),
                           _p(diag, c_double))
    return out_i, out_d, out_n, diag


def search_batch_sharded(queries, codebooks, rotation, coarse, ma, flat, prefix, R, init,
                         with_fsat=True, nthreads=None):
    """One shard's adc.search(method='qadc') results (C restatement,
    order-free form): `flat` = the shard's (blocks, blk_off, ids, count),
    `prefix` = (blocks, blk_off, ids, global_count) of the GLOBAL first
    codes of every list. Merging all shards' outputs by (dist, id) equals
    search_batch on the unsharded index."""
    blocks, blk_off, ids, _ = flat
    pblocks, pblk_off, pids, pcount = (np.ascontiguousarray(a) for a in prefix)
    q = np.ascontiguousarray(queries, np.float32)
    nq, d = q.shape
    cb = np.ascontiguousarray(codebooks, np.float32)
    m = cb.shape[0]
    rot = None if rotation is None else np.ascontiguousarray(rotation, np.float32)
    cent = None if coarse is None else np.ascontiguousarray(coarse, np.float32)
    K = 0 if cent is None else cent.shape[0]
    out_i = np.empty((nq, R), np.int64)
    out_d = np.empty((nq, R), np.float32)
    out_n = np.empty(nq, np.int32)
    lib().orc_search_batch_sharded(
        _p(q, c_float), nq, d, m, _p(cb, c_float), _p(rot, c_float), _p(cent, c_float), K, ma,
        _p(np.ascontiguousarray(blocks, np.uint8), c_uint8),
        _p(np.ascontiguousarray(blk_off, np.int64), c_int64),
        _p(np.ascontiguousarray(ids, np.int64), c_int64),
        _p(pblocks.astype(np.uint8, copy=False), c_uint8),
        _p(pblk_off.astype(np.int64, copy=False), c_int64),
        _p(pids.astype(np.int64, copy=False), c_int64),
        _p(pcount.astype(np.int64, copy=False), c_int64), R, init, int(bool(with_fsat)),
        nthreads or (os.cpu_count() or 1), _p(out_i, c_int64), _p(out_d, c_float),
        out_n.ctypes.data_as(_i32p))
    return out_i, out_d, out_n
