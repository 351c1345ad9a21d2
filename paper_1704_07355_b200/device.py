"""Device-resident index and the batched search entry point.

`DeviceIndex` owns a `qadc_b200_index` (include/qadc_b200.h): the coarse
centroids, the product quantizer and every inverted list repacked into the
interleaved32 HBM layout. It is built once from a reference-style index
(`from_ivf`) or straight from codes already on the GPU (`from_device_rows`)
and then answers whole query batches with `search`.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native


@dataclass
class BatchResult:
    ids: object  # (Q, R) int64, ascending (distance, id), -1 padding
    distances: object  # (Q, R) float32 midpoints, +inf padding
    counts: object  # (Q,) int32 results per query
    stats: dict


def _np(a, dtype):
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


class DeviceIndex:
    STAT_KEYS = ("codes", "candidates", "reruns", "scan_launches", "launches", "scan_us",
                 "scan_tc", "probe_us", "tables_us", "work_us", "select_us", "scan_tile_q")

    def __init__(self, handle: int, d: int, m: int, K: int, nlists: int, ncodes: int):
        self._h = handle
        self.d, self.m, self.K, self.nlists, self.ncodes = d, m, K, nlists, ncodes

    # ------------------------------------------------------------ building
    @classmethod
    def from_ivf(cls, index, pq) -> "DeviceIndex":
        """Upload a reference-layout IvfIndex (+ its ProductQuantizer)."""
        if (index.d, index.m, index.b) != (pq.m * pq.codebooks.shape[2], pq.m, pq.b):
            raise ValueError("index geometry does not match the quantizer")
        if index.b != 4:
            raise ValueError("the B200 scan needs 4-bit sub-codes")
        lib = _native.load_library()
        blocks, ids, blk_off, count = [], [], [0], []
        for lst in index.lists:
            if hasattr(lst, "blocks"):
                tb, ti, cnt = lst.blocks, lst.ids, lst.count
            else:  # standard layout: regroup on the host (byte moves only)
                from .qadc import transpose_list
                t = transpose_list(lst.codes, lst.ids)
                tb, ti, cnt = t.blocks, t.ids, t.count
            blocks.append(_np(tb, np.uint8).reshape(-1))
            ids.append(_np(ti, np.int64))
            blk_off.append(blk_off[-1] + tb.shape[0])
            count.append(cnt)
        blocks = np.concatenate(blocks) if blocks else np.zeros(0, np.uint8)
        ids = np.concatenate(ids) if ids else np.zeros(0, np.int64)
        blk_off = np.asarray(blk_off, dtype=np.int64)
        count = np.asarray(count, dtype=np.int64)
        coarse = None if index.coarse is None else _np(index.coarse.centroids, np.float32)
        cb = _np(pq.codebooks, np.float32)
        rot = None if getattr(pq, "rotation", None) is None else _np(pq.rotation, np.float32)
        h = ctypes.c_void_p()
        _native.check(lib.qadc_b200_index_create(
            index.d, index.m, len(index.lists), _native.ptr(coarse, ctypes.c_float),
            _native.ptr(blocks, ctypes.c_uint8), _native.ptr(blk_off, ctypes.c_int64),
            _native.ptr(ids, ctypes.c_int64), _native.ptr(count, ctypes.c_int64),
            _native.ptr(cb, ctypes.c_float), _native.ptr(rot, ctypes.c_float),
            ctypes.byref(h)), "index_create")
        return cls(h.value, index.d, index.m, index.K, len(index.lists), int(count.sum()))

    @classmethod
    def from_device_rows(cls, d: int, m: int, codes, row_off, codebooks, rotation=None,
                         coarse=None, ids=None) -> "DeviceIndex":
        """Index from packed rows already on the GPU (torch tensors):
        codes (n, m/2) uint8 in list order, row_off (nlists + 1) int64."""
        lib = _native.load_library()
        nl = row_off.shape[0] - 1
        h = ctypes.c_void_p()
        _native.check(lib.qadc_b200_index_create_device(
            d, m, nl, _native.dptr(coarse), _native.dptr(codes), _native.dptr(row_off),
            _native.dptr(ids), _native.dptr(codebooks), _native.dptr(rotation),
            ctypes.byref(h)), "index_create_device")
        return cls(h.value, d, m, 0 if coarse is None else nl, nl, int(codes.shape[0]))

    def set_prefix(self, rows, row_off, full_count, ids=None) -> None:
        """Install the GLOBAL first codes of every list (device rows in list
        order, row_off (nlists + 1) device int64, full_count host ints) as
        the prefix find_qmax / the saturation rule read: a shard holding
        part of a list then reproduces the unsharded search."""
        fc = _np(full_count, np.int64)
        _native.check(_native.load_library().qadc_b200_index_set_prefix_device(
            self._h, _native.dptr(rows), _native.dptr(row_off), _native.dptr(ids),
            _native.ptr(fc, ctypes.c_int64)), "index_set_prefix_device")

    # ------------------------------------------------------------ search
    def search(self, queries, R: int, ma: int = 1, init: int = 1000, lut=None, cells=None,
               stream=None, with_fsat: bool = True, scan: str = "auto") -> BatchResult:
        """Batched Quick ADC search. `queries` is a (Q, d) float32 torch
        tensor on the GPU (device I/O) or a numpy array (host I/O: the
        host<->device copies happen inside the call). lut/cells inject the
        float tables (Q, ma, m, 16) and probe order (Q, ma)."""
        import torch

        lib = _native.load_library()
        st = stream if stream is not None else torch.cuda.current_stream()
        stats = np.zeros(16, dtype=np.int64)
        flags = _native.LUT_IN if lut is not None else 0
        if not with_fsat:
            flags |= _native.NO_FSAT
        if scan not in ("auto", "prmt", "tc", "tc1", "tcw"):
            raise ValueError(f"unknown scan kernel {scan!r}")
        flags |= {"auto": 0, "prmt": _native.SCAN_PRMT, "tc": _native.SCAN_TC,
                  "tc1": _native.SCAN_TC | _native.SCAN_TC1, "tcw": _native.SCAN_TCW}[scan]
        if isinstance(queries, np.ndarray):
            q = _np(queries, np.float32).reshape(-1, self.d)
            nq = q.shape[0]
            ids = np.empty((nq, R), np.int64)
            dist = np.empty((nq, R), np.float32)
            cnt = np.empty(nq, np.int32)
            lut_h = None if lut is None else _np(lut, np.float32)
            cells_h = None if cells is None else _np(cells, np.int64)
            rc = lib.qadc_b200_search_batch(
                self._h, q.ctypes.data, nq, R, ma, init, flags | _native.HOST_IO,
                None if lut_h is None else lut_h.ctypes.data,
                None if cells_h is None else cells_h.ctypes.data,
                ids.ctypes.data, dist.ctypes.data, cnt.ctypes.data, st.cuda_stream,
                stats.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
        else:
            q = queries.to(dtype=torch.float32).contiguous()
            nq = q.shape[0]
            dev = q.device
            ids = torch.empty((nq, R), dtype=torch.int64, device=dev)
            dist = torch.empty((nq, R), dtype=torch.float32, device=dev)
            cnt = torch.empty(nq, dtype=torch.int32, device=dev)
            lut_d = None if lut is None else lut.to(dtype=torch.float32).contiguous()
            cells_d = None if cells is None else cells.to(dtype=torch.int64).contiguous()
            rc = lib.qadc_b200_search_batch(
                self._h, _native.dptr(q), nq, R, ma, init, flags, _native.dptr(lut_d),
                _native.dptr(cells_d), _native.dptr(ids), _native.dptr(dist), _native.dptr(cnt),
                st.cuda_stream, stats.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
        _native.check(rc, "search_batch")
        return BatchResult(ids, dist, cnt, {k: int(v) for k, v in zip(self.STAT_KEYS, stats)})

    # the per-query state between the two halves of a search (prepare ->
    # scan), in the order of qadc_b200_search_prepare's output arguments
    PREP_KEYS = ("cells", "qt", "qmin_f", "delta_f", "depth", "qmax", "M_bits", "fsat_n",
                 "fsat_mid", "fsat_id")

    def prep_buffers(self, nq: int, R: int, ma: int = 1, device="cuda") -> dict:
        """Empty prepared-state tensors for nq queries (see prepare)."""
        import torch

        w = ma if self.K else 1
        i64, f32, u8, i32 = torch.int64, torch.float32, torch.uint8, torch.int32
        return {"cells": torch.zeros((nq, w), dtype=i64, device=device),
                "qt": torch.empty((nq, w, self.m * 4), dtype=torch.int32, device=device),
                "qmin_f": torch.empty((nq, w), dtype=f32, device=device),
                "delta_f": torch.empty((nq, w), dtype=f32, device=device),
                "depth": torch.empty((nq, w), dtype=u8, device=device),
                "qmax": torch.empty(nq, dtype=f32, device=device),
                "M_bits": torch.empty(nq, dtype=i32, device=device),
                "fsat_n": torch.empty(nq, dtype=i32, device=device),
                # entries past fsat_n are never read; zeroed so that states
                # assembled from slices compare equal
                "fsat_mid": torch.zeros((nq, R), dtype=f32, device=device),
                "fsat_id": torch.zeros((nq, R), dtype=i64, device=device)}

    def prepare(self, queries, R: int, ma: int = 1, init: int = 1000, with_fsat: bool = True,
                out: dict | None = None, stream=None) -> dict:
        """First half of `search`: the Index + Tables phases (adc.py:140-174)
        of every query — probe order, uint8 tables, qmin / delta, qmax,
        initial bound and F_sat — into device tensors (`out`, or new ones).
        `queries` is a (Q, d) float32 device tensor."""
        import torch

        st = stream if stream is not None else torch.cuda.current_stream()
        q = queries.to(dtype=torch.float32).contiguous()
        p = out if out is not None else self.prep_buffers(q.shape[0], R, ma, q.device)
        flags = 0 if with_fsat else _native.NO_FSAT
        _native.check(_native.load_library().qadc_b200_search_prepare(
            self._h, _native.dptr(q), q.shape[0], R, ma, init, flags, None, None,
            *[_native.dptr(p[k]) for k in self.PREP_KEYS], st.cuda_stream, None), "search_prepare")
        return p

    def scan(self, prep: dict, R: int, ma: int = 1, init: int = 1000, stream=None,
             scan: str = "auto") -> BatchResult:
        """Second half of `search`: work list, scan and exact top-R over a
        prepared state (prepare, possibly assembled from other ranks)."""
        import torch

        st = stream if stream is not None else torch.cuda.current_stream()
        nq = prep["M_bits"].shape[0]
        dev = prep["M_bits"].device
        ids = torch.empty((nq, R), dtype=torch.int64, device=dev)
        dist = torch.empty((nq, R), dtype=torch.float32, device=dev)
        cnt = torch.empty(nq, dtype=torch.int32, device=dev)
        flags = {"auto": 0, "prmt": _native.SCAN_PRMT, "tc": _native.SCAN_TC,
                 "tc1": _native.SCAN_TC | _native.SCAN_TC1, "tcw": _native.SCAN_TCW}[scan]
        stats = np.zeros(16, dtype=np.int64)
        _native.check(_native.load_library().qadc_b200_search_scan(
            self._h, nq, R, ma, init, flags, *[_native.dptr(prep[k]) for k in self.PREP_KEYS
                                               if k != "qmax"],
            _native.dptr(ids), _native.dptr(dist), _native.dptr(cnt), st.cuda_stream,
            stats.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))), "search_scan")
        return BatchResult(ids, dist, cnt, {k: int(v) for k, v in zip(self.STAT_KEYS, stats)})

    def tables(self, queries, R: int, ma: int = 1, init: int = 1000, stream=None) -> dict:
        """The Index + Tables phases of `search` (adc.py:140-174) with their
        intermediates, for native-mode parity accounting: cells (Q, ma),
        fp32 LUTs (Q, ma, m, 16), qmax (Q,), uint8 tables (Q, ma, m, 16),
        and the fp32 qmin / delta (Q, ma) the scan uses. `queries` is a
        (Q, d) float32 device tensor."""
        import torch

        st = stream if stream is not None else torch.cuda.current_stream()
        q = queries.to(dtype=torch.float32).contiguous()
        nq, dev = q.shape[0], q.device
        slots = ma if self.K else 1
        out = {
            "cells": torch.zeros((nq, slots), dtype=torch.int64, device=dev),
            "lut": torch.empty((nq, slots, self.m, 16), dtype=torch.float32, device=dev),
            "qmax": torch.empty(nq, dtype=torch.float32, device=dev),
            "qt": torch.empty((nq, slots, self.m, 16), dtype=torch.uint8, device=dev),
            "qmin": torch.empty((nq, slots), dtype=torch.float32, device=dev),
            "delta": torch.empty((nq, slots), dtype=torch.float32, device=dev),
        }
        _native.check(_native.load_library().qadc_b200_search_tables(
            self._h, _native.dptr(q), nq, R, ma, init,
            _native.dptr(out["cells"]) if self.K else None, _native.dptr(out["lut"]),
            _native.dptr(out["qmax"]), _native.dptr(out["qt"]), _native.dptr(out["qmin"]),
            _native.dptr(out["delta"]), st.cuda_stream), "search_tables")
        return out

    @property
    def nbytes(self) -> int:
        return int(_native.load_library().qadc_b200_index_bytes(self._h)) if self._h else 0

    def close(self) -> None:
        if self._h:
            _native.load_library().qadc_b200_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
