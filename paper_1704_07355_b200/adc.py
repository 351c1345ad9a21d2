"""Search API (mirror of the reference's adc.py) on the B200.

Same names and semantics as /root/reference/pkg/src/qadc/adc.py:
`compute_tables` (:61-75), `adc_distance` (:84-93), `scan_list` (:96-105),
`search` (:114-187) with the reference's validation and result order
(ids ascending by (distance, id), fp32 distances). Additions:

  * `search_batch(index, pq, queries, R, ma, init)` — the whole batch in
    one device call (the reference only has the per-query loop of
    bench.py:182-191);
  * `device_index(index, pq)` — the cached device-resident index.

method="qadc" runs the batched B200 path (qadc_b200_search_batch) even for
a single query; method="adc" runs the float-table scan (adc_scan_f32).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _native, kernels
from . import ivf as ivfmod
from .device import BatchResult, DeviceIndex
from .heap import NeighborHeap

__all__ = ["LookupTables", "PhaseTimings", "SearchResult", "NeighborHeap", "compute_tables",
           "adc_distance", "scan_list", "search", "search_batch", "device_index"]

DEFAULT_INIT = 1000  # adc.py:27


@dataclass(frozen=True)
class LookupTables:
    tables: np.ndarray  # (m, k) float32
    query_ref: int | None = None

    @property
    def m(self) -> int:
        return self.tables.shape[0]

    @property
    def k(self) -> int:
        return self.tables.shape[1]


@dataclass(frozen=True)
class PhaseTimings:
    index_ms: float
    tables_ms: float
    scan_ms: float
    total_ms: float


@dataclass(frozen=True)
class SearchResult:
    ids: np.ndarray
    distances: np.ndarray
    timings: PhaseTimings


def _pq_d(pq) -> int:
    return pq.m * pq.codebooks.shape[2]


def compute_tables(pq, residual_query, query_ref: int | None = None) -> LookupTables:
    """(m, 16) fp32 squared distances in NumPy einsum order, on the GPU.
    The residual must already be rotated for an OPQ quantizer."""
    import torch

    r = np.ascontiguousarray(np.asarray(residual_query, dtype=np.float32).ravel())
    d = _pq_d(pq)
    if r.shape[0] != d:
        raise ValueError(f"query dim {r.shape[0]} != quantizer dim {d}")
    if pq.codebooks.shape[1] != 16:
        raise ValueError("the B200 table kernel serves 4-bit (16-centroid) quantizers")
    dev = torch.device("cuda")
    cb = torch.from_numpy(np.ascontiguousarray(pq.codebooks, dtype=np.float32)).to(dev)
    y = torch.from_numpy(r).to(dev)
    out = torch.empty((pq.m, 16), dtype=torch.float32, device=dev)
    _native.check(_native.load_library().qadc_b200_compute_tables(
        _native.dptr(cb), pq.m, pq.codebooks.shape[2], _native.dptr(y), 1, _native.dptr(out),
        torch.cuda.current_stream().cuda_stream), "compute_tables")
    return LookupTables(tables=out.cpu().numpy(), query_ref=query_ref)


def _tables_array(tables) -> np.ndarray:
    if isinstance(tables, LookupTables):
        return tables.tables
    return np.ascontiguousarray(tables, dtype=np.float32)


def adc_distance(code, tables) -> float:
    """One code's table sum, left to right in fp32 (adc.py:84-93)."""
    t = _tables_array(tables)
    idx = getattr(code, "codes", code)
    idx = np.asarray(idx)
    if idx.shape[0] != t.shape[0]:
        raise ValueError("code length does not match the table count")
    acc = np.float32(0.0)
    for j in range(t.shape[0]):
        acc = np.float32(acc + t[j, int(idx[j])])
    return float(acc)


def scan_list(lst, tables, heap: NeighborHeap, variant: str | None = None) -> NeighborHeap:
    """Float scan of a standard-layout list into `heap`."""
    t = _tables_array(tables)
    k = t.shape[1]
    b = int(k).bit_length() - 1
    if (1 << b) != k:
        raise ValueError("table length must be a power of two")
    kernels.scan_codes(lst.codes, lst.ids, t, b, heap, variant)
    return heap


def _rotate(pq, v: np.ndarray) -> np.ndarray:
    if getattr(pq, "rotation", None) is None:
        return v
    return (v @ pq.rotation.T).astype(np.float32)


def device_index(index, pq) -> DeviceIndex:
    """The DeviceIndex for (index, pq), built on first use and cached on
    the index object. The key holds the identity of the quantizer arrays
    and of every list (object, code / block array, count), so replacing or
    re-encoding a list, or a new quantizer, rebuilds the device copy; the
    cached entry keeps references to the keyed objects, so their ids cannot
    be recycled while it lives. `invalidate_device_index` drops it
    explicitly (in-place edits of a list's arrays are not detectable)."""
    parts = [pq, pq.codebooks, getattr(pq, "rotation", None), index.coarse]
    for lst in index.lists:
        parts += [lst, getattr(lst, "blocks", getattr(lst, "codes", None)), lst.ids]
    key = tuple(id(p) for p in parts) + tuple(int(lst.count) for lst in index.lists)
    cached = getattr(index, "_b200_device", None)
    if cached is not None and cached[0] == key:
        return cached[1]
    dev = DeviceIndex.from_ivf(index, pq)
    try:
        index._b200_device = (key, dev, parts)
    except AttributeError:
        pass
    return dev


def invalidate_device_index(index) -> None:
    """Drop the cached device copy of `index` (after editing its lists in
    place)."""
    cached = getattr(index, "_b200_device", None)
    if cached is not None:
        cached[1].close()
        index._b200_device = None


def _validate(index, pq, R: int, method: str) -> None:
    if R < 1:
        raise ValueError("R must be positive")
    if method not in ("adc", "qadc"):
        raise ValueError(f"unknown method {method!r}")
    if (index.d, index.m, index.b) != (_pq_d(pq), pq.m, pq.b):
        raise ValueError("index geometry does not match the quantizer")
    if method == "adc" and index.layout != ivfmod.LAYOUT_STANDARD:
        raise ValueError("adc search needs a standard-layout index")
    if method == "qadc":
        if index.layout != ivfmod.LAYOUT_TRANSPOSED:
            raise ValueError("qadc search needs a transposed16 index")
        if pq.b != 4:
            raise ValueError("qadc search needs 4-bit sub-codes")


def search_batch(index, pq, queries, R: int, ma: int = 1, init: int = DEFAULT_INIT,
                 lut=None, cells=None) -> BatchResult:
    """Quick ADC search of every row of `queries` (numpy (Q, d) or a CUDA
    tensor) in one device call; results as (Q, R) arrays padded with
    -1 / +inf and per-query counts. Equal, query by query, to
    search(index, pq, q, R, ma, method="qadc", init=init)."""
    _validate(index, pq, R, "qadc")
    if init < 1:
        raise ValueError("init must be positive")
    if index.coarse is not None:
        if ma < 1:
            raise ValueError("ma must be positive")
        if ma > index.K:
            raise ValueError(f"ma={ma} exceeds the cell count K={index.K}")
    if isinstance(queries, np.ndarray) or not hasattr(queries, "device"):
        q = np.ascontiguousarray(np.asarray(queries, dtype=np.float32))
        if q.ndim == 1:
            q = q[None]
        if q.shape[1] != index.d:
            raise ValueError("query dimension does not match the index")
        queries = q
    return device_index(index, pq).search(queries, R, ma=ma, init=init, lut=lut, cells=cells)


def search(index, pq, query, R: int, ma: int = 1, method: str = "adc",
           init: int = DEFAULT_INIT, variant: str | None = None) -> SearchResult:
    """Top-R ids of one query with per-phase wall times (adc.py:114-187)."""
    _validate(index, pq, R, method)
    kernels.resolve_variant(variant)
    q = np.asarray(query, dtype=np.float32).ravel()
    if q.shape[0] != index.d:
        raise ValueError("query dimension does not match the index")
    if method == "qadc":
        if init < 1:
            raise ValueError("init must be positive")
        if index.coarse is not None and not 1 <= ma <= index.K:
            raise ValueError("ma out of range")
        t0 = time.perf_counter()
        dev = device_index(index, pq)
        t1 = time.perf_counter()
        res = dev.search(q[None], R, ma=ma, init=init)
        t2 = time.perf_counter()
        n = int(res.counts[0])
        # phases from the device events of the call (adc.py:140-179): Index
        # = probe (+ the one-time index upload on the first call), Tables =
        # residual, rotation, LUT, qmax, quantize; Scan = the rest of the
        # call's wall time (work list, scan, exact top-R, host overhead)
        st = res.stats
        idx_ms = (t1 - t0) * 1e3 + st["probe_us"] / 1e3
        tab_ms = st["tables_us"] / 1e3
        scan_ms = max(0.0, (t2 - t1) * 1e3 - (st["probe_us"] + st["tables_us"]) / 1e3)
        return SearchResult(ids=res.ids[0, :n].copy(), distances=res.distances[0, :n].copy(),
                            timings=PhaseTimings(idx_ms, tab_ms, scan_ms,
                                                 idx_ms + tab_ms + scan_ms))
    # float-table ADC (method="adc")
    t0 = time.perf_counter()
    if index.coarse is None:
        cells, residuals = np.zeros(1, np.int64), q[None, :]
    else:
        ps = ivfmod.probe(index, q, ma)
        cells, residuals = ps.cells, ps.residual_queries
    index_ms = (time.perf_counter() - t0) * 1e3
    heap = NeighborHeap(R)
    tables_ms = scan_ms = 0.0
    for c, r in zip(cells, residuals):
        t1 = time.perf_counter()
        tabs = compute_tables(pq, _rotate(pq, r), query_ref=int(c))
        t2 = time.perf_counter()
        scan_list(index.lists[int(c)], tabs, heap, variant)
        t3 = time.perf_counter()
        tables_ms += (t2 - t1) * 1e3
        scan_ms += (t3 - t2) * 1e3
    ids, dists = heap.extract()
    return SearchResult(ids=ids, distances=dists,
                        timings=PhaseTimings(index_ms, tables_ms, scan_ms,
                                             index_ms + tables_ms + scan_ms))
