"""Inverted-file index types, GPU probe and GPU index build.

Mirrors /root/reference/pkg/src/qadc/ivf.py: `IvfIndex` (:66-92),
`StandardList` (:40-55), `ProbeSet` (:58-63), `probe` (:166-182),
`build_flat` (:154-163), QIVF v1 `save_index` / `load_index` (:185-244).
Reference index objects (and ProductQuantizer objects) are accepted
wherever these are (duck typing on .d/.m/.b/.coarse/.lists/.layout).

GPU parts: `probe` runs the einsum-order coarse distance + (d2, cell)
selection kernel; `build_flat` / `build_with_coarse` encode on the GPU
(qadc_b200_encode / qadc_b200_assign). Codebook and coarse
k-means *training* stay in the reference (BASELINE north_star).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from . import _native
from .qadc import TransposedList, transpose_list, untranspose_list

INDEX_MAGIC = b"QIVF"
INDEX_VERSION = 1
LAYOUT_STANDARD = "standard"
LAYOUT_TRANSPOSED = "transposed16"
_LAYOUT_TAGS = {LAYOUT_STANDARD: 0, LAYOUT_TRANSPOSED: 1}
_TAG_LAYOUTS = {v: k for k, v in _LAYOUT_TAGS.items()}


class FormatError(ValueError):
    """Malformed index file (the reference's vecio.FormatError)."""


@dataclass(frozen=True)
class Codebook:
    centroids: np.ndarray  # (k, dim) float32

    @property
    def k(self) -> int:
        return self.centroids.shape[0]

    @property
    def dim(self) -> int:
        return self.centroids.shape[1]


@dataclass(frozen=True)
class StandardList:
    ids: np.ndarray  # (n,) int64
    codes: np.ndarray  # (n, code_bytes) uint8

    def __post_init__(self):
        if self.codes.ndim != 2 or self.codes.dtype != np.uint8:
            raise ValueError("codes must be a uint8 matrix")
        if self.ids.shape != (self.codes.shape[0],):
            raise ValueError("ids must parallel the code rows")

    @property
    def count(self) -> int:
        return self.codes.shape[0]


@dataclass(frozen=True)
class ProbeSet:
    cells: np.ndarray  # (ma,) int64, ascending coarse distance, ties -> lower id
    residual_queries: np.ndarray  # (ma, d) float32


@dataclass
class IvfIndex:
    d: int
    m: int
    b: int
    coarse: object | None  # Codebook-like (.centroids) or None for a flat index
    lists: list
    layout: str

    def __post_init__(self):
        if self.layout not in _LAYOUT_TAGS:
            raise ValueError(f"unknown layout {self.layout!r}")
        want = self.coarse.centroids.shape[0] if self.coarse is not None else 1
        if len(self.lists) != want:
            raise ValueError("list count must match the coarse codebook")

    @property
    def nlists(self) -> int:
        return len(self.lists)

    @property
    def K(self) -> int:
        return self.coarse.centroids.shape[0] if self.coarse is not None else 0

    @property
    def count(self) -> int:
        return sum(lst.count for lst in self.lists)


def _row_bytes(m: int, b: int) -> int:
    if b == 4:
        return m // 2
    if b == 8:
        return m
    if b == 16:
        return 2 * m
    raise ValueError(f"unsupported b={b}")


def _make_list(codes: np.ndarray, ids: np.ndarray, layout: str):
    if layout == LAYOUT_TRANSPOSED:
        return transpose_list(codes, ids)
    return StandardList(ids=np.ascontiguousarray(ids, dtype=np.int64),
                        codes=np.ascontiguousarray(codes, dtype=np.uint8))


def _canonical(lst):
    if isinstance(lst, TransposedList) or hasattr(lst, "blocks"):
        return untranspose_list(lst)
    return lst.codes, lst.ids


def _check_layout(pq, layout: str) -> None:
    if layout not in _LAYOUT_TAGS:
        raise ValueError(f"unknown layout {layout!r}")
    if layout == LAYOUT_TRANSPOSED and pq.b != 4:
        raise ValueError("transposed16 layout requires 4-bit sub-codes")


# ---------------------------------------------------------------- probe

def probe(index, query, ma: int) -> ProbeSet:
    """ma nearest coarse cells (einsum-order d2, ties -> lower cell id) and
    the fp32 residual queries, computed on the GPU."""
    import torch

    if index.coarse is None:
        raise ValueError("a flat index has no cells to probe")
    if ma < 1:
        raise ValueError("ma must be positive")
    K = index.coarse.centroids.shape[0]
    if ma > K:
        raise ValueError(f"ma={ma} exceeds the cell count K={K}")
    q = np.asarray(query, dtype=np.float32).ravel()
    if q.shape[0] != index.d:
        raise ValueError("query dimension does not match the index")
    dev = torch.device("cuda")
    cent = torch.from_numpy(np.ascontiguousarray(index.coarse.centroids, dtype=np.float32)).to(dev)
    qd = torch.from_numpy(q).to(dev)
    cells = torch.empty(ma, dtype=torch.int64, device=dev)
    res = torch.empty((ma, index.d), dtype=torch.float32, device=dev)
    lib = _native.load_library()
    _native.check(lib.qadc_b200_probe(_native.dptr(cent), K, index.d, _native.dptr(qd), 1, ma,
                                      _native.dptr(cells), _native.dptr(res),
                                      torch.cuda.current_stream().cuda_stream), "probe")
    return ProbeSet(cells=cells.cpu().numpy(), residual_queries=res.cpu().numpy())


# ---------------------------------------------------------------- GPU build

def encode_device(pq, X):
    """Packed codes (n, m/2) uint8 of the rows of X (torch, on the GPU)."""
    import torch

    if pq.b != 4:
        raise ValueError("the B200 encoder produces 4-bit codes")
    X = X.to(dtype=torch.float32).contiguous()
    n, d = X.shape
    if d != pq.m * pq.codebooks.shape[2]:
        raise ValueError(f"vector dim {d} != quantizer dim")
    cb = torch.from_numpy(np.ascontiguousarray(pq.codebooks, dtype=np.float32)).to(X.device)
    rot = None
    if getattr(pq, "rotation", None) is not None:
        rot = torch.from_numpy(np.ascontiguousarray(pq.rotation, dtype=np.float32)).to(X.device)
    out = torch.empty((n, pq.m // 2), dtype=torch.uint8, device=X.device)
    lib = _native.load_library()
    _native.check(lib.qadc_b200_encode(_native.dptr(X), n, d, pq.m, _native.dptr(cb),
                                       _native.dptr(rot), _native.dptr(out),
                                       torch.cuda.current_stream().cuda_stream), "encode")
    return out


def assign_device(centroids, X):
    """Nearest coarse centroid per row of X (torch, on the GPU); centroids
    as a numpy array or a device tensor."""
    import torch

    if isinstance(centroids, torch.Tensor):
        C = centroids.to(device=X.device, dtype=torch.float32).contiguous()
    else:
        C = torch.as_tensor(np.ascontiguousarray(centroids, dtype=np.float32)).to(X.device)
    X = X.to(dtype=torch.float32).contiguous()
    labels = torch.empty(X.shape[0], dtype=torch.int64, device=X.device)
    lib = _native.load_library()
    _native.check(lib.qadc_b200_assign(_native.dptr(X), X.shape[0], X.shape[1], _native.dptr(C),
                                       C.shape[0], _native.dptr(labels),
                                       torch.cuda.current_stream().cuda_stream), "assign")
    return labels


def build_flat(pq, base, layout: str = LAYOUT_STANDARD) -> IvfIndex:
    """Single-list index of whole-vector codes, encoded on the GPU."""
    import torch

    _check_layout(pq, layout)
    X = np.ascontiguousarray(np.asarray(getattr(base, "data", base), dtype=np.float32))
    if X.ndim != 2 or X.shape[1] != pq.m * pq.codebooks.shape[2]:
        raise ValueError("base dimension does not match the quantizer")
    packed = encode_device(pq, torch.from_numpy(X).cuda()).cpu().numpy()
    ids = np.arange(X.shape[0], dtype=np.int64)
    return IvfIndex(d=X.shape[1], m=pq.m, b=pq.b, coarse=None,
                    lists=[_make_list(packed, ids, layout)], layout=layout)


def build_with_coarse(pq, coarse, base, layout: str = LAYOUT_STANDARD) -> IvfIndex:
    """IVF index for given (reference-trained) coarse centroids: GPU
    assignment, residual encoding, lists with ids ascending (ivf.py:109-151)."""
    import torch

    _check_layout(pq, layout)
    cent = np.ascontiguousarray(getattr(coarse, "centroids", coarse), dtype=np.float32)
    X = torch.from_numpy(np.ascontiguousarray(np.asarray(getattr(base, "data", base),
                                                         dtype=np.float32))).cuda()
    labels = assign_device(cent, X)
    resid = X - torch.from_numpy(cent).cuda()[labels]
    packed = encode_device(pq, resid).cpu().numpy()
    lab = labels.cpu().numpy()
    order = np.argsort(lab, kind="stable")
    bounds = np.concatenate([[0], np.cumsum(np.bincount(lab, minlength=cent.shape[0]))])
    lists = [_make_list(packed[order[bounds[c]:bounds[c + 1]]],
                        order[bounds[c]:bounds[c + 1]].astype(np.int64), layout)
             for c in range(cent.shape[0])]
    return IvfIndex(d=cent.shape[1], m=pq.m, b=pq.b, coarse=Codebook(cent), lists=lists,
                    layout=layout)


# ---------------------------------------------------------------- QIVF v1 I/O

def save_index(index, path) -> None:
    """QIVF v1: magic, <IIIIIB (version, d, m, b, K, layout), coarse f32,
    then per list u64 n + i64 ids + codes in standard row order."""
    with open(path, "wb") as f:
        f.write(INDEX_MAGIC)
        f.write(struct.pack("<IIIIIB", INDEX_VERSION, index.d, index.m, index.b, index.K,
                            _LAYOUT_TAGS[index.layout]))
        if index.coarse is not None:
            f.write(np.ascontiguousarray(index.coarse.centroids, dtype="<f4").tobytes())
        for lst in index.lists:
            codes, ids = _canonical(lst)
            f.write(struct.pack("<Q", codes.shape[0]))
            f.write(np.ascontiguousarray(ids, dtype="<i8").tobytes())
            f.write(np.ascontiguousarray(codes, dtype=np.uint8).tobytes())


def load_index(path) -> IvfIndex:
    with open(path, "rb") as f:
        raw = f.read()
    head = struct.calcsize("<IIIIIB")
    if len(raw) < 4 + head or raw[:4] != INDEX_MAGIC:
        raise FormatError(f"{path}: not an index file")
    version, d, m, b, K, tag = struct.unpack_from("<IIIIIB", raw, 4)
    if version != INDEX_VERSION:
        raise FormatError(f"{path}: unsupported index version {version}")
    if tag not in _TAG_LAYOUTS:
        raise FormatError(f"{path}: unknown layout tag {tag}")
    try:
        rb = _row_bytes(m, b)
    except ValueError as e:
        raise FormatError(f"{path}: {e}") from None
    off = 4 + head
    coarse = None
    if K:
        need = 4 * K * d
        if len(raw) < off + need:
            raise FormatError(f"{path}: truncated coarse codebook")
        coarse = Codebook(np.frombuffer(raw, "<f4", K * d, off).reshape(K, d).copy())
        off += need
    lists = []
    for _ in range(K or 1):
        if len(raw) < off + 8:
            raise FormatError(f"{path}: truncated list header")
        (n,) = struct.unpack_from("<Q", raw, off)
        off += 8
        if len(raw) < off + (8 + rb) * n:
            raise FormatError(f"{path}: truncated list data")
        ids = np.frombuffer(raw, "<i8", n, off).copy()
        off += 8 * n
        codes = np.frombuffer(raw, np.uint8, rb * n, off).reshape(n, rb).copy()
        off += rb * n
        lists.append(_make_list(codes, ids, _TAG_LAYOUTS[tag]))
    if off != len(raw):
        raise FormatError(f"{path}: trailing bytes after last list")
    return IvfIndex(d=d, m=m, b=b, coarse=coarse, lists=lists, layout=_TAG_LAYOUTS[tag])
