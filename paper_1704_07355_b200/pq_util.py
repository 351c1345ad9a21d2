"""4-bit code packing (host byte layout, /root/reference/pkg/src/qadc/pq.py:90-122):
two sub-codes per byte, low nibble = even sub-code."""

from __future__ import annotations

import numpy as np


def pack_codes(codes: np.ndarray, b: int = 4) -> np.ndarray:
    """(n, m) sub-indices -> (n, m/2) bytes for b = 4."""
    codes = np.ascontiguousarray(codes)
    if b != 4:
        raise ValueError("the B200 path packs 4-bit codes only")
    if codes.shape[1] % 2:
        raise ValueError("4-bit packing pairs sub-indices; m must be even")
    return np.ascontiguousarray((codes[:, 0::2] & 15).astype(np.uint8)
                                | ((codes[:, 1::2] & 15).astype(np.uint8) << 4))


def unpack_codes(packed: np.ndarray, m: int) -> np.ndarray:
    """(n, m/2) bytes -> (n, m) uint16 sub-indices."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    if packed.shape[1] * 2 != m:
        raise ValueError(f"packed width {packed.shape[1]} does not match m={m}")
    out = np.empty((packed.shape[0], m), dtype=np.uint16)
    out[:, 0::2] = packed & 15
    out[:, 1::2] = packed >> 4
    return out
