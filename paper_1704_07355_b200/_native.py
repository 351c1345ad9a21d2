"""ctypes binding of the C-ABI library ``_lib/libqadc_b200.so``.

This is the same binding a maintainer would add to the reference (its
Cython layer, /root/reference/pkg/src/qadc/_kernels.pyx, binds the four
functions of src/scan_kernels.h; here they are bound with ctypes). There is
no CPU fallback: if the library is missing or no B200 is visible, every
entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_int64, c_uint, c_void_p
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("QADC_B200_LIB") or
                Path(__file__).resolve().parent / "_lib" / "libqadc_b200.so")

QADC_KERNEL_B200 = 3
MAX_M = 128
HOST_IO = 1
LUT_IN = 2
NO_FSAT = 4
SCAN_PRMT = 8  # force the PRMT (CUDA-core) scan kernel
SCAN_TC = 16  # force the int8 tensor-core scan kernel (m = 16, 32)
SCAN_TC1 = 32  # tensor-core scan of an exhaustive list on one SM per tile (not CTA pairs)
SCAN_TCW = 64  # IVF: warpgroup-pipelined tensor-core scan (<= 32 queries per pass over a list)

_lib = None

_u8p = POINTER(ctypes.c_uint8)
_i64p = POINTER(c_int64)
_f32p = POINTER(c_float)
_i32p = POINTER(ctypes.c_int32)
_f64p = POINTER(ctypes.c_double)


def _bind(lib):
    lib.qadc_simd_level.restype = c_int
    lib.qadc_simd_level.argtypes = []
    lib.qadc_b200_last_error.restype = c_char_p
    lib.adc_scan_f32.restype = c_int
    lib.adc_scan_f32.argtypes = [_u8p, c_int64, _i64p, c_int, c_int, _f32p, _f32p, _i64p,
                                 c_int, c_int]
    lib.qadc_scan_u8.restype = c_int
    lib.qadc_scan_u8.argtypes = [_u8p, c_int64, _i64p, c_int, _u8p, c_float, c_float, _f32p,
                                 _i64p, c_int, c_int, c_int]
    lib.qadc_block_dists.restype = None
    lib.qadc_block_dists.argtypes = [_u8p, c_int64, c_int, _u8p, c_int, _u8p, c_int]
    lib.qadc_b200_index_create.restype = c_int
    lib.qadc_b200_index_create.argtypes = [c_int, c_int, c_int, _f32p, _u8p, _i64p, _i64p, _i64p,
                                           _f32p, _f32p, POINTER(c_void_p)]
    lib.qadc_b200_index_create_device.restype = c_int
    lib.qadc_b200_index_create_device.argtypes = [c_int, c_int, c_int, c_void_p, c_void_p,
                                                  c_void_p, c_void_p, c_void_p, c_void_p,
                                                  POINTER(c_void_p)]
    lib.qadc_b200_index_destroy.restype = None
    lib.qadc_b200_index_destroy.argtypes = [c_void_p]
    lib.qadc_b200_index_bytes.restype = c_int64
    lib.qadc_b200_index_bytes.argtypes = [c_void_p]
    lib.qadc_b200_search_batch.restype = c_int
    lib.qadc_b200_search_batch.argtypes = [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_uint,
                                           c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                           c_void_p, _i64p]
    lib.qadc_b200_search_prepare.restype = c_int
    lib.qadc_b200_search_prepare.argtypes = [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_uint,
                                             c_void_p, c_void_p] + [c_void_p] * 10 + [c_void_p,
                                                                                      _i64p]
    lib.qadc_b200_search_scan.restype = c_int
    lib.qadc_b200_search_scan.argtypes = [c_void_p, c_int, c_int, c_int, c_int, c_uint] + [
        c_void_p] * 12 + [c_void_p, _i64p]
    lib.qadc_b200_search_tables.restype = c_int
    lib.qadc_b200_search_tables.argtypes = [c_void_p, c_void_p, c_int, c_int, c_int, c_int,
                                            c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                            c_void_p, c_void_p]
    lib.qadc_b200_compute_tables.restype = c_int
    lib.qadc_b200_compute_tables.argtypes = [c_void_p, c_int, c_int, c_void_p, c_int, c_void_p,
                                             c_void_p]
    lib.qadc_b200_probe.restype = c_int
    lib.qadc_b200_probe.argtypes = [c_void_p, c_int, c_int, c_void_p, c_int, c_int, c_void_p,
                                    c_void_p, c_void_p]
    lib.qadc_b200_quantize_tables.restype = c_int
    lib.qadc_b200_quantize_tables.argtypes = [c_void_p, c_int, c_int, c_void_p, c_void_p,
                                              c_void_p, c_void_p, c_void_p]
    lib.qadc_b200_encode.restype = c_int
    lib.qadc_b200_encode.argtypes = [c_void_p, c_int64, c_int, c_int, c_void_p, c_void_p,
                                     c_void_p, c_void_p]
    lib.qadc_b200_assign.restype = c_int
    lib.qadc_b200_assign.argtypes = [c_void_p, c_int64, c_int, c_void_p, c_int, c_void_p,
                                     c_void_p]
    lib.qadc_b200_index_set_prefix_device.restype = c_int
    lib.qadc_b200_index_set_prefix_device.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p,
                                                      _i64p]
    lib.qadc_b200_int_peak.restype = c_int
    lib.qadc_b200_int_peak.argtypes = [_f64p]
    lib.qadc_b200_mma_peak.restype = c_int
    lib.qadc_b200_mma_peak.argtypes = [_f64p]
    return lib


def load_library():
    """The loaded library (dlopen on first use). Raises if it is not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
        _lib = _bind(ctypes.CDLL(str(LIB_PATH)))
    return _lib


def library_available() -> bool:
    return LIB_PATH.exists()


def last_error() -> str:
    return load_library().qadc_b200_last_error().decode("utf-8", "replace")


def check(rc: int, what: str) -> None:
    """Map a C status to the reference's exception types (ValueError for
    bad arguments, RuntimeError otherwise; _kernels.pyx:38-46)."""
    if rc == 0:
        return
    msg = f"{what}: {last_error()}"
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def device_level() -> int:
    """QADC_KERNEL_B200 when a usable sm_100 device is present, else -1."""
    return int(load_library().qadc_simd_level())


def require_device() -> None:
    if device_level() != QADC_KERNEL_B200:
        raise RuntimeError(f"no usable B200 (sm_100) device: {last_error()}")


def ptr(a: np.ndarray, ctype):
    """ctypes pointer to a C-contiguous numpy array (None for empty)."""
    if a is None:
        return None
    return a.ctypes.data_as(POINTER(ctype))


def dptr(t) -> int | None:
    """Raw device pointer of a torch tensor (or None)."""
    return None if t is None else int(t.data_ptr())
