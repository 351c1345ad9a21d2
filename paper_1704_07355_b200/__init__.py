"""qadc-b200: the Quick ADC search path (arXiv 1704.07355) on NVIDIA B200.

A drop-in for the search API of the reference package `qadc`
(/root/reference/pkg): the same module and function names (`kernels`,
`qadc`, `adc`, `heap`, `ivf`), backed by hand-written sm_100a kernels in
libqadc_b200.so (C ABI: include/qadc_b200.h). There is no CPU fallback.
"""

from . import adc, heap, ivf, kernels, qadc  # noqa: F401
from .adc import (DEFAULT_INIT, LookupTables, PhaseTimings, SearchResult, compute_tables,
                  device_index, search, search_batch)
from .device import BatchResult, DeviceIndex
from .heap import NeighborHeap
from .ivf import IvfIndex, LAYOUT_STANDARD, LAYOUT_TRANSPOSED, build_flat, probe
from .qadc import (QuantizedTables, TransposedList, find_qmax, qadc_scan, quantize_tables,
                   transpose_list, untranspose_list)

__version__ = "0.1.0"

__all__ = [
    "BatchResult", "DEFAULT_INIT", "DeviceIndex", "IvfIndex", "LAYOUT_STANDARD",
    "LAYOUT_TRANSPOSED", "LookupTables", "NeighborHeap", "PhaseTimings", "QuantizedTables",
    "SearchResult", "TransposedList", "build_flat", "compute_tables", "device_index",
    "find_qmax", "probe", "qadc_scan", "quantize_tables", "search", "search_batch",
    "transpose_list", "untranspose_list",
]
