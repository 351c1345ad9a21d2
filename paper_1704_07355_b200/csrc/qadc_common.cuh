// Shared device helpers for the B200 Quick ADC search path.
//
// Reference semantics (paths relative to /root/reference/pkg/src/qadc/):
//   * byte tables hold 0..127 (qadc.py:24, 124-147);
//   * lane distance = min(255, sum of table bytes) (scan_kernels.c:137-167;
//     saturating adds of non-negative values equal one final clamp);
//   * reported distance = fp32 qmin + ((float)q + 0.5f) * delta with two
//     roundings and no FMA (scan_kernels.c:294, _pykernels.py:86);
//   * admission order is lexicographic (distance, id) (scan_kernels.c:24-27).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace qadc {

constexpr int kMaxM = 128;        // QADC_MAX_M (scan_kernels.h:12)
constexpr int kChunkCodes = 256;  // codes per interleaved chunk (32 octets)
constexpr int kQuantBins = 127;   // QUANT_BINS (qadc.py:24)

// ---- bit-exact float helpers (no contraction) ----

// S7: qmin + ((float)q + 0.5f) * delta, product rounded before the add.
__device__ __forceinline__ float midpoint(float qmin, float delta, int q) {
  return __fadd_rn(qmin, __fmul_rn(__fadd_rn((float)q, 0.5f), delta));
}

// Largest t in [-1, 254] with midpoint(t) <= M (midpoint is monotone
// non-decreasing in t because delta >= 0). -1 means no lane can qualify.
// Saturated lanes (255) are never scan candidates, so the cap is 254.
// An estimate from the inverse of the midpoint formula is corrected by exact
// midpoint evaluations (usually 1-2): the result is the same as a binary
// search, at a fraction of the dependent instructions (this runs on the scan
// kernels' per-tile bound refresh).
__device__ __forceinline__ int q_threshold(float M, float qmin, float delta) {
  if (!(midpoint(qmin, delta, 0) <= M)) return -1;
  if (midpoint(qmin, delta, 254) <= M) return 254;
  // here delta > 0 and midpoint(0) <= M < midpoint(254)
  const float est = floorf(__fdiv_rn(M - qmin, delta) - 0.5f);
  int t = (est >= 0.f && est <= 253.f) ? (int)est : (est > 253.f ? 253 : 0);
  while (t < 253 && midpoint(qmin, delta, t + 1) <= M) t++;
  while (t > 0 && !(midpoint(qmin, delta, t) <= M)) t--;
  return t;
}

// (distance, id) strict order (scan_kernels.c:24-27).
__device__ __forceinline__ bool entry_less(float d1, int64_t i1, float d2, int64_t i2) {
  return d1 < d2 || (d1 == d2 && i1 < i2);
}

// Non-negative floats order like their bit patterns (all distances here
// are >= 0: squared distances, qmin >= 0, delta >= 0).
__device__ __forceinline__ unsigned fbits(float x) { return __float_as_uint(x); }

// ---- integer SIMD helpers (inline PTX keeps PRMT's full 4-bit selector;
// CUDA's __byte_perm masks it with 0x7777) ----

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}

// a * one + c on the FMA pipe (IMAD). `one` is a runtime 1 so ptxas cannot
// fold it into an ALU-pipe IADD3; this balances the LUT scan across the
// ALU (PRMT) and FMA (IMAD) pipes.
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t one, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(one), "r"(c));
  return d;
}

// ---- error codes shared with the C ABI ----
enum Status : int {
  kOk = 0,
  kErrArgs = 1,       // invalid argument (maps to ValueError in Python)
  kErrCuda = 2,       // CUDA runtime failure
  kErrCapacity = 3,   // internal candidate capacity exceeded (retried)
  kErrNoDevice = 4,   // no CUDA device
};

}  // namespace qadc
