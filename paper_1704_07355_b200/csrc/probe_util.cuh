// Device helpers shared by the probe kernels (lut.cu, probe_gemm.cu):
// NumPy's float32 einsum order and the warp-level exact u64 selection.
#pragma once

#include <cstdint>

namespace qadc {
namespace {

// NumPy float32 einsum("d,d->") of diff = a - b (adc.py:72-73,
// ivf.py:178-179): 4 lanes, product rounded then added (no FMA); blocks of
// 16 folded as v3, v2, v1, v0; tail in zero-padded 4-vectors; lanes reduce
// (l0 + l1) + (l2 + l3). Matches oracle/qadc_oracle.c orc_einsum_sqdist.
template <class FA>
__device__ __forceinline__ float einsum_sq(FA a, const float *__restrict__ b, int n) {
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  int i = 0;
  for (; n - i >= 16; i += 16) {
#pragma unroll
    for (int v = 3; v >= 0; v--) {
#pragma unroll
      for (int l = 0; l < 4; l++) {
        const float df = __fsub_rn(a(i + 4 * v + l), b[i + 4 * v + l]);
        acc[l] = __fadd_rn(acc[l], __fmul_rn(df, df));
      }
    }
  }
  for (; i < n; i += 4) {
#pragma unroll
    for (int l = 0; l < 4; l++) {
      float p = 0.f;
      if (i + l < n) {
        const float df = __fsub_rn(a(i + l), b[i + l]);
        p = __fmul_rn(df, df);
      }
      acc[l] = __fadd_rn(acc[l], p);
    }
  }
  return __fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3]));
}

// Warp-level exact selection of the ma smallest unique u64 keys: a running
// set `best` (sorted, nb <= ma) plus a candidate buffer; keys below the
// current ma-th best are appended; a full buffer is merged by a warp
// bitonic sort of (best U buffer) in shared memory.
constexpr int kSelBuf = 192;  // candidate slots per query (ma <= 64)

__device__ __forceinline__ void warp_sort_u64(uint64_t *v, int n_pow2) {
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= n_pow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < n_pow2; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = v[i], b = v[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) { v[i] = b; v[ixj] = a; }
        }
      }
      __syncwarp();
    }
  }
}

// Merge buffer entries into best (kept in v[0 .. nb)); v has room for
// ma + kSelBuf entries rounded up to a power of two.
__device__ __forceinline__ void warp_merge(uint64_t *v, int &nb, int &bn, int ma, uint64_t &T) {
  const int lane = threadIdx.x & 31;
  const int n = nb + bn;
  int p2 = 1;
  while (p2 < n) p2 <<= 1;
  for (int i = n + lane; i < p2; i += 32) v[i] = ~0ull;
  __syncwarp();
  warp_sort_u64(v, p2);
  nb = n < ma ? n : ma;
  bn = 0;
  T = nb == ma ? v[ma - 1] : ~0ull;
  __syncwarp();
}

}  // namespace
}  // namespace qadc
