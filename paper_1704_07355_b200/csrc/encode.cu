// GPU index build: PQ encoding and coarse assignment straight
// into device memory, so billion-scale indexes never round-trip through
// host NumPy. Semantics follow the reference's offline build:
//   * kmeans.assign_batch broadcast path (kmeans.py:52-78, k*d <= 2^20):
//     squared distances by einsum("nkd,nkd->nk") of diff = x - c, argmin
//     with ties to the lowest index;
//   * pq.encode_batch (pq.py:210-217): optional rotation x @ R^T, then the
//     per-subspace argmin, packed two sub-codes per byte, low nibble =
//     even sub-code (pq.py:90-105).
// The rotation is a sequential fp32 FMA chain (the reference's X @ R^T is an
// OpenBLAS sgemm whose blocking is not reproduced; codes near a sub-space
// tie may differ — the index is an input, parity is given the index), and
// k*d > 2^20 coarse assignment uses the same einsum form instead of the
// reference's clamped GEMM expansion.
#include <algorithm>

#include "qadc_b200.h"
#include "internal.cuh"

namespace qadc {
namespace {

__device__ __forceinline__ float sqdist_einsum(const float *__restrict__ a, const float *__restrict__ b,
                                               int n) {
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  int i = 0;
  for (; n - i >= 16; i += 16) {
#pragma unroll
    for (int v = 3; v >= 0; v--) {
#pragma unroll
      for (int l = 0; l < 4; l++) {
        const float df = __fsub_rn(a[i + 4 * v + l], b[i + 4 * v + l]);
        acc[l] = __fadd_rn(acc[l], __fmul_rn(df, df));
      }
    }
  }
  for (; i < n; i += 4) {
#pragma unroll
    for (int l = 0; l < 4; l++) {
      float p = 0.f;
      if (i + l < n) {
        const float df = __fsub_rn(a[i + l], b[i + l]);
        p = __fmul_rn(df, df);
      }
      acc[l] = __fadd_rn(acc[l], p);
    }
  }
  return __fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3]));
}

// y = R x for a tile of 32 vectors per CTA (pq.py:210-217's X @ R^T; the
// reference's sgemm order is not reproduced: the index is an input and
// parity is defined given the index). R^T rows are read coalesced through
// L1 (thread i owns output i), the vectors are staged in shared memory and
// broadcast; each thread accumulates 16 vectors (sequential fp32 FMA).
constexpr int kRotTile = 32;
__global__ void __launch_bounds__(256) k_rotate(const float *__restrict__ X, int64_t n, int d,
                                                const float *__restrict__ RT,
                                                float *__restrict__ Y) {
  extern __shared__ float sx[];  // kRotTile * d
  const int64_t v0 = (int64_t)blockIdx.x * kRotTile;
  const int nv = (int)(n - v0 < kRotTile ? n - v0 : kRotTile);
  for (int t = threadIdx.x; t < nv * d; t += blockDim.x) sx[t] = X[v0 * d + t];
  for (int t = nv * d + threadIdx.x; t < kRotTile * d; t += blockDim.x) sx[t] = 0.f;
  __syncthreads();
  const int half = threadIdx.x >> 7;  // vectors half*16 .. half*16+15
  for (int i = threadIdx.x & 127; i < d; i += 128) {
    float acc[16];
#pragma unroll
    for (int v = 0; v < 16; v++) acc[v] = 0.f;
    const float *xs = sx + (size_t)half * 16 * d;
    for (int k = 0; k < d; k++) {
      const float r = __ldg(RT + (size_t)k * d + i);
#pragma unroll
      for (int v = 0; v < 16; v++) acc[v] = __fmaf_rn(r, xs[(size_t)v * d + k], acc[v]);
    }
#pragma unroll
    for (int v = 0; v < 16; v++) {
      const int vv = half * 16 + v;
      if (vv < nv) Y[(v0 + vv) * d + i] = acc[v];
    }
  }
}

__global__ void k_transpose_sq(const float *__restrict__ in, int d, float *__restrict__ out) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < d * d; t += gridDim.x * blockDim.x)
    out[(size_t)(t % d) * d + t / d] = in[t];
}

// PQ encoding of a tile of 32 vectors per CTA: the tile (rows padded to
// d + 1 words: conflict-free column reads) and the codebooks sit in shared
// memory; warp w takes sub-spaces w, w + 8, ..., lane = vector, so every
// codebook read is a warp-wide broadcast. Per sub-space: argmin over the 16
// centroids of the einsum-order squared distance (ties to the lowest
// index), then two sub-codes per byte, low nibble = even sub-code.
constexpr int kEncTile = 32;
__global__ void __launch_bounds__(256) k_encode(const float *__restrict__ X, int64_t n, int m,
                                                int dsub, const float *__restrict__ codebooks,
                                                uint8_t *__restrict__ out) {
  extern __shared__ float esm[];
  const int d = m * dsub, dp = d + 1;
  float *sx = esm;                                  // [kEncTile][d + 1]
  float *scb = sx + (size_t)kEncTile * dp;          // [m][16][dsub]
  uint8_t *sc = (uint8_t *)(scb + (size_t)m * 16 * dsub);  // [kEncTile][m]
  const int64_t v0 = (int64_t)blockIdx.x * kEncTile;
  const int nv = (int)(n - v0 < kEncTile ? n - v0 : kEncTile);
  for (int t = threadIdx.x; t < m * 16 * dsub; t += blockDim.x) scb[t] = codebooks[t];
  for (int t = threadIdx.x; t < nv * d; t += blockDim.x) {
    const int v = t / d, c = t - v * d;
    sx[v * dp + c] = X[v0 * d + t];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane < nv) {
    for (int j = w; j < m; j += 8) {
      const float *x = sx + (size_t)lane * dp + (size_t)j * dsub;
      int best = 0;
      float bd = 0.f;
      for (int i = 0; i < 16; i++) {
        const float dd = sqdist_einsum(x, scb + ((size_t)j * 16 + i) * dsub, dsub);
        if (i == 0 || dd < bd) {
          bd = dd;
          best = i;
        }
      }
      sc[lane * m + j] = (uint8_t)best;
    }
  }
  __syncthreads();
  const int mrows = m / 2;
  for (int t = threadIdx.x; t < nv * mrows; t += blockDim.x) {
    const int v = t / mrows, b = t - v * mrows;
    out[(v0 + v) * mrows + b] = (uint8_t)(sc[v * m + 2 * b] | (sc[v * m + 2 * b + 1] << 4));
  }
}

// Coarse assignment: 128 vectors per CTA staged in shared memory; every
// thread walks all K centroids (rows read as warp-wide broadcasts).
__global__ void __launch_bounds__(128) k_assign(const float *__restrict__ X, int64_t n, int d,
                                                const float *__restrict__ C, int K,
                                                int64_t *__restrict__ labels) {
  extern __shared__ float sx[];  // 128 * d, row-major per vector
  const int64_t v0 = (int64_t)blockIdx.x * 128;
  const int nv = (int)(n - v0 < 128 ? n - v0 : 128);
  for (int t = threadIdx.x; t < nv * d; t += blockDim.x) sx[t] = X[v0 * d + t];
  __syncthreads();
  if ((int)threadIdx.x >= nv) return;
  const float *x = sx + (size_t)threadIdx.x * d;
  int best = 0;
  float bd = 0.f;
  for (int k = 0; k < K; k++) {
    // centroid first, query second: diff = x - c has the same magnitude
    const float dd = sqdist_einsum(x, C + (size_t)k * d, d);
    if (k == 0 || dd < bd) {
      bd = dd;
      best = k;
    }
  }
  labels[v0 + threadIdx.x] = best;
}

}  // namespace
}  // namespace qadc

using namespace qadc;

extern "C" int qadc_b200_encode(const float *X, int64_t n, int d, int m, const float *codebooks,
                                const float *rotation, uint8_t *out, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  set_error("");
  if (m < 2 || m % 2 || d % m || m > QADC_MAX_M || n < 0) {
    set_error("invalid encode geometry");
    return kErrArgs;
  }
  if (n == 0) return kOk;
  const float *src = X;
  float *rot = nullptr, *rt = nullptr;
  if (rotation) {
    QADC_CUDA(cudaMallocAsync(&rot, (size_t)n * d * 4, st));
    QADC_CUDA(cudaMallocAsync(&rt, (size_t)d * d * 4, st));
    k_transpose_sq<<<(d * d + 255) / 256, 256, 0, st>>>(rotation, d, rt);
    const size_t smem = (size_t)kRotTile * d * 4;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_rotate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_rotate<<<(unsigned)((n + kRotTile - 1) / kRotTile), 256, smem, st>>>(X, n, d, rt, rot);
    src = rot;
  }
  const size_t esmem = ((size_t)kEncTile * (d + 1) + (size_t)m * 16 * (d / m)) * 4 +
                       (size_t)kEncTile * m;
  if (esmem > 227 * 1024) {
    set_error("encode: d too large for the shared-memory tile");
    return kErrArgs;
  }
  if (esmem > 48 * 1024)
    cudaFuncSetAttribute(k_encode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esmem);
  k_encode<<<(unsigned)((n + kEncTile - 1) / kEncTile), 256, esmem, st>>>(src, n, m, d / m,
                                                                        codebooks, out);
  if (rot) cudaFreeAsync(rot, st);
  if (rt) cudaFreeAsync(rt, st);
  QADC_CUDA(cudaGetLastError());
  return kOk;
}

extern "C" int qadc_b200_assign(const float *X, int64_t n, int d, const float *C, int K,
                                int64_t *labels, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  set_error("");
  if (d < 1 || K < 1 || n < 0) {
    set_error("invalid assign geometry");
    return kErrArgs;
  }
  if (n == 0) return kOk;
  // the fused tensor-core nearest-centroid search (probe_tc.cu, ma = 1):
  // same result (exact einsum-order re-rank, ties to the lower index)
  if (probe_tc_supported(K, d, 1)) {
    float *mu = nullptr, *cn2 = nullptr;
    void *cs = nullptr;
    bool done = false;
    if (probe_tc_prepare(C, K, d, &mu, &cs, &cn2, st) == kOk) {
      done = true;
      for (int64_t v0 = 0; v0 < n && done; v0 += (1 << 30)) {
        const int nv = (int)std::min<int64_t>(n - v0, 1 << 30);
        done = launch_probe_tc(C, mu, cs, cn2, K, d, X + (size_t)v0 * d, nv, 1, labels + v0, st);
      }
    }
    cudaFreeAsync(mu, st);
    cudaFreeAsync(cs, st);
    cudaFreeAsync(cn2, st);
    if (done) {
      QADC_CUDA(cudaGetLastError());
      return kOk;
    }
  }
  const size_t smem = (size_t)128 * d * 4;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_assign<<<(unsigned)((n + 127) / 128), 128, smem, st>>>(X, n, d, C, K, labels);
  QADC_CUDA(cudaGetLastError());
  return kOk;
}
