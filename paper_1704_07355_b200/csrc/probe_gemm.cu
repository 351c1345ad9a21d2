// Tensor-core coarse probe (ivf.py:166-182): the Q x K dot
// products go through ONE cuBLAS bf16 GEMM on the tcgen05 tensor cores, the
// exact NumPy-einsum-order distance is computed only for the cells that can
// still reach a query's top ma.
//
//   * centring: q' = q - mu, c' = c - mu (mu = centroid mean) leaves every
//     squared distance unchanged and shrinks |q'| |c'|, hence the bound;
//   * split bf16: v = hi + lo (hi = bf16(v), lo = bf16(v - hi)); one GEMM
//     with k = 3d over rows [q_hi | q_hi | q_lo] . [c_hi | c_lo | c_hi]
//     gives q'.c' up to the dropped lo*lo term and the remainders
//     (<= 3.1 * 2^-18 |q'| |c'|) plus the fp32 accumulation error
//     (<= 3d u sum|terms|, u = 2^-24), all products exact in fp32;
//   * bounds: A = fl(|q'|^2 + |c'|^2 - 2 S) and
//       |A - D| <= mg = eps (|q'|^2 + |c'|^2),
//       eps = 2^-15 + 4 (3d) u + 16 u    (D: exact squared distance)
//     and the einsum value E the reference ranks by satisfies
//     |E - D| <= (d + 4) u D, so E lies in [L, U] with
//       U = (A + mg)(1 + g),  L = max(0, (A - mg)(1 - g)),  g = (d + 4) u
//     computed with directed rounding;
//   * selection: U* = the ma-th smallest (U, cell); every cell of the true
//     top ma by (E, cell) has L <= E <= U*, so the exact einsum distance is
//     computed for {L <= U*} only (<= kGemmCand per query, else the exact
//     scan of all K cells) and sorted by (E, cell) — bit-identical to
//     np.lexsort((cells, d2))[:ma] of the einsum distances.
#include <cublas_v2.h>
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.cuh"
#include "probe_util.cuh"

namespace qadc {
namespace {

constexpr int kGemmQ = 8;       // queries (warps) per selection CTA
constexpr int kGemmCand = 512;  // exact re-rank candidates per query

// Index side: centroid mean (fp64 accumulation), centred split-bf16 rows,
// |c'|^2.
__global__ void k_coarse_mean(const float *__restrict__ C, int K, int d, float *__restrict__ mu) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d) return;
  double s = 0.0;
  for (int k = 0; k < K; k++) s += (double)C[(size_t)k * d + t];
  mu[t] = (float)(s / K);
}

__device__ __forceinline__ void split_row(const float *__restrict__ v, const float *__restrict__ mu,
                                          int d, bool coarse_side, __nv_bfloat16 *__restrict__ out,
                                          float *__restrict__ n2) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int t = lane; t < d; t += 32) {
    const float x = __fsub_rn(v[t], mu[t]);
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    const __nv_bfloat16 lo = __float2bfloat16_rn(__fsub_rn(x, __bfloat162float(hi)));
    // coarse rows [hi | lo | hi], query rows [hi | hi | lo]
    out[t] = hi;
    out[d + t] = coarse_side ? lo : hi;
    out[2 * d + t] = coarse_side ? hi : lo;
    acc += (double)x * (double)x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) *n2 = (float)acc;
}

__global__ void k_split_rows(const float *__restrict__ V, int n, int d, const float *__restrict__ mu,
                             bool coarse_side, __nv_bfloat16 *__restrict__ out, float *__restrict__ n2) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n) return;
  split_row(V + (size_t)w * d, mu, d, coarse_side, out + (size_t)w * 3 * d, n2 + w);
}

// Per query (one warp): pass 1 keeps the ma smallest (U, cell) keys, pass 2
// gathers the cells with L <= U* and ranks them by the exact einsum value.
__global__ void __launch_bounds__(kGemmQ * 32) k_probe_select(
    const float *__restrict__ S, const float *__restrict__ qn2, const float *__restrict__ cn2,
    const float *__restrict__ coarse, const float *__restrict__ queries, int K, int d, int nq,
    int ma, int vcap, float eps, float gam, int64_t *__restrict__ cells) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t *v = (uint64_t *)smem + (size_t)w * vcap;                              // selection
  uint64_t *cq = (uint64_t *)smem + (size_t)kGemmQ * vcap + (size_t)w * kGemmCand;  // candidates
  float *sq = (float *)((uint64_t *)smem + (size_t)kGemmQ * (vcap + kGemmCand)) + (size_t)w * d;
  const int q = blockIdx.x * kGemmQ + w;
  if (q >= nq) return;
  for (int t = lane; t < d; t += 32) sq[t] = queries[(size_t)q * d + t];
  __syncwarp();
  const float *Sq = S + (size_t)q * K;
  const float a2 = qn2[q];
  const float onep = __fadd_ru(1.f, gam), onem = __fsub_rd(1.f, gam);
  int nb = 0, bn = 0;
  uint64_t T = ~0ull;
  // 8 rows of 32 cells per step: eight independent loads in flight per lane
  // (the S rows stream from HBM; one dependent load per step would leave the
  // kernel latency bound)
  for (int i0 = 0; i0 < K; i0 += 256) {
    float sv[8], cv[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int k = i0 + 32 * u + lane;
      sv[u] = k < K ? __ldcs(Sq + k) : 0.f;
      cv[u] = k < K ? cn2[k] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int k = i0 + 32 * u + lane;
      uint64_t key = ~0ull;
      if (k < K) {
        const float n2 = __fadd_ru(a2, cv[u]);
        const float A = __fmaf_rn(-2.f, sv[u], __fadd_rn(a2, cv[u]));
        const float mg = __fmul_ru(eps, n2);
        const float U = fmaxf(__fmul_ru(__fadd_ru(A, mg), onep), 0.f);
        key = ((uint64_t)__float_as_uint(U) << 32) | (uint32_t)k;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, key < T);
      if (bal) {
        if (bn + __popc(bal) > kSelBuf) warp_merge(v, nb, bn, ma, T);
        const bool take = key < T;
        const unsigned bal2 = __ballot_sync(0xffffffffu, take);
        if (take) v[nb + bn + __popc(bal2 & ((1u << lane) - 1))] = key;
        bn += __popc(bal2);
        __syncwarp();
      }
    }
  }
  warp_merge(v, nb, bn, ma, T);
  const float Ustar = __uint_as_float((uint32_t)(v[min(ma, K) - 1] >> 32));
  int nc = 0;
  bool overflow = false;
  for (int i0 = 0; i0 < K && !overflow; i0 += 256) {
    float sv[8], cv[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int k = i0 + 32 * u + lane;
      sv[u] = k < K ? __ldcs(Sq + k) : 0.f;
      cv[u] = k < K ? cn2[k] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int k = i0 + 32 * u + lane;
      bool take = false;
      if (k < K) {
        const float n2 = __fadd_ru(a2, cv[u]);
        const float A = __fmaf_rn(-2.f, sv[u], __fadd_rn(a2, cv[u]));
        const float mg = __fmul_ru(eps, n2);
        const float L = fmaxf(__fmul_rd(__fsub_rd(A, mg), onem), 0.f);
        take = L <= Ustar;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, take);
      if (nc + __popc(bal) > kGemmCand) {
        overflow = true;
        break;
      }
      if (take) cq[nc + __popc(bal & ((1u << lane) - 1))] = (uint64_t)k;
      nc += __popc(bal);
    }
  }
  __syncwarp();
  if (!overflow) {
    for (int i = lane; i < nc; i += 32) {
      const int k = (int)cq[i];
      const float *crow = coarse + (size_t)k * d;
      const float E = einsum_sq([&](int t) { return crow[t]; }, sq, d);
      cq[i] = ((uint64_t)__float_as_uint(E) << 32) | (uint32_t)k;
    }
    __syncwarp();
    int p2 = 1;
    while (p2 < nc) p2 <<= 1;
    for (int i = nc + lane; i < p2; i += 32) cq[i] = ~0ull;
    __syncwarp();
    warp_sort_u64(cq, p2);
    for (int i = lane; i < ma; i += 32)
      cells[(size_t)q * ma + i] = i < nc ? (int64_t)(cq[i] & 0xffffffffu) : -1;
    return;
  }
  // overflow (massive near-ties): exact einsum of every cell
  nb = 0;
  bn = 0;
  T = ~0ull;
  for (int i0 = 0; i0 < K; i0 += 32) {
    const int k = i0 + lane;
    uint64_t key = ~0ull;
    if (k < K) {
      const float *crow = coarse + (size_t)k * d;
      const float E = einsum_sq([&](int t) { return crow[t]; }, sq, d);
      key = ((uint64_t)__float_as_uint(E) << 32) | (uint32_t)k;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, key < T);
    if (bal) {
      if (bn + __popc(bal) > kSelBuf) warp_merge(v, nb, bn, ma, T);
      const bool take = key < T;
      const unsigned bal2 = __ballot_sync(0xffffffffu, take);
      if (take) v[nb + bn + __popc(bal2 & ((1u << lane) - 1))] = key;
      bn += __popc(bal2);
      __syncwarp();
    }
  }
  warp_merge(v, nb, bn, ma, T);
  for (int i = lane; i < ma; i += 32) cells[(size_t)q * ma + i] = (int64_t)(v[i] & 0xffffffffu);
}

cublasHandle_t blas_handle() {
  static cublasHandle_t h[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!h[dev] && cublasCreate(&h[dev]) != CUBLAS_STATUS_SUCCESS) h[dev] = nullptr;
  return h[dev];
}

}  // namespace

bool probe_gemm_supported(int K, int d) { return K >= 256 && d % 8 == 0 && d <= 4096; }

int probe_gemm_prepare(const float *coarse, int K, int d, float **mu, void **csplit, float **cn2,
                       cudaStream_t st) {
  QADC_CUDA(cudaMalloc(mu, (size_t)d * 4));
  QADC_CUDA(cudaMalloc(csplit, (size_t)K * 3 * d * sizeof(__nv_bfloat16)));
  QADC_CUDA(cudaMalloc(cn2, (size_t)K * 4));
  k_coarse_mean<<<(d + 127) / 128, 128, 0, st>>>(coarse, K, d, *mu);
  k_split_rows<<<(K * 32 + 255) / 256, 256, 0, st>>>(coarse, K, d, *mu, true,
                                                     (__nv_bfloat16 *)*csplit, *cn2);
  QADC_CUDA(cudaGetLastError());
  return kOk;
}

bool launch_probe_gemm(const float *coarse, const float *mu, const void *csplit, const float *cn2,
                       int K, int d, const float *queries, int nq, int ma, int64_t *cells,
                       cudaStream_t st) {
  if (nq <= 0) return true;
  if (!probe_gemm_supported(K, d) || ma > K || ma > 256) return false;
  cublasHandle_t h = blas_handle();
  if (!h) return false;
  int vcap = 1;
  while (vcap < ma + kSelBuf) vcap <<= 1;
  const size_t smem = (size_t)kGemmQ * (vcap + kGemmCand) * 8 + (size_t)kGemmQ * d * 4;
  if (smem > 220 * 1024) return false;
  cudaFuncSetAttribute(k_probe_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // query chunks: the dot-product block stays <= 2^28 floats (1 GiB)
  const int chunk = std::max(kGemmQ, std::min(nq, (int)(((int64_t)1 << 28) / K) / kGemmQ * kGemmQ));
  __nv_bfloat16 *qs = nullptr;
  float *qn2 = nullptr, *S = nullptr;
  if (cudaMallocAsync(&qs, (size_t)chunk * 3 * d * sizeof(__nv_bfloat16), st) != cudaSuccess ||
      cudaMallocAsync(&qn2, (size_t)chunk * 4, st) != cudaSuccess ||
      cudaMallocAsync(&S, (size_t)chunk * K * 4, st) != cudaSuccess)
    return false;
  const double u = 1.0 / 16777216.0;
  const float eps = (float)(1.0 / 32768.0 + (4.0 * 3 * d + 16.0) * u);
  const float gam = (float)((d + 4) * u);
  cublasSetStream(h, st);
  bool ok = true;
  for (int q0 = 0; q0 < nq && ok; q0 += chunk) {
    const int n = std::min(chunk, nq - q0);
    k_split_rows<<<(n * 32 + 255) / 256, 256, 0, st>>>(queries + (size_t)q0 * d, n, d, mu, false,
                                                       qs, qn2);
    const float one = 1.f, zero = 0.f;
    // S (n x K, row-major) = Qs (n x 3d) . Cs (K x 3d)^T: column-major
    // K x n = op(Cs^T) . Qs^T
    ok = cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, K, n, 3 * d, &one, csplit, CUDA_R_16BF, 3 * d,
                      qs, CUDA_R_16BF, 3 * d, &zero, S, CUDA_R_32F, K, CUBLAS_COMPUTE_32F,
                      CUBLAS_GEMM_DEFAULT) == CUBLAS_STATUS_SUCCESS;
    if (!ok) break;
    k_probe_select<<<(n + kGemmQ - 1) / kGemmQ, kGemmQ * 32, smem, st>>>(
        S, qn2, cn2, coarse, queries + (size_t)q0 * d, K, d, n, ma, vcap, eps, gam,
        cells + (size_t)q0 * ma);
  }
  cudaFreeAsync(qs, st);
  cudaFreeAsync(qn2, st);
  cudaFreeAsync(S, st);
  if (!ok) set_error("cuBLAS GEMM of the coarse probe failed");
  return ok;
}

}  // namespace qadc
