// Index + Tables phases of adc.py:114-187 (qadc branch), batched over
// queries: coarse probe, residual, rotation, float LUT, qmax, quantized
// LUT, and the per-query prefix facts (first-R-valid saturated lanes and
// the initial distance bound). Paths relative to /root/reference/pkg/src/qadc/.
#include <cfloat>

#include "internal.cuh"
#include "probe_util.cuh"

namespace qadc {
namespace {

// NumPy float32 pairwise sum for n <= 128 (find_qmax empty-cell bound,
// qadc.py:192-193).
__device__ float pairwise_sum(const float *x, int n) {
  if (n < 8) {
    float r = 0.f;
    for (int i = 0; i < n; i++) r = __fadd_rn(r, x[i]);
    return r;
  }
  float r[8];
  for (int j = 0; j < 8; j++) r[j] = x[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; j++) r[j] = __fadd_rn(r[j], x[i + j]);
  float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                        __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
  for (; i < n; i++) res = __fadd_rn(res, x[i]);
  return res;
}

// Nibble j of list-local code k in the interleaved32 layout.
__device__ __forceinline__ int code_nibble(const uint32_t *__restrict__ codes, int m,
                                           int64_t chunk0, int64_t k, int j) {
  const int64_t g = chunk0 + k / kChunkCodes;
  const int o = (int)((k % kChunkCodes) >> 3);
  const uint32_t w = codes[(g * m + j) * 32 + o];
  return (w >> (4 * (k & 7))) & 15;
}

// ---------------- compute_tables (adc.py:61-75) ----------------
__global__ void k_tables(const float *__restrict__ codebooks, int m, int dsub,
                         const float *__restrict__ y, float *__restrict__ out) {
  extern __shared__ float sy[];
  const int d = m * dsub;
  const float *yp = y + (size_t)blockIdx.x * d;
  for (int t = threadIdx.x; t < d; t += blockDim.x) sy[t] = yp[t];
  __syncthreads();
  for (int e = threadIdx.x; e < m * 16; e += blockDim.x) {
    const int j = e >> 4;
    const float *cb = codebooks + (size_t)e * dsub;
    out[(size_t)blockIdx.x * m * 16 + e] =
        einsum_sq([&](int t) { return cb[t]; }, sy + (size_t)j * dsub, dsub);
  }
}

// ---------------- probe (ivf.py:166-182) ----------------
// kProbeQ queries per CTA share every centroid load (coalesced reads of the
// transposed centroid array, reused from registers for all queries of the
// CTA). Coarse distances follow NumPy's einsum order exactly; keys are
// (d2 bits << 32 | cell), so lexsort((cell, d2)) order is plain u64 order
// (d2 >= 0). Per tile of cells, one warp per query keeps the ma smallest
// keys: keys below the running ma-th best are buffered and merged by a warp
// bitonic sort (exact; the running threshold only discards keys that
// already have ma smaller ones).
constexpr int kProbeQ = 8;
constexpr int kProbeTile = 2048;
constexpr int kBoundPrefix = 16384;

__global__ void __launch_bounds__(256) k_probe(const float *__restrict__ coarseT, int K, int d,
                                               const float *__restrict__ queries, int nq, int ma,
                                               int tile, int vcap, int64_t *__restrict__ cells) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t *keys = (uint64_t *)smem;                        // [kProbeQ][tile]
  uint64_t *sel = keys + (size_t)kProbeQ * tile;            // [kProbeQ][vcap]: best | buffer
  float *sq = (float *)(sel + (size_t)kProbeQ * vcap);      // [kProbeQ][d]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int q0 = blockIdx.x * kProbeQ;
  const int nqb = min(kProbeQ, nq - q0);
  for (int e = threadIdx.x; e < kProbeQ * d; e += blockDim.x) {
    const int q = e / d;
    sq[e] = q < nqb ? queries[(size_t)(q0 + q) * d + (e - q * d)] : 0.f;
  }
  int nb = 0, bn = 0;  // warp w's selection state (query w)
  uint64_t T = ~0ull;
  __syncthreads();
  for (int base = 0; base < K; base += tile) {
    const int n = min(tile, K - base);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int k = base + i;
      float acc[kProbeQ][4];
#pragma unroll
      for (int q = 0; q < kProbeQ; q++) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.f;
      // einsum order (see einsum_sq): blocks of 16 as v3..v0, tail in 4s
      int t0 = 0;
      for (; d - t0 >= 16; t0 += 16) {
#pragma unroll
        for (int v = 3; v >= 0; v--) {
#pragma unroll
          for (int l = 0; l < 4; l++) {
            const int t = t0 + 4 * v + l;
            const float c = coarseT[(size_t)t * K + k];
#pragma unroll
            for (int q = 0; q < kProbeQ; q++) {
              const float df = __fsub_rn(c, sq[q * d + t]);
              acc[q][l] = __fadd_rn(acc[q][l], __fmul_rn(df, df));
            }
          }
        }
      }
      for (; t0 < d; t0 += 4) {
#pragma unroll
        for (int l = 0; l < 4; l++) {
          const int t = t0 + l;
          const float c = t < d ? coarseT[(size_t)t * K + k] : 0.f;
#pragma unroll
          for (int q = 0; q < kProbeQ; q++) {
            float pr = 0.f;
            if (t < d) {
              const float df = __fsub_rn(c, sq[q * d + t]);
              pr = __fmul_rn(df, df);
            }
            acc[q][l] = __fadd_rn(acc[q][l], pr);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kProbeQ; q++) {
        const float d2 = __fadd_rn(__fadd_rn(acc[q][0], acc[q][1]), __fadd_rn(acc[q][2], acc[q][3]));
        keys[(size_t)q * tile + i] = ((uint64_t)__float_as_uint(d2) << 32) | (uint32_t)k;
      }
    }
    __syncthreads();
    if (w < nqb) {  // warp w selects for query w
      const uint64_t *kq = keys + (size_t)w * tile;
      uint64_t *v = sel + (size_t)w * vcap;
      for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        const uint64_t key = i < n ? kq[i] : ~0ull;
        const bool take = key < T;
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        if (bal) {
          if (bn + __popc(bal) > kSelBuf) warp_merge(v, nb, bn, ma, T);
          const bool take2 = key < T;
          const unsigned bal2 = __ballot_sync(0xffffffffu, take2);
          if (take2) v[nb + bn + __popc(bal2 & ((1u << lane) - 1))] = key;
          bn += __popc(bal2);
          __syncwarp();
        }
      }
    }
    __syncthreads();
  }
  if (w < nqb) {
    uint64_t *v = sel + (size_t)w * vcap;
    warp_merge(v, nb, bn, ma, T);
    for (int i = lane; i < ma; i += 32) cells[(size_t)(q0 + w) * ma + i] = (int64_t)(v[i] & 0xffffffffu);
  }
}

// ---------------- fast probe: FFMA pre-selection + exact re-rank ----------------
// The exact order needs einsum-order d2 only for cells that can reach the
// top ma. Pass 1 bounds every cell's einsum d2 from an FFMA dot product:
//   A = fl(|c|^2 - 2 q.c),  |A + |q|^2 - D| <= (d u + 4u)(|q|^2 + |c|^2)
//   |E - D| <= (d/2 + 12) u (|q|^2 + |c|^2)     (E: einsum fp32, D: exact)
// with u = 2^-24; the margin (2.5 d + 200) u (|q|^2 + |c|^2) covers both,
// so E lies in [L, U] = A + |q|^2 -/+ margin for every cell. With U* the
// ma-th smallest U, every cell of the true top ma has L <= E <= U*, and
// pass 2 recomputes the exact einsum d2 only for cells with L <= U*, then
// selects exactly by (d2, cell). A candidate overflow falls back to the
// exact scan of all cells for that query.
constexpr int kFastQ = 8;
constexpr int kFastTile = 1024;  // 256 threads x 4 cells
constexpr int kCandCap = 512;

__global__ void k_cnorm(const float *__restrict__ coarse, int K, int d, float *__restrict__ cn) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int t = 0; t < d; t++) {
      const double v = coarse[(size_t)k * d + t];
      acc += v * v;
    }
    cn[k] = (float)acc;
  }
}

__global__ void __launch_bounds__(256) k_probe_fast(
    const float *__restrict__ coarseT, const float *__restrict__ coarse,
    const float *__restrict__ cn, int K, int d, const float *__restrict__ queries, int nq, int ma,
    int vcap, float *__restrict__ Lbuf, int64_t *__restrict__ cells) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t *sel = (uint64_t *)smem;                             // [kFastQ][vcap]
  float *ub = (float *)(sel + (size_t)kFastQ * vcap);           // [kFastQ][kFastTile] U
  float *sqT = ub + (size_t)kFastQ * kFastTile;                 // [d][kFastQ]
  __shared__ float s_qn[kFastQ];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int q0 = blockIdx.x * kFastQ;
  const int nqb = min(kFastQ, nq - q0);
  for (int e = threadIdx.x; e < kFastQ * d; e += blockDim.x) {
    const int t = e / kFastQ, q = e - t * kFastQ;
    sqT[e] = q < nqb ? queries[(size_t)(q0 + q) * d + t] : 0.f;
  }
  __syncthreads();
  if (threadIdx.x < kFastQ) {
    double acc = 0.0;
    for (int t = 0; t < d; t++) {
      const double v = sqT[t * kFastQ + threadIdx.x];
      acc += v * v;
    }
    s_qn[threadIdx.x] = (float)acc;
  }
  __syncthreads();
  const double mu = (2.5 * d + 200.0) * 5.9604644775390625e-08;  // margin factor
  int nb = 0, bn = 0;
  uint64_t T = ~0ull;
  for (int base = 0; base < K; base += kFastTile) {
    const int k0 = base + 4 * threadIdx.x;
    float acc[4][kFastQ];
#pragma unroll
    for (int c = 0; c < 4; c++)
#pragma unroll
      for (int q = 0; q < kFastQ; q++) acc[c][q] = 0.f;
    if (k0 < K) {
      const bool vec = (k0 + 3 < K) && ((K & 3) == 0);
#pragma unroll 4
      for (int t = 0; t < d; t++) {
        float cv[4];
        if (vec) {
          const float4 c4 = *(const float4 *)(coarseT + (size_t)t * K + k0);
          cv[0] = c4.x; cv[1] = c4.y; cv[2] = c4.z; cv[3] = c4.w;
        } else {
#pragma unroll
          for (int c = 0; c < 4; c++) cv[c] = k0 + c < K ? coarseT[(size_t)t * K + k0 + c] : 0.f;
        }
        const float4 qa = *(const float4 *)(sqT + t * kFastQ);
        const float4 qb = *(const float4 *)(sqT + t * kFastQ + 4);
        const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
        for (int c = 0; c < 4; c++)
#pragma unroll
          for (int q = 0; q < kFastQ; q++) acc[c][q] = __fmaf_rn(cv[c], qv[q], acc[c][q]);
      }
    }
#pragma unroll
    for (int c = 0; c < 4; c++) {
      const int k = k0 + c;
      const int slot = 4 * threadIdx.x + c;
      const float cnk = k < K ? cn[k] : 0.f;
#pragma unroll
      for (int q = 0; q < kFastQ; q++) {
        float Uk = __int_as_float(0x7f800000);
        if (k < K && q < nqb) {
          const float A = __fmaf_rn(-2.f, acc[c][q], cnk);
          const double base_d = (double)A + (double)s_qn[q];
          const double mg = mu * ((double)s_qn[q] + (double)cnk);
          const float U = __double2float_ru(base_d + mg);
          const float L = fmaxf(__double2float_rd(base_d - mg), 0.f);
          Uk = fmaxf(U, 0.f);
          Lbuf[(size_t)(q0 + q) * K + k] = L;
        }
        ub[(size_t)q * kFastTile + slot] = Uk;
      }
    }
    __syncthreads();
    if (w < nqb) {
      const float *uq = ub + (size_t)w * kFastTile;
      uint64_t *v = sel + (size_t)w * vcap;
      for (int i0 = 0; i0 < kFastTile && base + i0 < K; i0 += 32) {
        const int k = base + i0 + lane;
        const uint64_t key = k < K ? ((uint64_t)__float_as_uint(uq[i0 + lane]) << 32) | (uint32_t)k
                                   : ~0ull;
        const unsigned bal = __ballot_sync(0xffffffffu, key < T);
        if (bal) {
          if (bn + __popc(bal) > kSelBuf) warp_merge(v, nb, bn, ma, T);
          const bool take2 = key < T;
          const unsigned bal2 = __ballot_sync(0xffffffffu, take2);
          if (take2) v[nb + bn + __popc(bal2 & ((1u << lane) - 1))] = key;
          bn += __popc(bal2);
          __syncwarp();
        }
      }
    }
    __syncthreads();
  }
  __threadfence_block();
  if (w >= nqb) return;
  uint64_t *v = sel + (size_t)w * vcap;
  warp_merge(v, nb, bn, ma, T);
  const float Ustar = __uint_as_float((uint32_t)(v[ma - 1] >> 32));
  // pass 2: candidates with L <= U* (reads this CTA's own Lbuf writes)
  uint64_t *cq = (uint64_t *)(ub + (size_t)w * kFastTile);  // own U row, now free
  const float *Lq = Lbuf + (size_t)(q0 + w) * K;
  int nc = 0;
  bool overflow = false;
  for (int i0 = 0; i0 < K; i0 += 32) {
    const int k = i0 + lane;
    const bool take = k < K && Lq[k] <= Ustar;
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (nc + __popc(bal) > kCandCap) { overflow = true; break; }
    if (take) cq[nc + __popc(bal & ((1u << lane) - 1))] = (uint64_t)k;
    nc += __popc(bal);
  }
  __syncwarp();
  const float *qcol = sqT;  // query w at sqT[t * kFastQ + w]
  if (!overflow) {
    for (int i = lane; i < nc; i += 32) {
      const int k = (int)cq[i];
      const float *crow = coarse + (size_t)k * d;
      float a4[4] = {0.f, 0.f, 0.f, 0.f};
      int t0 = 0;
      for (; d - t0 >= 16; t0 += 16)
#pragma unroll
        for (int vv = 3; vv >= 0; vv--)
#pragma unroll
          for (int l = 0; l < 4; l++) {
            const int t = t0 + 4 * vv + l;
            const float df = __fsub_rn(crow[t], qcol[t * kFastQ + w]);
            a4[l] = __fadd_rn(a4[l], __fmul_rn(df, df));
          }
      for (; t0 < d; t0 += 4)
#pragma unroll
        for (int l = 0; l < 4; l++) {
          float pr = 0.f;
          if (t0 + l < d) {
            const float df = __fsub_rn(crow[t0 + l], qcol[(t0 + l) * kFastQ + w]);
            pr = __fmul_rn(df, df);
          }
          a4[l] = __fadd_rn(a4[l], pr);
        }
      const float E = __fadd_rn(__fadd_rn(a4[0], a4[1]), __fadd_rn(a4[2], a4[3]));
      cq[i] = ((uint64_t)__float_as_uint(E) << 32) | (uint32_t)k;
    }
    __syncwarp();
    int p2 = 1;
    while (p2 < nc) p2 <<= 1;
    for (int i = nc + lane; i < p2; i += 32) cq[i] = ~0ull;
    __syncwarp();
    warp_sort_u64(cq, p2);
    for (int i = lane; i < ma; i += 32) cells[(size_t)(q0 + w) * ma + i] = (int64_t)(cq[i] & 0xffffffffu);
    return;
  }
  // overflow: exact einsum over every cell, exact running selection
  nb = 0;
  bn = 0;
  T = ~0ull;
  for (int i0 = 0; i0 < K; i0 += 32) {
    const int k = i0 + lane;
    uint64_t key = ~0ull;
    if (k < K) {
      const float *crow = coarse + (size_t)k * d;
      float a4[4] = {0.f, 0.f, 0.f, 0.f};
      int t0 = 0;
      for (; d - t0 >= 16; t0 += 16)
        for (int vv = 3; vv >= 0; vv--)
          for (int l = 0; l < 4; l++) {
            const int t = t0 + 4 * vv + l;
            const float df = __fsub_rn(crow[t], qcol[t * kFastQ + w]);
            a4[l] = __fadd_rn(a4[l], __fmul_rn(df, df));
          }
      for (; t0 < d; t0 += 4)
        for (int l = 0; l < 4; l++) {
          float pr = 0.f;
          if (t0 + l < d) {
            const float df = __fsub_rn(crow[t0 + l], qcol[(t0 + l) * kFastQ + w]);
            pr = __fmul_rn(df, df);
          }
          a4[l] = __fadd_rn(a4[l], pr);
        }
      key = ((uint64_t)__float_as_uint(__fadd_rn(__fadd_rn(a4[0], a4[1]), __fadd_rn(a4[2], a4[3]))) << 32) |
            (uint32_t)k;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, key < T);
    if (bal) {
      if (bn + __popc(bal) > kSelBuf) warp_merge(v, nb, bn, ma, T);
      const bool take2 = key < T;
      const unsigned bal2 = __ballot_sync(0xffffffffu, take2);
      if (take2) v[nb + bn + __popc(bal2 & ((1u << lane) - 1))] = key;
      bn += __popc(bal2);
      __syncwarp();
    }
  }
  warp_merge(v, nb, bn, ma, T);
  for (int i = lane; i < ma; i += 32) cells[(size_t)(q0 + w) * ma + i] = (int64_t)(v[i] & 0xffffffffu);
}

// ---------------- residual + rotation + LUT (adc.py:108-111, 141-148,
// ivf.py:181-182) ----------------
// kLutPairs (query, probe slot) pairs per CTA. residual = q - C[cell] in
// fp32. OPQ rotation y = R r in the reference's own arithmetic: _rotate
// computes (v @ R.T) with a 1-D v, i.e. OpenBLAS sgemv_t (numpy's
// scipy-openblas 0.3.30, DYNAMIC_ARCH core "SkylakeX" / Haswell kernels).
// Its order, identified bit-for-bit on this project's hosts (d >= 16,
// d % 8 == 0: 100 % of outputs, tests/test_oracle.py): eight fp32 FMA lane
// accumulators, lane l taking k = l, l + 8, l + 16, ... in ascending k; then
// t_l = acc_l + acc_{l+4} (l < 4) and y = (t0 + t1) + (t2 + t3). R^T is
// read through L1 (64 KB, float4 rows: 4 consecutive outputs per thread).
constexpr int kLutPairs = 32;  // (query, slot) pairs per CTA (4 pairs x 4 outputs per thread task)

__device__ __forceinline__ float blas8_fold(const float (&a)[8]) {
  return __fadd_rn(__fadd_rn(__fadd_rn(a[0], a[4]), __fadd_rn(a[1], a[5])),
                   __fadd_rn(__fadd_rn(a[2], a[6]), __fadd_rn(a[3], a[7])));
}

__global__ void __launch_bounds__(256) k_residual_lut(
    const float *__restrict__ queries, const float *__restrict__ coarse,
    const float *__restrict__ rotation, const float *__restrict__ rotT,
    const float *__restrict__ codebooks, const int64_t *__restrict__ cells, int d, int m,
    int nslots, int npairs, int ppc, float *__restrict__ lut) {
  extern __shared__ __align__(16) float smf[];
  float *sr = smf;                                              // [ppc][d]
  float *sy = sr + (size_t)ppc * d;                             // [ppc][d]
  const int p0 = blockIdx.x * ppc;
  const int np = min(ppc, npairs - p0);
  if ((d & 3) == 0) {  // residual rows as float4 (query and centroid rows are 16-byte aligned)
    const int d4 = d >> 2;
    for (int e = threadIdx.x; e < np * d4; e += blockDim.x) {
      const int p = e / d4, t = e - p * d4;
      const int pair = p0 + p;
      float4 qv = ((const float4 *)(queries + (size_t)(pair / nslots) * d))[t];
      if (coarse) {
        const float4 c = ((const float4 *)(coarse + (size_t)cells[pair] * d))[t];
        qv = make_float4(__fsub_rn(qv.x, c.x), __fsub_rn(qv.y, c.y), __fsub_rn(qv.z, c.z),
                         __fsub_rn(qv.w, c.w));
      }
      ((float4 *)sr)[e] = qv;
    }
  } else {
    for (int e = threadIdx.x; e < np * d; e += blockDim.x) {
      const int p = e / d, t = e - p * d;
      const int pair = p0 + p;
      const float qv = queries[(size_t)(pair / nslots) * d + t];
      sr[e] = coarse ? __fsub_rn(qv, coarse[(size_t)cells[pair] * d + t]) : qv;
    }
  }
  __syncthreads();
  const float *y = sr;
  if (rotation) {
    if ((d & 7) == 0 && (np & 3) == 0) {
      // thread task: 4 consecutive outputs x 4 pairs. The 8 lane sums of
      // the OpenBLAS order are produced one lane at a time (16 FMAs over
      // k = 8 kk + l each) in the fold's order l = 0, 4, 1, 5, 2, 6, 3, 7,
      // so only the running partial folds stay live: 16 accumulators + 3
      // partials per output, one float4 of R^T row k (L1, shared by the
      // 4 pairs) and 4 broadcast residual values per k.
      const int quads = d >> 2;
      for (int task = threadIdx.x; task < (np >> 2) * quads; task += blockDim.x) {
        const int pg = task / quads, i0 = (task - pg * quads) * 4;
        const float *r0 = sr + (size_t)(4 * pg) * d;
        float s0[4][4], s1[4][4], s2[4][4];
#pragma unroll
        for (int li = 0; li < 8; li++) {
          const int l = (li >> 1) + 4 * (li & 1);  // 0, 4, 1, 5, 2, 6, 3, 7
          float acc[4][4];
#pragma unroll
          for (int u = 0; u < 4; u++)
#pragma unroll
            for (int h = 0; h < 4; h++) acc[u][h] = 0.f;
#pragma unroll 4
          for (int k = l; k < d; k += 8) {
            const float4 c = __ldg((const float4 *)(rotT + (size_t)k * d + i0));
            const float cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int h = 0; h < 4; h++) {
              const float rv = r0[(size_t)h * d + k];
#pragma unroll
              for (int u = 0; u < 4; u++) acc[u][h] = __fmaf_rn(cc[u], rv, acc[u][h]);
            }
          }
#pragma unroll
          for (int u = 0; u < 4; u++)
#pragma unroll
            for (int h = 0; h < 4; h++) {
              const float x = acc[u][h];
              switch (li) {
                case 0: s0[u][h] = x; break;                                   // a0
                case 1: s0[u][h] = __fadd_rn(s0[u][h], x); break;              // a0 + a4
                case 2: s1[u][h] = x; break;                                   // a1
                case 3: s1[u][h] = __fadd_rn(s1[u][h], x);                     // a1 + a5
                        s0[u][h] = __fadd_rn(s0[u][h], s1[u][h]); break;       // (a0+a4)+(a1+a5)
                case 4: s1[u][h] = x; break;                                   // a2
                case 5: s1[u][h] = __fadd_rn(s1[u][h], x); break;              // a2 + a6
                case 6: s2[u][h] = x; break;                                   // a3
                default: s2[u][h] = __fadd_rn(s2[u][h], x);                    // a3 + a7
                         s1[u][h] = __fadd_rn(s1[u][h], s2[u][h]);             // (a2+a6)+(a3+a7)
                         s0[u][h] = __fadd_rn(s0[u][h], s1[u][h]);
              }
            }
        }
#pragma unroll
        for (int h = 0; h < 4; h++)
          *(float4 *)(sy + (size_t)(4 * pg + h) * d + i0) =
              make_float4(s0[0][h], s0[1][h], s0[2][h], s0[3][h]);
      }
    } else {
      for (int e = threadIdx.x; e < np * d; e += blockDim.x) {
        const int p = e / d, i = e - p * d;
        const float *r = sr + (size_t)p * d;
        float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int k0 = 0; k0 < d; k0 += 8) {
#pragma unroll
          for (int l = 0; l < 8; l++)
            if (k0 + l < d) a[l] = __fmaf_rn(rotT[(size_t)(k0 + l) * d + i], r[k0 + l], a[l]);
        }
        sy[e] = blas8_fold(a);
      }
    }
    __syncthreads();
    y = sy;
  }
  const int dsub = d / m;
  if (dsub == 4) {
    // the einsum of one 4-vector (NumPy order for n = 4: products rounded,
    // lanes (l0 + l1) + (l2 + l3)); entry (p, j, c) = (pair, sub-space, centroid)
    const int per = m * 16;
    for (int e = threadIdx.x; e < np * per; e += blockDim.x) {
      const int p = e / per, ent = e - p * per;
      const float4 c4 = __ldg((const float4 *)codebooks + ent);
      const float4 y4 = ((const float4 *)(y + (size_t)p * d))[ent >> 4];
      const float a0 = __fsub_rn(c4.x, y4.x), a1 = __fsub_rn(c4.y, y4.y);
      const float a2 = __fsub_rn(c4.z, y4.z), a3 = __fsub_rn(c4.w, y4.w);
      lut[(size_t)(p0 + p) * per + ent] =
          __fadd_rn(__fadd_rn(__fmul_rn(a0, a0), __fmul_rn(a1, a1)),
                    __fadd_rn(__fmul_rn(a2, a2), __fmul_rn(a3, a3)));
    }
    return;
  }
  for (int e = threadIdx.x; e < np * m * 16; e += blockDim.x) {
    const int p = e / (m * 16), ent = e - p * m * 16;
    const int j = ent >> 4;
    const float *cb = codebooks + (size_t)ent * dsub;
    lut[(size_t)(p0 + p) * m * 16 + ent] =
        einsum_sq([&](int t) { return cb[t]; }, y + (size_t)p * d + (size_t)j * dsub, dsub);
  }
}

// ---------------- find_qmax (qadc.py:157-194, adc.py:170-172) ----------------
// One CTA per query, first probed cell only. Each thread computes the fp32
// left-to-right ADC of prefix codes (_pykernels.py:24-27 order: per byte j,
// low nibble table 2j then high nibble table 2j+1), the block then selects
// the min(R, take)-th smallest value by an MSB radix select on the bit
// patterns (distances >= 0). Empty cell: NumPy pairwise sum of row maxima.
__global__ void __launch_bounds__(256) k_qmax(const uint32_t *__restrict__ codes,
                                              const int64_t *__restrict__ chunk_off,
                                              const int64_t *__restrict__ count,
                                              const float *__restrict__ lut,
                                              const int64_t *__restrict__ cells, int m, int nslots,
                                              int R, int init, unsigned *__restrict__ scratch,
                                              int scratch_per_q, int q0,
                                              float *__restrict__ qmax) {
  extern __shared__ unsigned char smem[];
  float *st = (float *)smem;  // m * 16
  __shared__ unsigned hist[256];
  __shared__ unsigned s_prefix;
  __shared__ int s_k;
  const int q = q0 + blockIdx.x;
  const int pair = q * nslots;
  const int64_t L = cells ? cells[pair] : 0;
  for (int e = threadIdx.x; e < m * 16; e += blockDim.x) st[e] = lut[(size_t)pair * m * 16 + e];
  __syncthreads();
  const int64_t cnt = count[L];
  const int take = (int)(cnt < (int64_t)init ? cnt : (int64_t)init);
  if (take <= 0) {
    if (threadIdx.x == 0) {
      float mx[kMaxM];
      for (int j = 0; j < m; j++) {
        float v = st[j * 16];
        for (int i = 1; i < 16; i++) v = fmaxf(v, st[j * 16 + i]);
        mx[j] = v;
      }
      qmax[q] = pairwise_sum(mx, m);
    }
    return;
  }
  unsigned *keys = scratch + (size_t)blockIdx.x * scratch_per_q;  // take <= scratch_per_q
  const int64_t c0 = chunk_off[L];
  for (int k = threadIdx.x; k < take; k += blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j < m; j += 2) {
      acc = __fadd_rn(acc, st[j * 16 + code_nibble(codes, m, c0, k, j)]);
      acc = __fadd_rn(acc, st[(j + 1) * 16 + code_nibble(codes, m, c0, k, j + 1)]);
    }
    keys[k] = __float_as_uint(acc);
  }
  __syncthreads();
  if (threadIdx.x == 0) { s_prefix = 0; s_k = min(R, take); }
  __syncthreads();
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const unsigned prefix = s_prefix;
    const unsigned hmask = shift == 24 ? 0u : (~0u << (shift + 8));
    for (int i = threadIdx.x; i < take; i += blockDim.x) {
      const unsigned key = keys[i];
      if ((key & hmask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int kk = s_k, dgt = 0;
      for (; dgt < 256; dgt++) {
        if ((int)hist[dgt] >= kk) break;
        kk -= hist[dgt];
      }
      s_k = kk;
      s_prefix = prefix | ((unsigned)dgt << shift);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) qmax[q] = __uint_as_float(s_prefix);
}

// ---------------- quantize_tables (qadc.py:124-147, adc.py:173-174) ----------------
// One CTA (64 threads) per (query, slot). qmin = min(LUT min, qmax) and
// delta = (qmax - qmin) / 127 in float64, bins floor((v - qmin) / delta)
// clipped to 0..127 (delta == 0: v <= qmin -> 0 else 127). Emits the byte
// tables as 4 words per sub-quantizer (entries 0-7 | 8-15), and the fp32
// casts of qmin / delta the Cython boundary makes (_kernels.pyx:82-83).
// One warp per (query, slot) pair, 8 pairs per CTA.
__global__ void __launch_bounds__(256) k_quantize(const float *__restrict__ lut, int m, int npairs,
                                                  const float *__restrict__ qmax_q, int nslots,
                                                  const double *__restrict__ qmin_in,
                                                  const double *__restrict__ qmax_in,
                                                  uint32_t *__restrict__ qt, float *__restrict__ qmin_f,
                                                  float *__restrict__ delta_f,
                                                  double *__restrict__ delta_out,
                                                  uint8_t *__restrict__ qt_bytes, int max_depth,
                                                  uint8_t *__restrict__ pair_depth) {
  __shared__ unsigned s_rmax[8][kMaxM];
  const int lane = threadIdx.x & 31;
  const int pair = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (pair >= npairs) return;
  unsigned *rmax = s_rmax[threadIdx.x >> 5];
  if (pair_depth) {
    for (int j = lane; j < m; j += 32) rmax[j] = 0;
    __syncwarp();
  }
  const float *t = lut + (size_t)pair * m * 16;
  // m <= 32: the pair's table (<= 512 floats) is read once, 4 float4 per
  // lane, and both passes (minimum, bins) run from registers
  const bool in_regs = m <= 32;
  float4 tv[4];
  if (in_regs) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int w = lane + 32 * i;
      tv[i] = w < m * 4 ? *(const float4 *)(t + w * 4) : make_float4(FLT_MAX, FLT_MAX, FLT_MAX, FLT_MAX);
    }
  }
  double qmin, qmax;
  if (qmin_in) {
    qmin = qmin_in[pair];
    qmax = qmax_in[pair];
  } else {
    float mn = FLT_MAX;
    if (in_regs) {
#pragma unroll
      for (int i = 0; i < 4; i++)
        mn = fminf(mn, fminf(fminf(tv[i].x, tv[i].y), fminf(tv[i].z, tv[i].w)));
    } else {
      for (int e = lane; e < m * 16; e += 32) mn = fminf(mn, t[e]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    qmax = (double)qmax_q[pair / nslots];
    qmin = fmin((double)mn, qmax);
  }
  const double delta = __ddiv_rn(__dsub_rn(qmax, qmin), (double)kQuantBins);
  // floor(fl(x / delta)) without a float64 division per entry (software
  // division: ~10 % of this kernel at configs[4]): k = floor(x *
  // fl(1 / delta)) is accepted when the exactly rounded residuals x - k delta
  // >= margin and x - (k + 1) delta <= -margin (margin = 2^-40 delta, far
  // above the spacing of doubles below 128): then k < x / delta < k + 1 -
  // 2^-41, so the rounded quotient lies in [k, k + 1) too. Anything else
  // (quotients within 2^-40 of an integer, overflow, NaN) takes the division.
  const double rdelta = delta > 0 ? __ddiv_rn(1.0, delta) : 0.0;
  const double marg = delta * 0x1p-40;
  auto quant_word = [&](int w, const float4 v4) {
    const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
    uint32_t word = 0;
#pragma unroll
    for (int b = 0; b < 4; b++) {
      const double v = (double)vv[b];
      double qq;
      if (delta > 0) {
        const double x = __dsub_rn(v, qmin);
        qq = floor(__dmul_rn(x, rdelta));
        const double r0 = __fma_rn(-qq, delta, x), r1 = __fma_rn(-(qq + 1.0), delta, x);
        if (!(r0 >= marg && r1 <= -marg)) qq = floor(__ddiv_rn(x, delta));
        qq = fmin(fmax(qq, 0.0), (double)kQuantBins);
      } else {
        qq = v <= qmin ? 0.0 : (double)kQuantBins;
      }
      const uint32_t byte = (uint32_t)qq;
      word |= byte << (8 * b);
      if (qt_bytes) qt_bytes[(size_t)pair * m * 16 + w * 4 + b] = (uint8_t)byte;
    }
    if (qt) qt[(size_t)pair * m * 4 + w] = word;
    if (pair_depth) {
      const uint32_t mx = __vmaxu4(word, word >> 16);
      atomicMax(&rmax[w >> 2], max(mx & 255u, (mx >> 8) & 255u));
    }
  };
  if (in_regs) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      if (lane + 32 * i < m * 4) quant_word(lane + 32 * i, tv[i]);
  } else {
    for (int w = lane; w < m * 4; w += 32) quant_word(w, *(const float4 *)(t + w * 4));
  }
  if (pair_depth) {
    // byte-sum depth of this pair's scan: the largest D in {16, 8, 4, 2}
    // (<= max_depth) such that every aligned group of D sub-quantizers has
    // row maxima summing to <= 255, so D byte lanes add without carry
    // (D = 2 always holds: entries are <= 127)
    __syncwarp();
    if (lane == 0) {
      int dd = max_depth;
      for (; dd > 2; dd >>= 1) {
        bool ok = true;
        for (int j0 = 0; j0 < m && ok; j0 += dd) {
          unsigned sum = 0;
          for (int j = j0; j < min(j0 + dd, m); j++) sum += rmax[j];
          ok = sum <= 255u;
        }
        if (ok) break;
      }
      pair_depth[pair] = (uint8_t)dd;
    }
  }
  if (lane == 0) {
    if (qmin_f) qmin_f[pair] = __double2float_rn(qmin);
    if (delta_f) delta_f[pair] = __double2float_rn(delta);
    if (delta_out) delta_out[pair] = delta;
  }
}

// ---------------- prefix facts per query ----------------
// (1) F_sat: saturated lanes among the first R valid lanes of the global
//     stream (cells in probe order, lanes in list order). The reference's
//     heap admits every lane while below capacity and saturated lanes never
//     afterwards (scan_kernels.c:279-308); the order-free equivalent keeps
//     exactly these (_pykernels.py:80-83).
// (2) Initial distance bound M: max midpoint of those first R valid lanes,
//     tightened by the R-th smallest non-saturated midpoint among the
//     first max(init, kBoundPrefix) codes of the first cell. Both are midpoints of members
//     of the candidate set, so at least R candidates lie at or below M.
__global__ void __launch_bounds__(256) k_prefix(const uint32_t *__restrict__ codes,
                                                const int64_t *__restrict__ chunk_off,
                                                const int64_t *__restrict__ lanes,
                                                const int64_t *__restrict__ ids,
                                                const uint32_t *__restrict__ qt,
                                                const float *__restrict__ qmin_f,
                                                const float *__restrict__ delta_f,
                                                const int64_t *__restrict__ cells, int m,
                                                int nslots, int R, int init, int bound_prefix,
                                                int prefix_div,
                                                unsigned *__restrict__ M_bits, int *__restrict__ fsat_n,
                                                float *__restrict__ fsat_mid,
                                                int64_t *__restrict__ fsat_id) {
  __shared__ __align__(16) unsigned char sqt[kMaxM * 16];
  __shared__ int warp_cnt[8];
  __shared__ unsigned hist[256];
  __shared__ unsigned whist[8][256];  // per-warp prefix histograms (no cross-warp atomic contention)
  __shared__ int s_seen, s_nsat;
  __shared__ unsigned s_maxmid;
  const int q = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) { s_seen = 0; s_nsat = 0; s_maxmid = 0; }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&whist[0][0])[i] = 0;
  __syncthreads();
  for (int s = 0; s < nslots; s++) {
    // later cells matter only while fewer than R valid lanes have been seen
    // (s_seen is stable here: last written before a barrier); without this
    // exit every query staged the tables of all its probed cells
    if (s > 0 && s_seen >= R) break;
    const int pair = q * nslots + s;
    const int64_t L = cells ? cells[pair] : 0;
    const int64_t c0 = chunk_off[L], n = lanes[L];
    const float qmin = qmin_f[pair], delta = delta_f[pair];
    // bound prefix of cell 0: at least init codes, and up to kBoundPrefix
    // (at most 1/64 of the list) so the initial bound starts near the
    // R/prefix quantile without costing more than ~2% of the scan
    int64_t want = n / prefix_div < bound_prefix ? n / prefix_div : bound_prefix;
    if (want < init) want = init;
    const int64_t pref = (s == 0) ? (want < n ? want : n) : 0;
    for (int e = threadIdx.x; e < m * 4; e += blockDim.x)
      ((uint32_t *)sqt)[e] = qt[(size_t)pair * m * 4 + e];
    __syncthreads();
    // (1) stream order, only until R valid lanes are seen
    for (int64_t base = 0; base < n; base += blockDim.x) {
      if (s_seen >= R) break;
      const int64_t k = base + threadIdx.x;
      bool valid = false;
      int qv = 255;
      int64_t id = -1;
      if (k < n) {
        id = ids[c0 * kChunkCodes + k];
        valid = id >= 0;
        int acc = 0;
        for (int j = 0; j < m; j++) acc += sqt[j * 16 + code_nibble(codes, m, c0, k, j)];
        qv = min(acc, 255);
      }
      // block exclusive scan of valid flags -> stream rank
      const unsigned bal = __ballot_sync(0xffffffffu, valid);
      if (lane == 0) warp_cnt[wid] = __popc(bal);
      __syncthreads();
      int before = 0, total = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
        if (w < wid) before += warp_cnt[w];
        total += warp_cnt[w];
      }
      const int rank = s_seen + before + __popc(bal & ((1u << lane) - 1));
      if (valid && rank < R) {
        const float mid = midpoint(qmin, delta, qv);
        atomicMax(&s_maxmid, fbits(mid));
        if (qv == 255) {
          const int p = atomicAdd(&s_nsat, 1);
          fsat_mid[(size_t)q * R + p] = mid;
          fsat_id[(size_t)q * R + p] = id;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) s_seen += total;
      __syncthreads();
    }
    // (2) bound histogram of the prefix: one octet (8 codes) per thread,
    // each interleaved word read once (coalesced across the CTA)
    // PRMT lookups (entries <= 127): prmt(t0, t1, sel) gives entries 0-7 and
    // 0 for selectors >= 8 (sign replicate of a non-negative byte); with
    // sel ^ 0x8888 and (t2, t3) the other half. Bytes of two sub-quantizers
    // add without carry (<= 254), then widen into 16-bit lanes. The words of
    // 8 sub-quantizers are loaded together (independent L2 round trips).
    for (int64_t o = threadIdx.x; o * 8 < pref; o += blockDim.x) {
      const int64_t g = c0 + o / 32;
      const uint32_t *wp = codes + g * m * 32 + (o % 32);
      uint32_t a02 = 0, a13 = 0, a46 = 0, a57 = 0;  // 16-bit lanes: codes (0,2), (1,3), (4,6), (5,7)
      for (int j0 = 0; j0 < m; j0 += 8) {
        uint32_t wv[8];
#pragma unroll
        for (int jj = 0; jj < 8; jj++) wv[jj] = j0 + jj < m ? __ldg(wp + (j0 + jj) * 32) : 0u;
#pragma unroll
        for (int jj = 0; jj < 8; jj += 2) {
          uint32_t lo = 0, hi = 0;  // bytes: codes 0-3 / 4-7, two sub-quantizers
#pragma unroll
          for (int u = 0; u < 2; u++) {
            const int j = j0 + jj + u;
            if (j < m) {
              const uint32_t w = wv[jj + u];
              const uint4 t = *(const uint4 *)(sqt + j * 16);
              const uint32_t s1 = w >> 16;
              lo += prmt(t.x, t.y, w) | prmt(t.z, t.w, w ^ 0x8888u);
              hi += prmt(t.x, t.y, s1) | prmt(t.z, t.w, s1 ^ 0x8888u);
            }
          }
          a02 += lo & 0x00ff00ffu;
          a13 += (lo >> 8) & 0x00ff00ffu;
          a46 += hi & 0x00ff00ffu;
          a57 += (hi >> 8) & 0x00ff00ffu;
        }
      }
      const uint32_t acc[8] = {a02 & 0xffffu, a13 & 0xffffu, a02 >> 16, a13 >> 16,
                               a46 & 0xffffu, a57 & 0xffffu, a46 >> 16, a57 >> 16};
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const int64_t kk = o * 8 + k;
        if (kk < pref && acc[k] < 255 && ids[c0 * kChunkCodes + kk] >= 0)
          atomicAdd(&whist[wid][acc[k]], 1u);
      }
    }
    __syncthreads();
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 256; t += blockDim.x) {
    unsigned c = 0;
#pragma unroll
    for (int w = 0; w < 8; w++) c += whist[w][t];
    hist[t] += c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = __int_as_float(0x7f800000);  // +inf
    if (s_seen >= R) M = __uint_as_float(s_maxmid);
    int cum = 0;
    for (int t = 0; t < 255; t++) {
      cum += hist[t];
      if (cum >= R) {
        const int pair0 = q * nslots;
        M = fminf(M, midpoint(qmin_f[pair0], delta_f[pair0], t));
        break;
      }
    }
    M_bits[q] = fbits(M);
    fsat_n[q] = s_nsat;
  }
}

}  // namespace

void launch_compute_tables(const float *codebooks, int m, int dsub, const float *y, int npairs,
                           float *out, cudaStream_t st) {
  if (npairs <= 0) return;
  k_tables<<<npairs, 256, (size_t)m * dsub * 4, st>>>(codebooks, m, dsub, y, out);
}

void launch_probe(const float *coarseT, int K, int d, const float *queries, int nq, int ma,
                  int64_t *cells, cudaStream_t st) {
  if (nq <= 0) return;
  int vcap = 1;
  while (vcap < ma + kSelBuf) vcap <<= 1;
  int tile = kProbeTile;
  size_t smem = 0;
  for (;; tile >>= 1) {
    smem = (size_t)kProbeQ * tile * 8 + (size_t)kProbeQ * vcap * 8 + (size_t)kProbeQ * d * 4;
    if (smem <= 220 * 1024 || tile <= 256) break;
  }
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_probe<<<(nq + kProbeQ - 1) / kProbeQ, 256, smem, st>>>(coarseT, K, d, queries, nq, ma, tile,
                                                          vcap, cells);
}

void launch_cnorm(const float *coarse, int K, int d, float *cn, cudaStream_t st) {
  k_cnorm<<<(K + 255) / 256, 256, 0, st>>>(coarse, K, d, cn);
}

bool launch_probe_fast(const float *coarseT, const float *coarse, const float *cn, int K, int d,
                       const float *queries, int nq, int ma, int64_t *cells, cudaStream_t st) {
  if (nq <= 0) return true;
  if (ma > kCandCap / 2 || ma > K) return false;
  int vcap = 1;
  while (vcap < ma + kSelBuf) vcap <<= 1;
  static_assert(kCandCap * 8 <= kFastTile * 4, "candidates reuse a U row");
  const size_t smem = (size_t)kFastQ * vcap * 8 + (size_t)kFastQ * kFastTile * 4 +
                      (size_t)kFastQ * d * 4;
  if (smem > 220 * 1024) return false;
  float *Lbuf = nullptr;
  if (cudaMallocAsync(&Lbuf, (size_t)nq * K * 4, st) != cudaSuccess) return false;
  cudaFuncSetAttribute(k_probe_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_probe_fast<<<(nq + kFastQ - 1) / kFastQ, 256, smem, st>>>(coarseT, coarse, cn, K, d, queries,
                                                             nq, ma, vcap, Lbuf, cells);
  cudaFreeAsync(Lbuf, st);
  return true;
}

void launch_residual_lut(const qadc_b200_index *idx, const float *queries, const int64_t *cells,
                         int nq, int nslots, float *lut, cudaStream_t st) {
  if (nq <= 0) return;
  const int npairs = nq * nslots, d = idx->d;
  // residual + rotated vectors of ppc pairs in shared memory (fp32): fewer
  // pairs per CTA for large d so any d fits the 227 KB limit
  const int ppc = (int)std::max<int64_t>(1, std::min<int64_t>(kLutPairs, (220LL << 10) / (8LL * d)));
  const size_t smem = (size_t)ppc * d * 8;
  cudaFuncSetAttribute(k_residual_lut, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_residual_lut<<<(npairs + ppc - 1) / ppc, 256, smem, st>>>(
      queries, idx->K ? idx->coarse : nullptr, idx->rotation, idx->rotationT, idx->codebooks,
      cells, d, idx->m, nslots, npairs, ppc, lut);
}

int launch_qmax(const qadc_b200_index *idx, const float *lut, const int64_t *cells, int nq,
                int nslots, int R, int init, float *qmax, cudaStream_t st) {
  if (nq <= 0) return kOk;
  // per-query key scratch: min(init, longest list) values; queries run in
  // chunks so the workspace stays <= 256 MB for any init / batch size
  int64_t longest = 0;
  for (int64_t c : idx->h_count) longest = std::max(longest, c);
  const int per_q = (int)std::max<int64_t>(1, std::min<int64_t>(init, longest));
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(nq, (256LL << 20) / 4 / per_q));
  unsigned *scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, (size_t)chunk * per_q * 4, st);
  if (e != cudaSuccess) return cuda_fail(e, "alloc qmax scratch");
  for (int64_t q0 = 0; q0 < nq; q0 += chunk) {
    const int n = (int)std::min<int64_t>(chunk, nq - q0);
    k_qmax<<<n, 256, (size_t)idx->m * 64, st>>>(idx->pcodes, idx->pchunk_off, idx->count, lut,
                                                 idx->K ? cells : nullptr, idx->m, nslots, R, init,
                                                 scratch, per_q, (int)q0, qmax);
  }
  cudaFreeAsync(scratch, st);
  e = cudaGetLastError();
  return e == cudaSuccess ? kOk : cuda_fail(e, "k_qmax");
}

void launch_quantize(const float *lut, int npairs, int m, const float *qmax_per_query, int nslots,
                     const double *qmin_in, const double *qmax_in, uint32_t *qt, float *qmin_f,
                     float *delta_f, double *delta_out, uint8_t *qt_bytes_out, cudaStream_t st,
                     int max_depth, uint8_t *pair_depth) {
  if (npairs <= 0) return;
  k_quantize<<<(npairs + 7) / 8, 256, 0, st>>>(lut, m, npairs, qmax_per_query, nslots, qmin_in,
                                                qmax_in, qt, qmin_f, delta_f, delta_out,
                                                qt_bytes_out, max_depth, pair_depth);
}

void launch_prefix(const qadc_b200_index *idx, const uint32_t *qt, const float *qmin_f,
                   const float *delta_f, const int64_t *cells, int nq, int nslots, int R, int init,
                   unsigned *M_bits, int *fsat_n, float *fsat_mid, int64_t *fsat_id,
                   cudaStream_t st) {
  if (nq <= 0) return;
  // codes of the first cell's prefix behind the initial bound (tuning knob)
  static const int bound_prefix = std::max(256, scan_env_int("QADC_B200_BOUND_PREFIX", kBoundPrefix));
  // share of the first cell behind the initial bound: 1/64 of an exhaustive
  // list (~2 % of the scan); an inverted list is one of many, so all of it
  // (up to bound_prefix codes) — the streaming candidate count of an exact
  // top-R is ~R ln(n / prefix)
  static const int div_env = scan_env_int("QADC_B200_BOUND_PREFIX_DIV", 0);
  const int prefix_div = div_env > 0 ? div_env : (idx->K && nslots > 1 ? 1 : 64);
  k_prefix<<<nq, 256, 0, st>>>(idx->pcodes, idx->pchunk_off, idx->planes, idx->pids, qt, qmin_f,
                               delta_f, idx->K ? cells : nullptr, idx->m, nslots, R, init,
                               bound_prefix, prefix_div, M_bits,
                               fsat_n, fsat_mid, fsat_id);
}

}  // namespace qadc
