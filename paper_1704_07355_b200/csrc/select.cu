// Final exact top-R per query (heap.py:112-115 extract order): the union of
// the scan's surviving candidates (midpoint <= the query's final bound M)
// and the saturated first-R lanes F_sat is sorted by (midpoint, id) and
// the first R are written out. The candidate set is exactly the one the
// reference heap would have admitted, filtered only by a bound
// that at least R candidates satisfy, so the top-R is identical.
#include "internal.cuh"

namespace qadc {
namespace {

constexpr int kSelCap = 8192;  // candidates sorted in shared memory (96 KB)

__global__ void __launch_bounds__(512) k_select(int R, const unsigned *__restrict__ M_bits,
                                                const unsigned *__restrict__ cand_n,
                                                const float *__restrict__ cand_mid,
                                                const int64_t *__restrict__ cand_id, int cap_g,
                                                const int *__restrict__ fsat_n,
                                                const float *__restrict__ fsat_mid,
                                                const int64_t *__restrict__ fsat_id,
                                                int64_t *__restrict__ out_ids, float *__restrict__ out_d,
                                                int32_t *__restrict__ out_n, int *__restrict__ overflow) {
  extern __shared__ __align__(16) unsigned char dsm[];
  int64_t *si = (int64_t *)dsm;
  float *sm = (float *)(dsm + (size_t)kSelCap * 8);
  __shared__ int s_cnt;
  const int q = blockIdx.x;
  const unsigned total = cand_n[q];
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  if (total > (unsigned)cap_g) {  // candidates were dropped: rerun needed
    if (threadIdx.x == 0) overflow[q] = (int)min(total, 0x7fffffffu);
    return;
  }
  const float M = __uint_as_float(M_bits[q]);
  const int nf = fsat_n[q];
  for (int i = threadIdx.x; i < (int)total + nf; i += blockDim.x) {
    float d;
    int64_t id;
    if (i < (int)total) {
      d = cand_mid[(size_t)q * cap_g + i];
      id = cand_id[(size_t)q * cap_g + i];
      if (!(d <= M)) continue;
    } else {
      d = fsat_mid[(size_t)q * R + (i - total)];
      id = fsat_id[(size_t)q * R + (i - total)];
    }
    const int p = atomicAdd(&s_cnt, 1);
    if (p < kSelCap) { sm[p] = d; si[p] = id; }
  }
  __syncthreads();
  const int n = s_cnt;
  if (n > kSelCap) {
    if (threadIdx.x == 0) overflow[q] = n;
    return;
  }
  int p2 = 1;
  while (p2 < n) p2 <<= 1;
  for (int i = n + threadIdx.x; i < p2; i += blockDim.x) {
    sm[i] = __int_as_float(0x7f800000);
    si[i] = INT64_MAX;
  }
  __syncthreads();
  for (int k = 2; k <= p2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < p2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const float a = sm[i], b = sm[ixj];
          const int64_t ia = si[i], ib = si[ixj];
          const bool up = (i & k) == 0;
          const bool gt = entry_less(b, ib, a, ia);
          if (gt == up) { sm[i] = b; sm[ixj] = a; si[i] = ib; si[ixj] = ia; }
        }
      }
      __syncthreads();
    }
  }
  const int nout = min(n, R);
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    out_ids[(size_t)q * R + i] = i < nout ? si[i] : -1;
    out_d[(size_t)q * R + i] = i < nout ? sm[i] : __int_as_float(0x7f800000);
  }
  if (threadIdx.x == 0) {
    out_n[q] = nout;
    overflow[q] = 0;
  }
}

}  // namespace

int select_capacity() { return kSelCap; }

void launch_select(int nq, int R, const unsigned *M_bits, const unsigned *cand_n,
                   const float *cand_mid, const int64_t *cand_id, int cap_g, const int *fsat_n,
                   const float *fsat_mid, const int64_t *fsat_id, int64_t *out_ids, float *out_d,
                   int32_t *out_n, int *overflow, cudaStream_t st) {
  if (nq <= 0) return;
  const size_t smem = (size_t)kSelCap * 12;
  cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_select<<<nq, 512, smem, st>>>(R, M_bits, cand_n, cand_mid, cand_id, cap_g, fsat_n, fsat_mid,
                               fsat_id, out_ids, out_d, out_n, overflow);
}

}  // namespace qadc
