// Final exact top-R per query (heap.py:112-115 extract order): the union of
// the scan's surviving candidates (midpoint <= the query's final bound M)
// and the saturated first-R lanes F_sat, ordered by (midpoint, id); the
// first R are written out. The candidate set is exactly the one the
// reference heap would have admitted, filtered only by a bound
// that at least R candidates satisfy, so the top-R is identical.
//
// One CTA per query. Up to kSmall entries are bitonic-sorted in shared
// memory. Larger sets (heavy ties at the boundary level) run an exact
// radix select instead: three histogram passes over the midpoint bits
// find the R-th smallest midpoint m* and the number of entries below it;
// the k = R - below smallest ids among the entries AT m* come from a
// shared-memory sort of those ties (or, beyond kSmall ties, six more
// histogram passes over the id bits); then exactly R entries
// {mid < m*} U {mid = m*, id <= id*} are gathered and sorted.
#include "internal.cuh"

namespace qadc {
namespace {

constexpr int kSmall = 2048;  // entries sorted directly in shared memory
constexpr int kThreads = 256;
constexpr int kBins = 2048;   // radix digit of 11 bits

struct SelectIn {
  const float *cm;      // candidate midpoints of this query
  const int64_t *ci;    // candidate ids
  unsigned total;       // candidates (<= cap_g)
  const float *fm;      // F_sat midpoints
  const int64_t *fi;
  int nf;
  float M;              // final bound
  __device__ __forceinline__ bool get(int i, float &d, int64_t &id) const {
    if (i < (int)total) {
      d = cm[i];
      id = ci[i];
      return d <= M;
    }
    d = fm[i - total];
    id = fi[i - total];
    return true;
  }
  __device__ __forceinline__ int size() const { return (int)total + nf; }
};

__device__ __forceinline__ void bitonic_sort(float *sm, int64_t *si, int p2) {
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
}

// Bin holding the k-th (1-based) entry of a kBins histogram, and the
// number of entries in lower bins. All threads return the same values.
__device__ __forceinline__ void find_bin(const unsigned *hist, unsigned k, int &bin,
                                         unsigned &below, unsigned *s_part, int *s_bin,
                                         unsigned *s_below) {
  constexpr int per = kBins / kThreads;  // bins per thread
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  unsigned c = 0;
#pragma unroll
  for (int i = 0; i < per; i++) c += hist[t * per + i];
  unsigned incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_part[w] = incl;
  __syncthreads();
  unsigned off = 0;
  for (int i = 0; i < w; i++) off += s_part[i];
  const unsigned lo = off + incl - c;  // entries in bins below this thread's
  if (lo < k && k <= lo + c) {
    unsigned cum = lo;
    int b = t * per;
    for (int i = 0; i < per; i++, b++) {
      if (cum + hist[b] >= k) break;
      cum += hist[b];
    }
    *s_bin = b;
    *s_below = cum;
  }
  __syncthreads();
  bin = *s_bin;
  below = *s_below;
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) k_select(int R, const unsigned *__restrict__ M_bits,
                                                     const unsigned *__restrict__ cand_n,
                                                     const float *__restrict__ cand_mid,
                                                     const int64_t *__restrict__ cand_id, int cap_g,
                                                     const int *__restrict__ fsat_n,
                                                     const float *__restrict__ fsat_mid,
                                                     const int64_t *__restrict__ fsat_id,
                                                     int64_t *__restrict__ out_ids,
                                                     float *__restrict__ out_d,
                                                     int32_t *__restrict__ out_n,
                                                     int *__restrict__ overflow) {
  __shared__ int64_t si[kSmall];
  __shared__ float sm[kSmall];
  __shared__ unsigned hist[kBins];
  __shared__ unsigned s_part[kThreads / 32];
  __shared__ int s_cnt, s_bin;
  __shared__ unsigned s_below;
  const int q = blockIdx.x;
  const unsigned total = cand_n[q];
  if (total > (unsigned)cap_g) {  // candidates were dropped: rerun needed
    if (threadIdx.x == 0) overflow[q] = (int)min(total, 0x7fffffffu);
    return;
  }
  SelectIn in;
  in.cm = cand_mid + (size_t)q * cap_g;
  in.ci = cand_id + (size_t)q * cap_g;
  in.total = total;
  in.fm = fsat_mid + (size_t)q * R;
  in.fi = fsat_id + (size_t)q * R;
  in.nf = fsat_n[q];
  in.M = __uint_as_float(M_bits[q]);
  const int size = in.size();
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  // ---- count (and gather while they fit) the valid entries ----
  for (int i = threadIdx.x; i < size; i += blockDim.x) {
    float d;
    int64_t id;
    if (!in.get(i, d, id)) continue;
    const int p = atomicAdd(&s_cnt, 1);
    if (p < kSmall) { sm[p] = d; si[p] = id; }
  }
  __syncthreads();
  const int n = s_cnt;
  int nsel = n;  // entries in sm/si to sort
  if (n > kSmall) {
    if (R > kSmall) {  // the exact R-set itself exceeds shared memory
      if (threadIdx.x == 0) overflow[q] = n;
      return;
    }
    // ---- radix select of the R-th smallest midpoint (3 x 11 bits) ----
    unsigned k = (unsigned)R, val = 0, mask = 0;
    const int shifts[3] = {21, 10, 0};
    const unsigned widths[3] = {0x7ffu, 0x7ffu, 0x3ffu};
    unsigned ties = 0;
    for (int p = 0; p < 3; p++) {
      for (int i = threadIdx.x; i < kBins; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < size; i += blockDim.x) {
        float d;
        int64_t id;
        if (!in.get(i, d, id)) continue;
        const unsigned key = __float_as_uint(d);
        if ((key & mask) == val) atomicAdd(&hist[(key >> shifts[p]) & widths[p]], 1u);
      }
      __syncthreads();
      int b;
      unsigned below;
      find_bin(hist, k, b, below, s_part, &s_bin, &s_below);
      ties = hist[b];
      __syncthreads();  // hist is cleared by the next pass
      k -= below;
      val |= (unsigned)b << shifts[p];
      mask |= widths[p] << shifts[p];
    }
    const float mstar = __uint_as_float(val);
    // ---- the k smallest ids among the `ties` entries at m* ----
    int64_t idstar;
    if (ties <= (unsigned)kSmall) {
      if (threadIdx.x == 0) s_cnt = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < size; i += blockDim.x) {
        float d;
        int64_t id;
        if (!in.get(i, d, id) || __float_as_uint(d) != val) continue;
        const int p = atomicAdd(&s_cnt, 1);
        sm[p] = d;
        si[p] = id;
      }
      __syncthreads();
      int p2 = 1;
      while (p2 < (int)ties) p2 <<= 1;
      for (int i = (int)ties + threadIdx.x; i < p2; i += blockDim.x) {
        sm[i] = mstar;
        si[i] = INT64_MAX;
      }
      __syncthreads();
      bitonic_sort(sm, si, p2);
      idstar = si[k - 1];
      __syncthreads();
    } else {  // ids are non-negative: 6 x 11-bit digits from bit 55 down
      uint64_t iv = 0, im = 0;
      for (int p = 0; p < 6; p++) {
        const int sh = 55 - 11 * p;
        const uint64_t wd = 0x7ffull;
        for (int i = threadIdx.x; i < kBins; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < size; i += blockDim.x) {
          float d;
          int64_t id;
          if (!in.get(i, d, id) || __float_as_uint(d) != val) continue;
          const uint64_t u = (uint64_t)id;
          if ((u & im) == iv) atomicAdd(&hist[(u >> sh) & wd], 1u);
        }
        __syncthreads();
        int b;
        unsigned below;
        find_bin(hist, k, b, below, s_part, &s_bin, &s_below);
        k -= below;
        iv |= (uint64_t)b << sh;
        im |= wd << sh;
      }
      idstar = (int64_t)iv;
    }
    // ---- gather exactly R entries: below m*, or at m* with id <= id* ----
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < size; i += blockDim.x) {
      float d;
      int64_t id;
      if (!in.get(i, d, id)) continue;
      const unsigned key = __float_as_uint(d);
      if (key < val || (key == val && id <= idstar)) {
        const int p = atomicAdd(&s_cnt, 1);
        sm[p] = d;
        si[p] = id;
      }
    }
    __syncthreads();
    nsel = s_cnt;  // == R
  }
  int p2 = 1;
  while (p2 < nsel) p2 <<= 1;
  for (int i = nsel + threadIdx.x; i < p2; i += blockDim.x) {
    sm[i] = __int_as_float(0x7f800000);
    si[i] = INT64_MAX;
  }
  __syncthreads();
  bitonic_sort(sm, si, p2);
  const int nout = min(nsel, R);
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

int select_capacity() { return kSmall; }

void launch_select(int nq, int R, const unsigned *M_bits, const unsigned *cand_n,
                   const float *cand_mid, const int64_t *cand_id, int cap_g, const int *fsat_n,
                   const float *fsat_mid, const int64_t *fsat_id, int64_t *out_ids, float *out_d,
                   int32_t *out_n, int *overflow, cudaStream_t st) {
  if (nq <= 0) return;
  k_select<<<nq, kThreads, 0, st>>>(R, M_bits, cand_n, cand_mid, cand_id, cap_g, fsat_n, fsat_mid,
                                    fsat_id, out_ids, out_d, out_n, overflow);
}

}  // namespace qadc
