// General-table engine on the reference's own layouts, for the per-list
// reference ABI (scan_kernels.h:15-46) where tables may hold any byte and
// the caller brings a partially filled heap:
//   * qadc_block_dists (scan_kernels.c:384-419): saturated lane sums;
//   * qadc_scan_u8 (scan_kernels.c:362-382): candidates = heap entries
//     U valid non-saturated lanes U saturated lanes among the first
//     (R - size) valid lanes (_pykernels.py:63-87), exact
//     top-R by (distance, id);
//   * adc_scan_f32 (scan_kernels.c:78-125): fp32 left-to-right float ADC,
//     top-R of heap U valid codes.
// The exact top-R of an arbitrary-size candidate set uses two stable
// device radix sorts (id, then distance) so (distance, id) order holds
// for any number of ties.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "internal.cuh"

namespace qadc {
namespace {

// One thread per (block, lane); saturating sum == min(255, plain sum).
__global__ void k_block_dists(const uint8_t *__restrict__ blocks, int64_t nblocks, int mrows,
                              const uint8_t *__restrict__ qt, int per_block, uint8_t *__restrict__ out) {
  const int64_t total = nblocks * 16;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bi = t >> 4;
    const int l = (int)(t & 15);
    const uint8_t *blk = blocks + (size_t)bi * mrows * 16;
    const uint8_t *tb = per_block ? qt + (size_t)bi * mrows * 32 : qt;
    int acc = 0;
    for (int j = 0; j < mrows; j++) {
      const uint8_t byte = blk[16 * j + l];
      acc += tb[32 * j + (byte & 15)] + tb[32 * j + 16 + (byte >> 4)];
    }
    out[t] = (uint8_t)min(acc, 255);
  }
}

__global__ void k_valid_flags(const int64_t *__restrict__ ids, int64_t n, int *__restrict__ flags) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    flags[t] = ids[t] >= 0;
}

// Candidate keys for the quantized per-list scan.
__global__ void k_u8_candidates(const uint8_t *__restrict__ lane_q, const int64_t *__restrict__ ids,
                                const int *__restrict__ rank, int64_t n, int free_slots, float qmin,
                                float delta, float *__restrict__ cd, int64_t *__restrict__ ci) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t id = ids[t];
    const int q = lane_q[t];
    const bool ok = id >= 0 && (q < 255 || rank[t] < free_slots);
    cd[t] = ok ? midpoint(qmin, delta, q) : __int_as_float(0x7f800000);
    ci[t] = ok ? id : INT64_MAX;
  }
}

// fp32 left-to-right float ADC (scan_kernels.c:78-125 accumulation order).
__global__ void k_adc_candidates(const uint8_t *__restrict__ codes, int64_t n,
                                 const int64_t *__restrict__ ids, int m, int b,
                                 const float *__restrict__ tables, float *__restrict__ cd,
                                 int64_t *__restrict__ ci) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float d = 0.f;
    if (b == 8) {
      const uint8_t *c = codes + (size_t)i * m;
      for (int j = 0; j < m; j++) d = __fadd_rn(d, tables[(size_t)j * 256 + c[j]]);
    } else if (b == 4) {
      const uint8_t *c = codes + (size_t)i * (m / 2);
      for (int j = 0; j < m / 2; j++) {
        d = __fadd_rn(d, tables[(size_t)(2 * j) * 16 + (c[j] & 15)]);
        d = __fadd_rn(d, tables[(size_t)(2 * j + 1) * 16 + (c[j] >> 4)]);
      }
    } else {
      const uint8_t *c = codes + (size_t)i * m * 2;
      for (int j = 0; j < m; j++) {
        const unsigned idx = (unsigned)c[2 * j] | ((unsigned)c[2 * j + 1] << 8);
        d = __fadd_rn(d, tables[(size_t)j * 65536 + idx]);
      }
    }
    const int64_t id = ids[i];
    cd[i] = id >= 0 ? d : __int_as_float(0x7f800000);
    ci[i] = id >= 0 ? id : INT64_MAX;
  }
}

__global__ void k_count_real(const int64_t *__restrict__ ci, int64_t n, int R, int *out) {
  __shared__ int c;
  if (threadIdx.x == 0) c = 0;
  __syncthreads();
  const int64_t lim = n < R ? n : R;
  for (int64_t i = threadIdx.x; i < lim; i += blockDim.x)
    if (ci[i] != INT64_MAX) atomicAdd(&c, 1);
  __syncthreads();
  if (threadIdx.x == 0) *out = c;
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)std::min<int64_t>(std::max<int64_t>(g, 1), 148 * 32);
}

}  // namespace

void launch_block_dists(const uint8_t *blocks, int64_t nblocks, int mrows, const uint8_t *qt,
                        int per_block, uint8_t *out, cudaStream_t st) {
  if (nblocks <= 0) return;
  k_block_dists<<<grid_for(nblocks * 16), 256, 0, st>>>(blocks, nblocks, mrows, qt, per_block, out);
}

int topr_sorted(const float *d, const int64_t *id, int64_t n, int R, float *out_d, int64_t *out_i,
                int *out_n, cudaStream_t st) {
  if (n <= 0) {
    *out_n = 0;
    return kOk;
  }
  float *d1 = nullptr, *d2 = nullptr;
  int64_t *i1 = nullptr, *i2 = nullptr;
  void *tmp = nullptr;
  int *dcnt = nullptr;
  size_t tb1 = 0, tb2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb1, id, i1, d, d1, n, 0, 64, st);
  cub::DeviceRadixSort::SortPairs(nullptr, tb2, d1, d2, i1, i2, n, 0, 32, st);
  QADC_CUDA(cudaMallocAsync(&d1, n * 4, st));
  QADC_CUDA(cudaMallocAsync(&d2, n * 4, st));
  QADC_CUDA(cudaMallocAsync(&i1, n * 8, st));
  QADC_CUDA(cudaMallocAsync(&i2, n * 8, st));
  QADC_CUDA(cudaMallocAsync(&tmp, std::max(tb1, tb2), st));
  QADC_CUDA(cudaMallocAsync(&dcnt, 4, st));
  size_t tb = std::max(tb1, tb2);
  // stable LSD composition: by id, then by distance (both stable)
  cub::DeviceRadixSort::SortPairs(tmp, tb, id, i1, d, d1, n, 0, 64, st);
  tb = std::max(tb1, tb2);
  cub::DeviceRadixSort::SortPairs(tmp, tb, d1, d2, i1, i2, n, 0, 32, st);
  k_count_real<<<1, 256, 0, st>>>(i2, n, R, dcnt);
  const int64_t lim = std::min<int64_t>(n, R);
  QADC_CUDA(cudaMemcpyAsync(out_d, d2, lim * 4, cudaMemcpyDeviceToDevice, st));
  QADC_CUDA(cudaMemcpyAsync(out_i, i2, lim * 8, cudaMemcpyDeviceToDevice, st));
  QADC_CUDA(cudaMemcpyAsync(out_n, dcnt, 4, cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(d1, st);
  cudaFreeAsync(d2, st);
  cudaFreeAsync(i1, st);
  cudaFreeAsync(i2, st);
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(dcnt, st);
  QADC_CUDA(cudaStreamSynchronize(st));
  return kOk;
}

// Returns the new heap size (>= 0) or a negative status.
int scan_u8_device(const uint8_t *blocks, int64_t nblocks, const int64_t *ids, int mrows,
                   const uint8_t *qt, float qmin, float delta, const float *heap_d,
                   const int64_t *heap_i, int size, int R, float *out_d, int64_t *out_i,
                   cudaStream_t st) {
  const int64_t lanes = nblocks * 16;
  const int64_t n = lanes + size;
  uint8_t *lane_q = nullptr;
  int *flags = nullptr, *rank = nullptr;
  float *cd = nullptr;
  int64_t *ci = nullptr;
  void *tmp = nullptr;
  size_t tb = 0;
  QADC_CUDA(cudaMallocAsync(&lane_q, std::max<int64_t>(lanes, 1), st));
  QADC_CUDA(cudaMallocAsync(&flags, std::max<int64_t>(lanes, 1) * 4, st));
  QADC_CUDA(cudaMallocAsync(&rank, std::max<int64_t>(lanes, 1) * 4, st));
  QADC_CUDA(cudaMallocAsync(&cd, std::max<int64_t>(n, 1) * 4, st));
  QADC_CUDA(cudaMallocAsync(&ci, std::max<int64_t>(n, 1) * 8, st));
  if (lanes > 0) {
    launch_block_dists(blocks, nblocks, mrows, qt, 0, lane_q, st);
    k_valid_flags<<<grid_for(lanes), 256, 0, st>>>(ids, lanes, flags);
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flags, rank, lanes, st);
    QADC_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), st));
    cub::DeviceScan::ExclusiveSum(tmp, tb, flags, rank, lanes, st);
    k_u8_candidates<<<grid_for(lanes), 256, 0, st>>>(lane_q, ids, rank, lanes, R - size, qmin,
                                                      delta, cd, ci);
  }
  if (size > 0) {
    QADC_CUDA(cudaMemcpyAsync(cd + lanes, heap_d, size * 4, cudaMemcpyDeviceToDevice, st));
    QADC_CUDA(cudaMemcpyAsync(ci + lanes, heap_i, size * 8, cudaMemcpyDeviceToDevice, st));
  }
  int nout = 0;
  int rc = topr_sorted(cd, ci, n, R, out_d, out_i, &nout, st);
  cudaFreeAsync(lane_q, st);
  cudaFreeAsync(flags, st);
  cudaFreeAsync(rank, st);
  cudaFreeAsync(cd, st);
  cudaFreeAsync(ci, st);
  if (tmp) cudaFreeAsync(tmp, st);
  if (rc) return -rc;
  return nout;
}

int adc_f32_device(const uint8_t *codes, int64_t n, const int64_t *ids, int m, int b,
                   const float *tables, const float *heap_d, const int64_t *heap_i, int size, int R,
                   float *out_d, int64_t *out_i, cudaStream_t st) {
  const int64_t tot = n + size;
  float *cd = nullptr;
  int64_t *ci = nullptr;
  QADC_CUDA(cudaMallocAsync(&cd, std::max<int64_t>(tot, 1) * 4, st));
  QADC_CUDA(cudaMallocAsync(&ci, std::max<int64_t>(tot, 1) * 8, st));
  if (n > 0) k_adc_candidates<<<grid_for(n), 256, 0, st>>>(codes, n, ids, m, b, tables, cd, ci);
  if (size > 0) {
    QADC_CUDA(cudaMemcpyAsync(cd + n, heap_d, size * 4, cudaMemcpyDeviceToDevice, st));
    QADC_CUDA(cudaMemcpyAsync(ci + n, heap_i, size * 8, cudaMemcpyDeviceToDevice, st));
  }
  int nout = 0;
  int rc = topr_sorted(cd, ci, tot, R, out_d, out_i, &nout, st);
  cudaFreeAsync(cd, st);
  cudaFreeAsync(ci, st);
  if (rc) return -rc;
  return nout;
}

// Query q of a search batch whose candidates did not fit the shared-memory
// select: gather (candidates with midpoint <= M) U F_sat and radix-sort.
__global__ void k_gather_large(const unsigned *__restrict__ M_bits, const unsigned *__restrict__ cand_n,
                               const float *__restrict__ cand_mid, const int64_t *__restrict__ cand_id,
                               int cap_g, const int *__restrict__ fsat_n,
                               const float *__restrict__ fsat_mid, const int64_t *__restrict__ fsat_id,
                               int q, int R, float *__restrict__ cd, int64_t *__restrict__ ci) {
  const int64_t total = min(cand_n[q], (unsigned)cap_g);
  const int nf = fsat_n[q];
  const float M = __uint_as_float(M_bits[q]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total + nf;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < total) {
      const float d = cand_mid[(size_t)q * cap_g + i];
      const bool ok = d <= M;
      cd[i] = ok ? d : __int_as_float(0x7f800000);
      ci[i] = ok ? cand_id[(size_t)q * cap_g + i] : INT64_MAX;
    } else {
      cd[i] = fsat_mid[(size_t)q * R + (i - total)];
      ci[i] = fsat_id[(size_t)q * R + (i - total)];
    }
  }
}

__global__ void k_write_out(const float *__restrict__ d, const int64_t *__restrict__ id, int nout,
                            int R, int q, int64_t *__restrict__ out_ids, float *__restrict__ out_d,
                            int32_t *__restrict__ out_n) {
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    out_ids[(size_t)q * R + i] = i < nout ? id[i] : -1;
    out_d[(size_t)q * R + i] = i < nout ? d[i] : __int_as_float(0x7f800000);
  }
  if (threadIdx.x == 0) out_n[q] = nout;
}

int select_large(int q, int R, const unsigned *M_bits, const unsigned *cand_n,
                 const float *cand_mid, const int64_t *cand_id, int cap_g, const int *fsat_n,
                 const float *fsat_mid, const int64_t *fsat_id, int64_t *out_ids, float *out_d,
                 int32_t *out_n, cudaStream_t st) {
  unsigned h_n = 0;
  int h_f = 0;
  QADC_CUDA(cudaMemcpyAsync(&h_n, cand_n + q, 4, cudaMemcpyDeviceToHost, st));
  QADC_CUDA(cudaMemcpyAsync(&h_f, fsat_n + q, 4, cudaMemcpyDeviceToHost, st));
  QADC_CUDA(cudaStreamSynchronize(st));
  const int64_t n = (int64_t)std::min<unsigned>(h_n, (unsigned)cap_g) + h_f;
  float *cd = nullptr, *od = nullptr;
  int64_t *ci = nullptr, *oi = nullptr;
  QADC_CUDA(cudaMallocAsync(&cd, std::max<int64_t>(n, 1) * 4, st));
  QADC_CUDA(cudaMallocAsync(&ci, std::max<int64_t>(n, 1) * 8, st));
  QADC_CUDA(cudaMallocAsync(&od, (size_t)R * 4, st));
  QADC_CUDA(cudaMallocAsync(&oi, (size_t)R * 8, st));
  k_gather_large<<<grid_for(n), 256, 0, st>>>(M_bits, cand_n, cand_mid, cand_id, cap_g, fsat_n,
                                               fsat_mid, fsat_id, q, R, cd, ci);
  int nout = 0;
  int rc = topr_sorted(cd, ci, n, R, od, oi, &nout, st);
  if (rc == kOk) k_write_out<<<1, 256, 0, st>>>(od, oi, nout, R, q, out_ids, out_d, out_n);
  cudaFreeAsync(cd, st);
  cudaFreeAsync(ci, st);
  cudaFreeAsync(od, st);
  cudaFreeAsync(oi, st);
  return rc;
}

}  // namespace qadc
