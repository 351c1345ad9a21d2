// Index layout: repack reference lists into the interleaved32 HBM layout.
//
// Input layouts (reference):
//   * transposed16 blocks (qadc.py:27-51, 96-113): (nblocks, m/2, 16) bytes,
//     row j byte l = sub-codes (2j, 2j+1) of code l, low nibble first
//     (pack_codes nibble order, pq.py:90-105); ids 16 per block, -1 padding;
//   * packed code rows (pq.py:90-105): (n, m/2) bytes per list.
// Output: see internal.cuh (interleaved32 + validity + padded ids).
#include <algorithm>
#include <mutex>

#include "internal.cuh"

namespace qadc {
namespace {

// One thread per output word (chunk g, sub-quantizer j, octet o).
template <bool FROM_ROWS>
__global__ void k_pack(const uint8_t *__restrict__ src, const int64_t *__restrict__ src_off,
                       const int64_t *__restrict__ src_ids, const int32_t *__restrict__ chunk_list,
                       const int64_t *__restrict__ chunk_off, const int64_t *__restrict__ lanes,
                       int m, int64_t total_chunks, uint32_t *__restrict__ codes) {
  const int64_t words = total_chunks * m * 32;
  const int mrows = m / 2;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int o = (int)(w & 31);
    const int j = (int)((w >> 5) % m);
    const int64_t g = w / (32 * (int64_t)m);
    const int L = chunk_list[g];
    const int64_t c = g - chunk_off[L];
    const int64_t n = lanes[L];
    uint32_t word = 0;
#pragma unroll
    for (int p = 0; p < 8; p++) {
      const int64_t k = c * kChunkCodes + 8 * o + p;
      if (k >= n) continue;
      uint8_t byte;
      if (FROM_ROWS) {
        byte = src[(src_off[L] + k) * mrows + (j >> 1)];
      } else {
        byte = src[((src_off[L] + k / 16) * mrows + (j >> 1)) * 16 + (k & 15)];
      }
      const uint32_t nib = (j & 1) ? (byte >> 4) : (byte & 15);
      word |= nib << (4 * p);
    }
    codes[w] = word;
  }
}

// One thread per code slot: padded ids and validity bits.
template <bool FROM_ROWS>
__global__ void k_ids(const int64_t *__restrict__ src_off, const int64_t *__restrict__ src_ids,
                      const int32_t *__restrict__ chunk_list, const int64_t *__restrict__ chunk_off,
                      const int64_t *__restrict__ lanes, int64_t total_chunks,
                      int64_t *__restrict__ ids, uint8_t *__restrict__ valid) {
  const int64_t slots = total_chunks * kChunkCodes;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < slots;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = s / kChunkCodes;
    const int L = chunk_list[g];
    const int64_t k = (g - chunk_off[L]) * kChunkCodes + (s % kChunkCodes);
    int64_t id = -1;
    if (k < lanes[L]) {
      if (FROM_ROWS)
        id = src_ids ? src_ids[src_off[L] + k] : (src_off[L] + k);
      else
        id = src_ids[src_off[L] * 16 + k];
    }
    ids[s] = id;
    // validity byte per octet: lanes of one octet are 8 consecutive
    // threads of one warp; gather with a ballot.
    const unsigned bal = __ballot_sync(0xffffffffu, id >= 0);
    const int lane = threadIdx.x & 31;
    if ((lane & 7) == 0) valid[s / 8] = (uint8_t)((bal >> (lane & 24)) & 0xff);
  }
}

__global__ void k_chunk_list(const int64_t *__restrict__ chunk_off, int nlists,
                             int32_t *__restrict__ chunk_list) {
  for (int L = blockIdx.x * blockDim.x + threadIdx.x; L < nlists; L += gridDim.x * blockDim.x)
    for (int64_t g = chunk_off[L]; g < chunk_off[L + 1]; g++) chunk_list[g] = L;
}

// One thread per (code slot, word i): gathers sub-codes 8i..8i+7 of the code
// from the interleaved words.
__global__ void k_code_major(const uint32_t *__restrict__ codes, int m, int64_t total_chunks,
                             uint32_t *__restrict__ out) {
  const int wpc = m / 8;
  const int64_t n = total_chunks * kChunkCodes * wpc;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % wpc);
    const int64_t slot = t / wpc;
    const int64_t g = slot / kChunkCodes;
    const int c = (int)(slot % kChunkCodes);
    const uint32_t *src = codes + ((size_t)g * m + 8 * i) * 32 + (c >> 3);
    const int sh = 4 * (c & 7);
    uint32_t w = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) w |= ((src[k * 32] >> sh) & 15u) << (4 * k);
    out[t] = w;
  }
}

int common_alloc(qadc_b200_index *idx, cudaStream_t st) {
  const int64_t tc = idx->total_chunks;
  // one chunk of zeroed padding: the scan's linear prefetch reads up to 12
  // rows past the last chunk it scans
  const size_t chunk_bytes = (size_t)idx->m * 32 * 4;
  QADC_CUDA(cudaMalloc(&idx->codes, (size_t)(std::max<int64_t>(tc, 1) + 1) * chunk_bytes));
  QADC_CUDA(cudaMemsetAsync((char *)idx->codes + (size_t)std::max<int64_t>(tc, 1) * chunk_bytes, 0,
                            chunk_bytes, st));
  QADC_CUDA(cudaMalloc(&idx->valid, (size_t)std::max<int64_t>(tc, 1) * 32));
  QADC_CUDA(cudaMalloc(&idx->ids, (size_t)std::max<int64_t>(tc, 1) * kChunkCodes * 8));
  QADC_CUDA(cudaMalloc(&idx->chunk_list, (size_t)std::max<int64_t>(tc, 1) * 4));
  idx->bytes += tc * idx->m * 128 + tc * 32 + tc * kChunkCodes * 8 + tc * 4;
  k_chunk_list<<<(idx->nlists + 255) / 256, 256, 0, st>>>(idx->chunk_off, idx->nlists,
                                                         idx->chunk_list);
  return kOk;
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)std::min<int64_t>(std::max<int64_t>(g, 1), 148 * 64);
}

}  // namespace

// ids are 16 per block (reference transposed layout), device pointers.
int pack_from_blocks(qadc_b200_index *idx, const uint8_t *d_blocks,
                     const int64_t *d_blk_off, const int64_t *d_ids, cudaStream_t st) {
  int rc = common_alloc(idx, st);
  if (rc) return rc;
  const int64_t tc = idx->total_chunks;
  if (tc == 0) return kOk;
  k_pack<false><<<grid_for(tc * idx->m * 32), 256, 0, st>>>(
      d_blocks, d_blk_off, d_ids, idx->chunk_list, idx->chunk_off, idx->lanes, idx->m, tc,
      idx->codes);
  k_ids<false><<<grid_for(tc * kChunkCodes), 256, 0, st>>>(
      d_blk_off, d_ids, idx->chunk_list, idx->chunk_off, idx->lanes, tc, idx->ids, idx->valid);
  QADC_CUDA(cudaGetLastError());
  return kOk;
}

int ensure_code_major(qadc_b200_index *idx, cudaStream_t st) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (idx->codes_cm) return kOk;
  if (idx->m % 8) {
    set_error("code-major copy needs m % 8 == 0");
    return kErrArgs;
  }
  const int64_t tc = std::max<int64_t>(idx->total_chunks, 1);
  const size_t bytes = (size_t)tc * kChunkCodes * (idx->m / 8) * 4;
  uint32_t *p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    set_error("code-major copy of the codes: out of device memory");
    return kErrCuda;
  }
  if (idx->total_chunks > 0)
    k_code_major<<<grid_for(idx->total_chunks * kChunkCodes * (idx->m / 8)), 256, 0, st>>>(
        idx->codes, idx->m, idx->total_chunks, p);
  else
    cudaMemsetAsync(p, 0, bytes, st);
  QADC_CUDA(cudaGetLastError());
  // one-time: the copy is complete before any stream can see the pointer
  QADC_CUDA(cudaStreamSynchronize(st));
  idx->codes_cm = p;
  idx->bytes += (int64_t)bytes;
  return kOk;
}

int pack_from_rows(qadc_b200_index *idx, const uint8_t *d_rows, const int64_t *d_row_off,
                   const int64_t *d_ids, cudaStream_t st) {
  int rc = common_alloc(idx, st);
  if (rc) return rc;
  const int64_t tc = idx->total_chunks;
  if (tc == 0) return kOk;
  k_pack<true><<<grid_for(tc * idx->m * 32), 256, 0, st>>>(
      d_rows, d_row_off, d_ids, idx->chunk_list, idx->chunk_off, idx->lanes, idx->m, tc,
      idx->codes);
  k_ids<true><<<grid_for(tc * kChunkCodes), 256, 0, st>>>(
      d_row_off, d_ids, idx->chunk_list, idx->chunk_off, idx->lanes, tc, idx->ids, idx->valid);
  QADC_CUDA(cudaGetLastError());
  return kOk;
}

}  // namespace qadc
