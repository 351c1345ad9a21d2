// Internal declarations shared by the qadc_b200 translation units.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "qadc_common.cuh"

// Device-resident index (the opaque qadc_b200_index of the C ABI).
//
// Data layout in HBM ("interleaved32"): every list is padded to whole
// chunks of 256 codes; chunk g holds m x 32 uint32 words, word (j, o) =
// 4-bit sub-code j of codes 8o..8o+7 of the chunk, code 8o+k at bits
// 4k..4k+3. A warp reads one 128-byte row per sub-quantizer (coalesced)
// and each word's low / high 16 bits are ready-made PRMT selectors for
// four codes. valid[g][o] bit k flags code 8o+k as admissible (id >= 0).
struct qadc_b200_index {
  int d = 0, m = 0, dsub = 0, nlists = 0, K = 0;
  int64_t total_chunks = 0;
  int64_t max_list_chunks = 0;
  float *coarse = nullptr;     // [K][d]
  float *coarseT = nullptr;    // [d][K] (coalesced probe reads)
  float *cnorm = nullptr;      // [K] |c|^2 (probe pre-selection bounds)
  float *pmu = nullptr;        // [d] centroid mean (tensor-core probe centring)
  void *pcsplit = nullptr;     // [K_pad][3d] bf16 centred split rows [hi | lo | hi], tiled
  float *pcn2 = nullptr;       // [K] |c - mu|^2
  float *codebooks = nullptr;  // [m][16][dsub]
  float *rotation = nullptr;   // [d][d] or null
  float *rotationT = nullptr;  // [d][d] R^T (coalesced float4 rows for the residual rotation)
  uint32_t *codes = nullptr;   // [total_chunks][m][32]
  // Code-major copy for the one-SM tensor-core scan (built on first use,
  // ensure_code_major): [total_chunks * 256][m / 8] words, word i of a code
  // = its sub-codes 8i..8i+7, sub-code 8i+k at bits 4k..4k+3 (each 16-bit
  // half is a PRMT selector over four sub-quantizers of ONE code).
  uint32_t *codes_cm = nullptr;
  uint8_t *valid = nullptr;    // [total_chunks][32]
  int64_t *ids = nullptr;      // [total_chunks * 256], -1 padding
  int32_t *chunk_list = nullptr;  // [total_chunks] owning list
  int64_t *chunk_off = nullptr;   // [nlists + 1]
  int64_t *lanes = nullptr;       // [nlists] lanes in layout (16 * nblocks)
  int64_t *count = nullptr;       // [nlists] GLOBAL code count (find_qmax prefix)
  int64_t *scan_count = nullptr;  // [nlists] codes in this index's scan region
  // Prefix region read by find_qmax / F_sat / the initial bound. By default
  // it aliases the scan region; a shard of a distributed index stores the
  // global list prefixes here (qadc_b200_index_set_prefix_device).
  uint32_t *pcodes = nullptr;
  int64_t *pids = nullptr;
  int64_t *pchunk_off = nullptr;
  int64_t *planes = nullptr;
  bool own_prefix = false;
  std::vector<int64_t> h_chunk_off, h_lanes, h_count;
  int64_t bytes = 0;
};

namespace qadc {

void set_error(const std::string &msg);
int cuda_fail(cudaError_t e, const char *where);
#define QADC_CUDA(call)                                   \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);   \
  } while (0)

// ---- layout.cu ----
int pack_from_blocks(qadc_b200_index *idx, const uint8_t *d_blocks,
                     const int64_t *d_blk_off, const int64_t *d_ids,
                     cudaStream_t st);
int pack_from_rows(qadc_b200_index *idx, const uint8_t *d_rows,
                   const int64_t *d_row_off, const int64_t *d_ids,
                   cudaStream_t st);
// Builds idx->codes_cm from the interleaved codes if absent (m % 8 == 0).
int ensure_code_major(qadc_b200_index *idx, cudaStream_t st);

// ---- lut.cu ----
void launch_compute_tables(const float *codebooks, int m, int dsub,
                           const float *y, int npairs, float *out, cudaStream_t st);
void launch_probe(const float *coarseT, int K, int d, const float *queries,
                  int nq, int ma, int64_t *cells, cudaStream_t st);
void launch_cnorm(const float *coarse, int K, int d, float *cn, cudaStream_t st);
// FFMA pre-selection + exact re-rank probe; false = not applicable (caller
// uses launch_probe).
bool launch_probe_fast(const float *coarseT, const float *coarse, const float *cn, int K, int d,
                       const float *queries, int nq, int ma, int64_t *cells, cudaStream_t st);
// ---- probe_tc.cu ----
// Fused tcgen05 probe: split-bf16 GEMM with on-the-fly candidate selection
// + exact einsum re-rank (supported: K >= 256, d % 64 == 0, d <= 128,
// ma <= 64); false = not applicable (callers use launch_probe_fast).
bool probe_tc_supported(int K, int d, int ma);
int probe_tc_prepare(const float *coarse, int K, int d, float **mu, void **ctiled, float **cn2,
                     cudaStream_t st);
bool launch_probe_tc(const float *coarse, const float *mu, const void *ctiled, const float *cn2,
                     int K, int d, const float *queries, int nq, int ma, int64_t *cells,
                     cudaStream_t st, float *dbg_S = nullptr, int *dbg_counts = nullptr);
void launch_residual_lut(const qadc_b200_index *idx, const float *queries,
                         const int64_t *cells, int nq, int nslots,
                         float *lut, cudaStream_t st);
int launch_qmax(const qadc_b200_index *idx, const float *lut,
                 const int64_t *cells, int nq, int nslots, int R, int init,
                 float *qmax, cudaStream_t st);
void launch_quantize(const float *lut, int npairs, int m, const float *qmax_per_query,
                     int nslots, const double *qmin_in, const double *qmax_in,
                     uint32_t *qt, float *qmin_f, float *delta_f,
                     double *delta_out, uint8_t *qt_bytes_out, cudaStream_t st,
                     int max_depth = 16, uint8_t *pair_depth = nullptr);
void launch_prefix(const qadc_b200_index *idx, const uint32_t *qt,
                   const float *qmin_f, const float *delta_f,
                   const int64_t *cells, int nq, int nslots, int R, int init,
                   unsigned *M_bits, int *fsat_n, float *fsat_mid,
                   int64_t *fsat_id, cudaStream_t st);

// ---- scan.cu ----
struct WorkItem {
  int32_t list;
  int32_t pair_begin;   // index into the list-grouped pair arrays
  int32_t pair_count;   // <= QT
  int32_t variant;      // depth | half << 8 | class << 16 (order_items)
  int64_t chunk_begin;  // absolute chunk index
  int64_t chunk_end;
};

struct ScanArgs {
  const uint32_t *codes;
  const uint32_t *codes_cm;  // code-major copy (k_scan_tc only; may be null otherwise)
  const uint8_t *valid;
  const int64_t *ids;
  const WorkItem *items;
  const int *n_items;
  int *item_counter;
  const int32_t *pair_q;   // grouped pairs: query index
  const int32_t *pair_t;   // grouped pairs: table index (q * nslots + s)
  const uint32_t *qt;      // [npairs][m][4] words
  const float *qmin_f;     // [npairs]
  const float *delta_f;    // [npairs]
  unsigned *M_bits;        // [nq] running distance bound
  unsigned *cand_n;        // [nq]
  float *cand_mid;         // [nq][cap_g]
  int64_t *cand_id;        // [nq][cap_g]
  unsigned *hist;          // [nq][kHistWords] midpoint histogram of appended candidates
  const float *hist_w;     // [nq] bucket width (0 disables)
  int cap_g;
  int cap_l;               // per-warp per-query buffer capacity
  int m;
  int R;
  int bound_every;         // appended candidates between global-histogram bound reads
  int linear;              // 1: linear fixed-m loop (long items), 0: interleaved loop
  int tcw;                 // 1: warpgroup-pipelined tensor-core scan for lists with few queries (k_scan_tcw)
  int pair_cta;            // tensor-core scan on CTA pairs (static item order): 1 k_scan_tc2 (flusher rings), 2 k_scan_tc2i (inline survivors)
  int dbg;                 // timing experiments only (QADC_B200_TC_DEBUG; results invalid if != 0)
};

constexpr int kHistBins = 1024;                 // 32 coarse x 32 fine
constexpr int kHistWords = kHistBins + 32;      // fine bins, then coarse sums
int scan_qt_per_cta(int m);
// Tensor-core scan in use for this m; queries per work item of the scan.
// prmt: the caller asked for the PRMT kernel (QADC_B200_SCAN_PRMT).
bool scan_use_tc(int m, bool prmt);
void tc_stats_dump();  // debug counters of the tensor-core scan (QADC_B200_TC_DEBUG & 64)
int scan_tile_queries(int m, bool prmt, bool tcw = false);
// Resident scan CTAs on the device (occupancy x SMs) for this shape.
int scan_resident_ctas(int m, int cap_l, int nsm, int linear, bool prmt);
int scan_env_int(const char *name, int dflt);
void launch_scan(const ScanArgs &a, int nsm, cudaStream_t st, bool prmt);
// Work-list construction (device side). scratch: build_work_scratch ints.
int64_t build_work_scratch(int nlists, int nslots);
int64_t build_work(const qadc_b200_index *idx, const int64_t *cells, int nq,
                   int nslots, int qt_tile, int64_t range_chunks,
                   int32_t *pair_q, int32_t *pair_t, WorkItem *items,
                   int *n_items, int *scratch_list_pairs, int64_t max_items,
                   cudaStream_t st);

// Tag every item with its scan loop variant (byte-sum depth = min over its
// pairs' depth, half tile or not) and reorder items class by class, so the
// CTAs running at any moment share one loop body (instruction cache).
// scratch: order_items_scratch(max_items) unsigned, [0, 8) = items per
// class afterwards. qh: pair_count <= qh runs the half loop.
int64_t order_items_scratch(int64_t max_items);
void order_items(const WorkItem *items, const int *n_items, int64_t max_items,
                 const int32_t *pair_t, const uint8_t *pair_depth, int qh, int nslots,
                 unsigned *scratch, WorkItem *out, cudaStream_t st);

// ---- select.cu ----
int select_capacity();
void launch_select(int nq, int R, const unsigned *M_bits, const unsigned *cand_n,
                   const float *cand_mid, const int64_t *cand_id, int cap_g,
                   const int *fsat_n, const float *fsat_mid, const int64_t *fsat_id,
                   int64_t *out_ids, float *out_d, int32_t *out_n,
                   int *overflow, cudaStream_t st);

// ---- simple.cu (general-table engine, reference layout) ----
void launch_block_dists(const uint8_t *blocks, int64_t nblocks, int mrows,
                        const uint8_t *qt, int per_block, uint8_t *out,
                        cudaStream_t st);
// Exact top-R by (dist, id) of n (dist, id) pairs (device), pairs with
// id == INT64_MAX are padding. Writes up to R results ascending to
// out_d/out_i (device) and returns the count via *out_n (host).
int topr_sorted(const float *d, const int64_t *id, int64_t n, int R, float *out_d,
                int64_t *out_i, int *out_n, cudaStream_t st);
// Reference-ABI scans on device buffers (simple.cu).
int scan_u8_device(const uint8_t *blocks, int64_t nblocks, const int64_t *ids, int mrows,
                   const uint8_t *qt, float qmin, float delta, const float *heap_d,
                   const int64_t *heap_i, int size, int R, float *out_d, int64_t *out_i,
                   cudaStream_t st);
int adc_f32_device(const uint8_t *codes, int64_t n, const int64_t *ids, int m, int b,
                   const float *tables, const float *heap_d, const int64_t *heap_i, int size,
                   int R, float *out_d, int64_t *out_i, cudaStream_t st);
// Large-candidate fallback for search_batch queries that overflowed the
// shared-memory select (massive ties): exact top-R via device radix sort.
int select_large(int q, int R, const unsigned *M_bits, const unsigned *cand_n,
                 const float *cand_mid, const int64_t *cand_id, int cap_g, const int *fsat_n,
                 const float *fsat_mid, const int64_t *fsat_id, int64_t *out_ids, float *out_d,
                 int32_t *out_n, cudaStream_t st);

}  // namespace qadc
