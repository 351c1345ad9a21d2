/*
 * qadc_b200 — B200-native (sm_100a) Quick ADC search path, C ABI.
 *
 * Drop-in boundary for the reference package `qadc` (arXiv 1704.07355,
 * /root/reference/pkg). Paths below are relative to /root/reference/pkg/src/qadc/.
 *
 * Part 1 replaces the reference's native kernel ABI one-for-one
 * (src/scan_kernels.h:15-46, bound by _kernels.pyx:33-152): same names,
 * same argument meaning, HOST pointers, caller-owned buffers. Each call
 * stages its inputs to the current CUDA device, runs the sm_100a kernels,
 * and copies the results back. The reference has no error path; here an
 * int-returning entry point returns -1 on failure and
 * qadc_b200_last_error() explains why.
 *
 * Part 2 is the batched, device-resident interface a B200 caller wants
 * (the reference has no batched API; bench.py:182-191 loops over queries):
 * an index uploaded once into the interleaved HBM layout, and
 * search_batch over Q queries in one stream-ordered call.
 *
 * All entry points are plain C: pointers, sizes, and an opaque handle.
 */
#ifndef QADC_B200_H
#define QADC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define QADC_API __attribute__((visibility("default")))
#else
#define QADC_API
#endif

/* ---- reference kernel variant ids (scan_kernels.h:7-9) plus ours ---- */
#define QADC_KERNEL_SCALAR 0
#define QADC_KERNEL_SIMD128 1
#define QADC_KERNEL_SIMD256 2
#define QADC_KERNEL_B200 3
#define QADC_MAX_M 128 /* scan_kernels.h:12 */

/* ======================= Part 1: reference ABI ======================== */

/* Replaces qadc_simd_level (scan_kernels.h:15, scan_kernels.c:11-20):
 * QADC_KERNEL_B200 when an sm_100 device is usable, else -1. */
QADC_API int qadc_simd_level(void);

/* Replaces adc_scan_f32 (scan_kernels.h:24-26, scan_kernels.c:78-125):
 * float ADC scan of n packed codes (b = 4, 8, 16), merging the best into
 * the caller's (hd, hi) max-heap of capacity R holding `size` entries.
 * Returns the new size (-1 on error). On return the heap arrays hold the
 * same multiset the reference leaves, arranged as a valid max-heap
 * (descending (dist, id) order). */
QADC_API int adc_scan_f32(const uint8_t *codes, int64_t n, const int64_t *ids,
                 int m, int b, const float *tables,
                 float *hd, int64_t *hi, int size, int R);

/* Replaces qadc_scan_u8 (scan_kernels.h:35-37, scan_kernels.c:362-382):
 * quantized scan of a transposed (nblocks, mrows, 16) list; lanes enter
 * with qmin + (q + 0.5) * delta; padding (id < 0) never; saturated lanes
 * only while the heap is below capacity. `variant` is accepted for ABI
 * compatibility and ignored (there is one B200 kernel). Returns the new
 * heap size (-1 on error). */
QADC_API int qadc_scan_u8(const uint8_t *blocks, int64_t nblocks, const int64_t *ids,
                 int mrows, const uint8_t *qt, float qmin, float delta,
                 float *hd, int64_t *hi, int size, int R, int variant);

/* Replaces qadc_block_dists (scan_kernels.h:43-45, scan_kernels.c:384-419):
 * saturated lane sums, one 16-byte row per block; per_block != 0 means qt
 * holds one (2*mrows, 16) table set per block. Table bytes may be 0..255. */
QADC_API void qadc_block_dists(const uint8_t *blocks, int64_t nblocks, int mrows,
                      const uint8_t *qt, int per_block, uint8_t *out,
                      int variant);

/* ====================== Part 2: batched B200 API ====================== */

/* Last error message of this thread ("" if none). */
QADC_API const char *qadc_b200_last_error(void);

/* Opaque device-resident index: coarse centroids (IVF) or none (flat),
 * the product quantizer, and every inverted list repacked into the
 * interleaved layout. */
typedef struct qadc_b200_index qadc_b200_index;

/*
 * Build a device index from reference-layout lists (ivf.py:40-93,
 * qadc.py:27-51): `blocks` concatenates every list's transposed
 * (nblocks_c, m/2, 16) bytes; list c spans blocks [blk_off[c],
 * blk_off[c+1]) and ids [16*blk_off[c], 16*blk_off[c+1]) with count[c]
 * valid codes. coarse (K x d, row-major) is NULL for a flat index (then
 * nlists must be 1). codebooks is the (m, 16, d/m) PQ codebook array and
 * rotation the optional (d, d) OPQ matrix (pq.py:25-62). All pointers are
 * HOST pointers; the data is copied to the current device.
 */
QADC_API int qadc_b200_index_create(int d, int m, int nlists, const float *coarse,
                           const uint8_t *blocks, const int64_t *blk_off,
                           const int64_t *ids, const int64_t *count,
                           const float *codebooks, const float *rotation,
                           qadc_b200_index **out);

/*
 * Build a device index from packed code rows that are ALREADY on the
 * device (e.g. produced by a GPU encoder): `codes` is (n, m/2) packed
 * rows (pq.py:90-105 nibble order) in list order, list c owning rows
 * [row_off[c], row_off[c+1]); ids (n,) int64 device array, or NULL for
 * ids = row index. coarse/codebooks/rotation are DEVICE pointers here.
 */
QADC_API int qadc_b200_index_create_device(int d, int m, int nlists,
                                  const float *coarse, const uint8_t *codes,
                                  const int64_t *row_off, const int64_t *ids,
                                  const float *codebooks,
                                  const float *rotation,
                                  qadc_b200_index **out);

QADC_API void qadc_b200_index_destroy(qadc_b200_index *idx);

/*
 * Shard support: replace the index's prefix region — the codes
 * find_qmax (qadc.py:157-194), the first-R-valid saturation rule and the
 * initial bound read — by the GLOBAL first codes of each list, so a shard
 * that scans only part of a list still reproduces the single-index
 * semantics. rows (n, m/2) / row_off (nlists + 1) / ids (n or NULL) are
 * device arrays like qadc_b200_index_create_device's; full_count (nlists,
 * host) is each list's global code count.
 */
QADC_API int qadc_b200_index_set_prefix_device(qadc_b200_index *idx,
                                               const uint8_t *rows,
                                               const int64_t *row_off,
                                               const int64_t *ids,
                                               const int64_t *full_count);

/* Device bytes held by the index (codes, ids, validity, centroids). */
QADC_API int64_t qadc_b200_index_bytes(const qadc_b200_index *idx);

/* Flags for qadc_b200_search_batch. */
#define QADC_B200_HOST_IO 1u   /* queries / outputs are host pointers */
#define QADC_B200_LUT_IN 2u    /* lut_in / cells_in supplied (device) */
#define QADC_B200_NO_FSAT 4u   /* leave the saturated first-R lanes out (every
                                  shard but the owner of the global prefix) */
#define QADC_B200_SCAN_PRMT 8u /* scan with the PRMT (CUDA-core) kernel even
                                  where the tensor-core scan applies */
#define QADC_B200_SCAN_TC 16u  /* the all-warps-on-one-tile tensor-core scan
                                  (m = 16, 32; up to 256 queries per pass)
                                  whatever the batch */
#define QADC_B200_SCAN_TC1 32u /* with the tensor-core scan of one exhaustive
                                  list: one SM per tile instead of CTA pairs
                                  (cta_group::2, the default) */
#define QADC_B200_SCAN_TCW 64u /* IVF index, m = 16, 32: the warpgroup-
                                  pipelined tensor-core scan (<= 32 queries
                                  per pass over a list) whatever the batch;
                                  default: from ~4 queries per probed list */

/*
 * adc.py:114-187 search(method="qadc") for nq queries at once:
 * probe (IVF) -> residual, rotation, float LUT -> qmax from the first
 * probed cell's first `init` codes -> per-cell qmin/delta and uint8 LUT ->
 * scan with streaming thresholds (int8 tcgen05 one-hot GEMM for m = 16, 32:
 * CTA pairs on an exhaustive list, warpgroup-pipelined passes of <= 32 queries
 * over inverted lists; interleaved PRMT lookups otherwise) -> exact top-R by
 * (distance, id). Outputs (nq, R) ids / fp32 midpoint distances sorted
 * ascending, padded with -1 / +inf, and out_n (nq) = result count.
 * With QADC_B200_LUT_IN, lut_in (nq, ma, m, 16) fp32 and cells_in (nq, ma)
 * replace the probe and table phases ("reference-LUT-injected" mode).
 * stream is a cudaStream_t (NULL = legacy default stream).
 * stats (optional, 16 int64): [0] codes scanned, [1] scan candidates,
 * [2] overflow reruns, [3] scan kernel launches, [4] total kernel launches,
 * [5] scan kernel microseconds (event timed), [6] 1 if the scan ran on the
 * tensor cores, then event-timed microseconds of the other phases of the
 * first pass (adc.py:140-179's Index / Tables / Scan split): [7] probe,
 * [8] tables (residual, rotation, LUT, qmax, quantize, prefix facts),
 * [9] work list, [10] exact top-R select; [11..15] reserved (0).
 */
QADC_API int qadc_b200_search_batch(qadc_b200_index *idx, const float *queries,
                           int nq, int R, int ma, int init, unsigned flags,
                           const float *lut_in, const int64_t *cells_in,
                           int64_t *out_ids, float *out_d, int32_t *out_n,
                           void *stream, int64_t *stats);

/*
 * search_batch in two halves, for callers that move the per-query state
 * between them (the query-sharded Tables phase of a multi-GPU search:
 * every rank prepares a slice of the batch, the slices are all-gathered,
 * then every rank scans its own codes for the whole batch). Device
 * pointers only; npairs = nq * (ma for IVF, 1 for a flat index).
 *
 * prepare = the Index + Tables phases (adc.py:140-174): cells (npairs)
 * int64 probe order (IVF; ignored for a flat index), qt (npairs * m * 4)
 * uint32 words of the uint8 tables (entries 4w..4w+3 of sub-quantizer
 * w / 4), qmin_f / delta_f (npairs) fp32, depth (npairs) uint8 byte-sum
 * depth, qmax (nq) fp32, M_bits (nq) uint32 initial distance bound
 * (float bits), fsat_n (nq) int32 / fsat_mid (nq * R) fp32 / fsat_id
 * (nq * R) int64 the saturated first-R lanes (QADC_B200_NO_FSAT: none).
 * With QADC_B200_LUT_IN, lut_in / cells_in replace the probe and LUT.
 *
 * scan = work list, scan, exact top-R over those arrays (M_bits is
 * tightened in place); outputs as search_batch. stats as search_batch
 * (each call fills the phases it ran).
 */
QADC_API int qadc_b200_search_prepare(qadc_b200_index *idx, const float *queries, int nq,
                                      int R, int ma, int init, unsigned flags,
                                      const float *lut_in, const int64_t *cells_in,
                                      int64_t *cells, uint32_t *qt, float *qmin_f,
                                      float *delta_f, uint8_t *depth, float *qmax,
                                      uint32_t *M_bits, int32_t *fsat_n, float *fsat_mid,
                                      int64_t *fsat_id, void *stream, int64_t *stats);
QADC_API int qadc_b200_search_scan(qadc_b200_index *idx, int nq, int R, int ma, int init,
                                   unsigned flags, const int64_t *cells, const uint32_t *qt,
                                   const float *qmin_f, const float *delta_f,
                                   const uint8_t *depth, uint32_t *M_bits,
                                   const int32_t *fsat_n, const float *fsat_mid,
                                   const int64_t *fsat_id, int64_t *out_ids, float *out_d,
                                   int32_t *out_n, void *stream, int64_t *stats);

/* ---- device-pointer building blocks (parity tests, diagnostics) ---- */

/* The Index + Tables phases of search_batch (adc.py:140-174) with their
 * intermediates, for parity accounting of native mode: cells_out (nq, ma)
 * int64 (IVF; ignored for a flat index), lut_out (nq, ma, m, 16) fp32
 * (residual, OPQ rotation, compute_tables), qmax_out (nq) fp32 (find_qmax
 * on the first probed cell), qt_out (nq, ma, m, 16) uint8
 * (quantize_tables), qmin_out / delta_out (nq, ma) the fp32 casts the scan
 * uses. Device pointers; ma is 1 for a flat index. */
QADC_API int qadc_b200_search_tables(qadc_b200_index *idx, const float *queries, int nq,
                                     int R, int ma, int init, int64_t *cells_out,
                                     float *lut_out, float *qmax_out, uint8_t *qt_out,
                                     float *qmin_out, float *delta_out, void *stream);

/* adc.py:61-75 compute_tables for npairs residual queries y (npairs, d):
 * out (npairs, m, 16) fp32, NumPy einsum summation order. */
QADC_API int qadc_b200_compute_tables(const float *codebooks, int m, int dsub,
                             const float *y, int npairs, float *out,
                             void *stream);

/* ivf.py:166-182 probe for nq queries: cells (nq, ma) int64 and residual
 * queries (nq, ma, d) fp32. coarse is (K, d) row-major, device. */
QADC_API int qadc_b200_probe(const float *coarse, int K, int d, const float *queries,
                    int nq, int ma, int64_t *cells, float *residuals,
                    void *stream);

/* qadc.py:124-147 quantize_tables for npairs (m, 16) fp32 tables with
 * per-pair qmin / qmax (float64): out (npairs, m, 16) uint8 and
 * delta (npairs) float64. */
QADC_API int qadc_b200_quantize_tables(const float *tables, int npairs, int m,
                              const double *qmin, const double *qmax,
                              uint8_t *out, double *delta, void *stream);

/* ---- GPU index build, device pointers ---- */

/* pq.py:210-217 encode_batch: rows of X (n, d) fp32 -> packed codes
 * (n, m/2) uint8, low nibble = even sub-code (pq.py:90-105). Optional
 * rotation (d, d) is applied first (x @ R^T). Per sub-space argmin of the
 * einsum-order squared distance, ties to the lowest index
 * (kmeans.py:52-78). */
QADC_API int qadc_b200_encode(const float *X, int64_t n, int d, int m,
                     const float *codebooks, const float *rotation,
                     uint8_t *out, void *stream);

/* Integer issue-rate microbenchmark (roofline denominator R_int): out[0]
 * = sustained PRMT+IMAD lane-instructions/s (both integer-capable pipes),
 * out[1] = PRMT-only (ALU pipe) lane-instructions/s, on this device. */
QADC_API int qadc_b200_int_peak(double *out);

/* int8 tensor-core microbenchmark (roofline denominator of the tensor-core
 * scan): out[0] = dense tcgen05.mma.kind::i8 ops/s (2 per MAC; M=128,
 * N=256, K=32 instructions, one CTA per SM) on this device. */
QADC_API int qadc_b200_mma_peak(double *out);

/* Diagnostics of the fused tensor-core probe (probe_tc.cu), device
 * pointers: cells (nq, ma); S (128 x 256 fp32) = the raw split-bf16 dot
 * products of the first CTA's first centroid tile; counts = [slices, then
 * per-(slice, query) candidate counts]; mu_out (d) = the centring mean. */
QADC_API int qadc_b200_debug_probe_tc(const float *coarse, int K, int d, const float *queries,
                                      int nq, int ma, int64_t *cells, float *S, int *counts,
                                      float *mu_out, void *stream);

/* kmeans.py:52-78 assign_batch: nearest of K centroids (K, d) per row of
 * X (n, d), einsum-order distances, ties to the lowest index. */
QADC_API int qadc_b200_assign(const float *X, int64_t n, int d, const float *C,
                     int K, int64_t *labels, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* QADC_B200_H */
