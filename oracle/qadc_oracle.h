/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's Quick ADC
 * search path (arXiv 1704.07355 reference package `qadc`, /root/reference/pkg).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as the checker or the timed CPU
 * baseline — never as part of the product path.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/pkg/src/qadc/). Layout conventions follow the reference:
 * transposed lists are (nblocks, mrows, 16) bytes, row j byte l packs
 * sub-codes (2j, 2j+1) of code l (low nibble first), ids int64 with -1
 * marking padding (qadc.py:19-22, 96-113).
 */
#ifndef QADC_ORACLE_H
#define QADC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* numpy einsum("d,d->") float32 order of diff = a - b. */
float orc_einsum_sqdist(const float *a, const float *b, int n);

/* numpy float32 pairwise sum for n <= 128. */
float orc_sum_f32(const float *x, int n);

/* adc.py:61-75 compute_tables: out (m,16) f32 from codebooks (m,16,dsub). */
void orc_compute_tables(const float *codebooks, int m, int dsub,
                        const float *y, float *out);

/* ivf.py:166-182 probe: ma nearest cells (ties -> lower id) + residuals. */
void orc_probe(const float *cent, int K, int d, const float *q, int ma,
               int64_t *cells, float *residuals);

/* adc.py:108-111 _rotate (v @ R^T) in OpenBLAS sgemv_t's summation order
 * (SkylakeX/Haswell kernels: 8 FMA lanes, folded (l, l+4), then pairwise),
 * identified bit-for-bit against numpy on this host (tests/test_oracle.py). */
void orc_rotate(const float *R, int d, const float *v, float *out);

/* qadc.py:157-194 find_qmax over ONE cell (the search path only ever
 * passes the first probed cell, adc.py:172). blocks: transposed list. */
float orc_find_qmax(const float *tables, int m, const uint8_t *blocks,
                    int64_t count, int R, int init);

/* qadc.py:124-147 quantize_tables (float64 arithmetic). Returns delta. */
double orc_quantize_tables(const float *tables, int m, double qmin,
                           double qmax, uint8_t *out);

/* scan_kernels.c:384-419 qadc_block_dists (saturating lane sums). */
void orc_block_dists(const uint8_t *blocks, int64_t nblocks, int mrows,
                     const uint8_t *qt, int per_block, uint8_t *out);

/* scan_kernels.c:279-382 qadc_scan_u8: sequential bounded heap with the
 * saturation and padding rules. Returns the new heap size. */
int orc_qadc_scan(const uint8_t *blocks, int64_t nblocks, const int64_t *ids,
                  int mrows, const uint8_t *qt, float qmin, float delta,
                  float *hd, int64_t *hi, int size, int R);

/* scan_kernels.c:78-125 adc_scan_f32 (b = 4, 8, 16). */
int orc_adc_scan_f32(const uint8_t *codes, int64_t n, const int64_t *ids,
                     int m, int b, const float *tables, float *hd,
                     int64_t *hi, int size, int R);

/* heap.py:112-115 extract: sort (hd, hi) ascending by (dist, id). */
void orc_heap_extract(float *hd, int64_t *hi, int size);

/*
 * adc.py:114-187 search(method="qadc") for a batch of queries.
 * Index: nlists transposed lists concatenated; list c occupies blocks
 * [blk_off[c], blk_off[c+1]) and ids [16*blk_off[c], 16*blk_off[c+1]),
 * with count[c] valid codes. cent == NULL means a flat index (one list).
 * rotation may be NULL. lut_in, if non-NULL, injects the float LUT per
 * (query, probe slot) as (nq, ma, m, 16) instead of computing it
 * ("reference-LUT-injected" parity mode); cells_in likewise
 * injects the probe order (nq, ma).
 * scan_fn selects the block scan: NULL = this restatement, otherwise a
 * function with the reference qadc_scan_u8 signature (oracle/_ref).
 * Outputs: out_ids / out_d (nq, R), padded with -1 / +inf; out_n (nq).
 * Optional diag (nq, 2): qmax and qmin of the first probed cell.
 */
typedef int (*orc_scan_fn)(const uint8_t *, int64_t, const int64_t *, int,
                           const uint8_t *, float, float, float *, int64_t *,
                           int, int, int);

void orc_search_batch(const float *queries, int nq, int d, int m,
                      const float *codebooks, const float *rotation,
                      const float *cent, int K, int ma,
                      const uint8_t *blocks, const int64_t *blk_off,
                      const int64_t *ids, const int64_t *count, int R,
                      int init, const float *lut_in, const int64_t *cells_in,
                      orc_scan_fn scan_fn, int scan_variant, int nthreads,
                      int64_t *out_ids, float *out_d, int32_t *out_n,
                      double *diag);

/*
 * Sharded search, order-free restatement of the heap
 * semantics: the shard's lists (blocks / blk_off / ids, any subset of each
 * list's lanes) are scanned; qmax and F_sat come from the GLOBAL first
 * codes of each list (pblocks / pblk_off / pids; pcount = global list
 * lengths); only with_fsat != 0 contributes F_sat. Probe and LUT as in
 * orc_search_batch (no injection). Merging every shard's (nq, R) output by
 * (dist, id) gives orc_search_batch's result on the unsharded index.
 */
void orc_search_batch_sharded(const float *queries, int nq, int d, int m,
                              const float *codebooks, const float *rotation,
                              const float *cent, int K, int ma,
                              const uint8_t *blocks, const int64_t *blk_off,
                              const int64_t *ids, const uint8_t *pblocks,
                              const int64_t *pblk_off, const int64_t *pids,
                              const int64_t *pcount, int R, int init,
                              int with_fsat, int nthreads, int64_t *out_ids,
                              float *out_d, int32_t *out_n);

#ifdef __cplusplus
}
#endif

#endif
