/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference Quick ADC
 * search path. See qadc_oracle.h for the usage rule and conventions.
 * Reference paths are relative to /root/reference/pkg/src/qadc/.
 *
 * Compiled with -ffp-contract=off (no FMA contraction): every float
 * operation below rounds exactly where the reference's NumPy / C code
 * rounds.
 */
#include "qadc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---------- NumPy arithmetic orders the reference inherits ---------- */

/*
 * einsum("mkd,mkd->mk") / einsum("kd,kd->k") on float32 (adc.py:72-73,
 * ivf.py:178-179). NumPy 2.3 sum_of_products_contig_outstride0_two with a
 * 4-lane SSE vector and no FMA: products rounded to f32; while >= 16
 * elements remain, four 4-vectors are folded into the accumulator in the
 * order v3, v2, v1, v0; the tail is folded 4 at a time, zero padded; the
 * lanes reduce as (l0 + l1) + (l2 + l3). Pinned against numpy in
 * tests/test_oracle.py.
 */
float orc_einsum_sqdist(const float *a, const float *b, int n)
{
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    int i = 0, l, v;
    for (; n - i >= 16; i += 16) {
        for (v = 3; v >= 0; v--) {
            for (l = 0; l < 4; l++) {
                float df = a[i + 4 * v + l] - b[i + 4 * v + l];
                float p = df * df;
                acc[l] = acc[l] + p;
            }
        }
    }
    for (; i < n; i += 4) {
        for (l = 0; l < 4; l++) {
            float p = 0.0f;
            if (i + l < n) {
                float df = a[i + l] - b[i + l];
                p = df * df;
            }
            acc[l] = acc[l] + p;
        }
    }
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

/* ndarray.sum() on float32, n <= 128: NumPy pairwise_sum,
 * used by find_qmax's empty-cell bound (qadc.py:192-193). */
float orc_sum_f32(const float *x, int n)
{
    int i, j;
    if (n < 8) {
        float res = 0.0f;
        for (i = 0; i < n; i++)
            res = res + x[i];
        return res;
    }
    {
        float r[8], res;
        for (j = 0; j < 8; j++)
            r[j] = x[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (j = 0; j < 8; j++)
                r[j] = r[j] + x[i + j];
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++)
            res = res + x[i];
        return res;
    }
}

/* ---------- Tables / Index phase ---------- */

/* adc.py:61-75: D[j,i] = sum_t (C[j,i,t] - y[j,t])^2 in einsum order. */
void orc_compute_tables(const float *codebooks, int m, int dsub,
                        const float *y, float *out)
{
    int j, i;
    for (j = 0; j < m; j++)
        for (i = 0; i < 16; i++)
            out[j * 16 + i] = orc_einsum_sqdist(
                codebooks + ((size_t)j * 16 + i) * dsub, y + (size_t)j * dsub, dsub);
}

/* ivf.py:166-182: d2 by einsum, lexsort((arange K, d2))[:ma], then the
 * fp32 residual q - C[cell]. Selection keeps the ma smallest (d2, cell)
 * pairs by insertion (ma is small). */
void orc_probe(const float *cent, int K, int d, const float *q, int ma,
               int64_t *cells, float *residuals)
{
    float *bd = (float *)malloc(sizeof(float) * (size_t)ma);
    int n = 0, k, s, t;
    for (k = 0; k < K; k++) {
        float dk = orc_einsum_sqdist(cent + (size_t)k * d, q, d);
        /* position of (dk, k) among the kept pairs; k is increasing, so a
         * tie on dk always lands after the kept entry */
        if (n == ma && !(dk < bd[n - 1]))
            continue;
        s = n < ma ? n : ma - 1;
        while (s > 0 && dk < bd[s - 1]) {
            bd[s] = bd[s - 1];
            cells[s] = cells[s - 1];
            s--;
        }
        bd[s] = dk;
        cells[s] = k;
        if (n < ma)
            n++;
    }
    for (s = 0; s < ma; s++)
        for (t = 0; t < d; t++)
            residuals[(size_t)s * d + t] = q[t] - cent[(size_t)cells[s] * d + t];
    free(bd);
}

/* adc.py:108-111 _rotate: (v @ R.T) with a 1-D v = OpenBLAS sgemv_t
 * (numpy 2.3 + scipy-openblas 0.3.30 DYNAMIC_ARCH, core "SkylakeX";
 * the Haswell kernel family). Its summation order, identified bit-for-bit
 * against numpy on this project's hosts for every d >= 16 with d % 8 == 0
 * (tests/test_oracle.py pins it): eight fp32 FMA lane accumulators, lane l
 * taking k = l, l + 8, ... ascending; t_l = acc_l + acc_{l+4} (l < 4);
 * y = (t0 + t1) + (t2 + t3). Other d keep the same formula (OpenBLAS
 * takes a different tail path there; no configuration uses them with a
 * rotation). */
void orc_rotate(const float *R, int d, const float *v, float *out)
{
    int i, k, l;
    for (i = 0; i < d; i++) {
        float a[8] = {0, 0, 0, 0, 0, 0, 0, 0}, t0, t1, t2, t3;
        for (k = 0; k < d; k++) {
            l = k & 7;
            a[l] = fmaf(R[(size_t)i * d + k], v[k], a[l]);
        }
        t0 = a[0] + a[4];
        t1 = a[1] + a[5];
        t2 = a[2] + a[6];
        t3 = a[3] + a[7];
        out[i] = (t0 + t1) + (t2 + t3);
    }
}

/* ---------- QADC layer ---------- */

static int cmp_float(const void *a, const void *b)
{
    float x = *(const float *)a, y = *(const float *)b;
    return (x > y) - (x < y);
}

/* qadc.py:157-194 for one cell. The float ADC of each prefix code is
 * _pykernels.adc_batch's left-to-right fp32 order (_pykernels.py:24-27);
 * the size-R heap's worst entry is the R-th smallest value (or the max
 * when fewer than R codes exist). Codes are read straight from the
 * transposed blocks (the reference untransposes the whole list first,
 * qadc.py:179-180; only the prefix values matter). */
float orc_find_qmax(const float *tables, int m, const uint8_t *blocks,
                    int64_t count, int R, int init)
{
    int mrows = m / 2;
    int64_t take = count < init ? count : init, k;
    float *d, out;
    int j;
    if (take <= 0) {
        float mx[256];
        for (j = 0; j < m; j++) {
            int i;
            float v = tables[j * 16];
            for (i = 1; i < 16; i++)
                if (tables[j * 16 + i] > v)
                    v = tables[j * 16 + i];
            mx[j] = v;
        }
        return orc_sum_f32(mx, m);
    }
    d = (float *)malloc(sizeof(float) * (size_t)take);
    for (k = 0; k < take; k++) {
        const uint8_t *blk = blocks + (size_t)(k / 16) * mrows * 16 + (k % 16);
        float acc = 0.0f;
        for (j = 0; j < mrows; j++) {
            uint8_t byte = blk[16 * j];
            acc = acc + tables[(2 * j) * 16 + (byte & 0x0f)];
            acc = acc + tables[(2 * j + 1) * 16 + (byte >> 4)];
        }
        d[k] = acc;
    }
    qsort(d, (size_t)take, sizeof(float), cmp_float);
    out = d[(take < R ? take : R) - 1];
    free(d);
    return out;
}

/* qadc.py:124-147, float64: delta = (qmax - qmin) / 127,
 * q = clip(floor((v - qmin) / delta), 0, 127); delta == 0 maps
 * v <= qmin to 0 and everything else to 127. */
double orc_quantize_tables(const float *tables, int m, double qmin,
                           double qmax, uint8_t *out)
{
    double delta = (qmax - qmin) / 127.0;
    int i;
    for (i = 0; i < m * 16; i++) {
        double v = (double)tables[i];
        double q;
        if (delta > 0) {
            q = floor((v - qmin) / delta);
            if (q < 0)
                q = 0;
            if (q > 127)
                q = 127;
        } else {
            q = v <= qmin ? 0 : 127;
        }
        out[i] = (uint8_t)q;
    }
    return delta;
}

/* scan_kernels.c:137-167 lane sums (saturating at 255 after every add). */
static void lane_sums(const uint8_t *blk, int mrows, const uint8_t *qt,
                      uint8_t *lane_d)
{
    int j, l;
    for (l = 0; l < 16; l++) {
        unsigned acc = 0;
        for (j = 0; j < mrows; j++) {
            uint8_t byte = blk[16 * j + l];
            acc += qt[32 * j + (byte & 0x0f)];
            if (acc > 255)
                acc = 255;
            acc += qt[32 * j + 16 + (byte >> 4)];
            if (acc > 255)
                acc = 255;
        }
        lane_d[l] = (uint8_t)acc;
    }
}

/* scan_kernels.c:384-419. */
void orc_block_dists(const uint8_t *blocks, int64_t nblocks, int mrows,
                     const uint8_t *qt, int per_block, uint8_t *out)
{
    int64_t bi;
    for (bi = 0; bi < nblocks; bi++)
        lane_sums(blocks + (size_t)bi * mrows * 16, mrows,
                  per_block ? qt + (size_t)bi * mrows * 32 : qt, out + bi * 16);
}

/* ---------- bounded (dist, id) max-heap: scan_kernels.c:22-74 ---------- */

static int entry_less(float d1, int64_t i1, float d2, int64_t i2)
{
    return d1 < d2 || (d1 == d2 && i1 < i2);
}

static void sift_down(float *hd, int64_t *hi, int size, int pos)
{
    for (;;) {
        int left = 2 * pos + 1, right = left + 1, big = pos;
        float td;
        int64_t ti;
        if (left < size && entry_less(hd[big], hi[big], hd[left], hi[left]))
            big = left;
        if (right < size && entry_less(hd[big], hi[big], hd[right], hi[right]))
            big = right;
        if (big == pos)
            return;
        td = hd[pos]; hd[pos] = hd[big]; hd[big] = td;
        ti = hi[pos]; hi[pos] = hi[big]; hi[big] = ti;
        pos = big;
    }
}

static void sift_up(float *hd, int64_t *hi, int pos)
{
    while (pos > 0) {
        int parent = (pos - 1) / 2;
        float td;
        int64_t ti;
        if (!entry_less(hd[parent], hi[parent], hd[pos], hi[pos]))
            return;
        td = hd[pos]; hd[pos] = hd[parent]; hd[parent] = td;
        ti = hi[pos]; hi[pos] = hi[parent]; hi[parent] = ti;
        pos = parent;
    }
}

static int heap_push(float *hd, int64_t *hi, int size, int R, float d, int64_t id)
{
    if (size < R) {
        hd[size] = d;
        hi[size] = id;
        sift_up(hd, hi, size);
        return size + 1;
    }
    if (entry_less(d, id, hd[0], hi[0])) {
        hd[0] = d;
        hi[0] = id;
        sift_down(hd, hi, R, 0);
    }
    return size;
}

/* scan_kernels.c:260-277 byte_threshold (conservative prefilter). */
static int byte_threshold(float root, float qmin, float delta)
{
    double x;
    int t;
    if (delta <= 0.0f)
        return 254;
    x = ((double)root - (double)qmin) / (double)delta - 0.5;
    x += (fabs((double)root) + fabs((double)qmin)) * 3e-7 / (double)delta;
    if (x < -0.5)
        return -1;
    if (x >= 254.0)
        return 254;
    t = (int)floor(x) + 1;
    return t > 254 ? 254 : t;
}

/* scan_kernels.c:279-308 admit_lanes + :318-350 scan loop. */
int orc_qadc_scan(const uint8_t *blocks, int64_t nblocks, const int64_t *ids,
                  int mrows, const uint8_t *qt, float qmin, float delta,
                  float *hd, int64_t *hi, int size, int R)
{
    uint8_t lane_d[16];
    int thr = 255, have = 0, l;
    float root_at = 0.0f;
    int64_t bi;
    for (bi = 0; bi < nblocks; bi++) {
        if (size < R) {
            thr = 255;
            have = 0;
        } else if (!have || hd[0] != root_at) {
            root_at = hd[0];
            thr = byte_threshold(root_at, qmin, delta);
            have = 1;
        }
        if (thr < 0)
            continue;
        lane_sums(blocks + (size_t)bi * mrows * 16, mrows, qt, lane_d);
        for (l = 0; l < 16; l++) {
            int64_t id = ids[bi * 16 + l];
            unsigned q = lane_d[l];
            float d;
            if (thr < 255 && (int)q > thr)
                continue;
            if (id < 0)
                continue;
            d = qmin + ((float)q + 0.5f) * delta;
            if (size == R) {
                if (q == 255)
                    continue;
                if (!entry_less(d, id, hd[0], hi[0]))
                    continue;
                hd[0] = d;
                hi[0] = id;
                sift_down(hd, hi, R, 0);
            } else {
                size = heap_push(hd, hi, size, R, d, id);
            }
        }
    }
    return size;
}

/* scan_kernels.c:78-125 float ADC scan. */
int orc_adc_scan_f32(const uint8_t *codes, int64_t n, const int64_t *ids,
                     int m, int b, const float *tables, float *hd,
                     int64_t *hi, int size, int R)
{
    int64_t i;
    int j;
    for (i = 0; i < n; i++) {
        float d = 0.0f;
        if (b == 8) {
            const uint8_t *c = codes + (size_t)i * m;
            for (j = 0; j < m; j++)
                d = d + tables[(size_t)j * 256 + c[j]];
        } else if (b == 4) {
            const uint8_t *c = codes + (size_t)i * (m / 2);
            for (j = 0; j < m / 2; j++) {
                d = d + tables[(size_t)(2 * j) * 16 + (c[j] & 0x0f)];
                d = d + tables[(size_t)(2 * j + 1) * 16 + (c[j] >> 4)];
            }
        } else {
            const uint8_t *c = codes + (size_t)i * m * 2;
            for (j = 0; j < m; j++) {
                unsigned idx = (unsigned)c[2 * j] | ((unsigned)c[2 * j + 1] << 8);
                d = d + tables[(size_t)j * 65536 + idx];
            }
        }
        if (ids[i] < 0)
            continue;
        size = heap_push(hd, hi, size, R, d, ids[i]);
    }
    return size;
}

/* heap.py:112-115: ascending (dist, id); insertion sort is fine for R. */
void orc_heap_extract(float *hd, int64_t *hi, int size)
{
    int i, j;
    for (i = 1; i < size; i++) {
        float d = hd[i];
        int64_t id = hi[i];
        for (j = i; j > 0 && entry_less(d, id, hd[j - 1], hi[j - 1]); j--) {
            hd[j] = hd[j - 1];
            hi[j] = hi[j - 1];
        }
        hd[j] = d;
        hi[j] = id;
    }
}

/* ---------- adc.py:114-187 search(method="qadc"), batched ---------- */

static void search_one(int qi, const float *queries, int d, int m,
                       const float *codebooks, const float *rotation,
                       const float *cent, int K, int ma,
                       const uint8_t *blocks, const int64_t *blk_off,
                       const int64_t *ids, const int64_t *count, int R,
                       int init, const float *lut_in, const int64_t *cells_in,
                       orc_scan_fn scan_fn, int scan_variant,
                       int64_t *out_ids, float *out_d, int32_t *out_n,
                       double *diag)
{
    int dsub = d / m, mrows = m / 2, nslots = cent ? ma : 1, s, i;
    const float *q = queries + (size_t)qi * d;
    int64_t *cells = (int64_t *)malloc(sizeof(int64_t) * (size_t)nslots);
    float *res = (float *)malloc(sizeof(float) * (size_t)nslots * d);
    float *y = (float *)malloc(sizeof(float) * (size_t)d);
    float *hd = (float *)malloc(sizeof(float) * (size_t)R);
    int64_t *hi = (int64_t *)malloc(sizeof(int64_t) * (size_t)R);
    float tab[128 * 16];
    uint8_t qt[128 * 16];
    double qmax = 0.0;
    int size = 0;

    if (!cent) {
        cells[0] = 0;
        memcpy(res, q, sizeof(float) * (size_t)d);
    } else if (cells_in) {
        for (s = 0; s < nslots; s++) {
            int t;
            cells[s] = cells_in[(size_t)qi * ma + s];
            for (t = 0; t < d; t++)
                res[(size_t)s * d + t] = q[t] - cent[(size_t)cells[s] * d + t];
        }
    } else {
        orc_probe(cent, K, d, q, ma, cells, res);
    }
    for (s = 0; s < nslots; s++) {
        int64_t c = cells[s];
        const uint8_t *cb = blocks + (size_t)blk_off[c] * mrows * 16;
        int64_t nb = blk_off[c + 1] - blk_off[c];
        const int64_t *cid = ids + (size_t)blk_off[c] * 16;
        float tmin;
        double qmin, delta;
        if (lut_in) {
            memcpy(tab, lut_in + ((size_t)qi * ma + s) * m * 16,
                   sizeof(float) * (size_t)m * 16);
        } else {
            const float *r = res + (size_t)s * d;
            if (rotation) {
                orc_rotate(rotation, d, r, y);
                r = y;
            }
            orc_compute_tables(codebooks, m, dsub, r, tab);
        }
        if (s == 0)
            qmax = (double)orc_find_qmax(tab, m, cb, count[c], R, init);
        tmin = tab[0];
        for (i = 1; i < m * 16; i++)
            if (tab[i] < tmin)
                tmin = tab[i];
        qmin = (double)tmin < qmax ? (double)tmin : qmax;
        delta = orc_quantize_tables(tab, m, qmin, qmax, qt);
        if (s == 0 && diag) {
            diag[2 * (size_t)qi] = qmax;
            diag[2 * (size_t)qi + 1] = qmin;
        }
        if (nb == 0)
            continue;
        if (scan_fn)
            size = scan_fn(cb, nb, cid, mrows, qt, (float)qmin, (float)delta,
                           hd, hi, size, R, scan_variant);
        else
            size = orc_qadc_scan(cb, nb, cid, mrows, qt, (float)qmin,
                                 (float)delta, hd, hi, size, R);
    }
    orc_heap_extract(hd, hi, size);
    for (i = 0; i < R; i++) {
        out_ids[(size_t)qi * R + i] = i < size ? hi[i] : -1;
        out_d[(size_t)qi * R + i] = i < size ? hd[i] : INFINITY;
    }
    out_n[qi] = size;
    free(cells);
    free(res);
    free(y);
    free(hd);
    free(hi);
}

typedef struct {
    const float *queries; int nq, d, m; const float *codebooks, *rotation, *cent;
    int K, ma; const uint8_t *blocks; const int64_t *blk_off, *ids, *count;
    int R, init; const float *lut_in; const int64_t *cells_in;
    orc_scan_fn scan_fn; int scan_variant; int64_t *out_ids; float *out_d;
    int32_t *out_n; double *diag; int next; pthread_mutex_t mu;
} batch_args;

static void *batch_worker(void *p)
{
    batch_args *a = (batch_args *)p;
    for (;;) {
        int qi;
        pthread_mutex_lock(&a->mu);
        qi = a->next++;
        pthread_mutex_unlock(&a->mu);
        if (qi >= a->nq)
            return NULL;
        search_one(qi, a->queries, a->d, a->m, a->codebooks, a->rotation,
                   a->cent, a->K, a->ma, a->blocks, a->blk_off, a->ids,
                   a->count, a->R, a->init, a->lut_in, a->cells_in, a->scan_fn,
                   a->scan_variant, a->out_ids, a->out_d, a->out_n, a->diag);
    }
}

/* Queries are independent (adc.py:114-187 holds no shared state), so the
 * batch is spread over nthreads POSIX threads pulling query indices. */
void orc_search_batch(const float *queries, int nq, int d, int m,
                      const float *codebooks, const float *rotation,
                      const float *cent, int K, int ma,
                      const uint8_t *blocks, const int64_t *blk_off,
                      const int64_t *ids, const int64_t *count, int R,
                      int init, const float *lut_in, const int64_t *cells_in,
                      orc_scan_fn scan_fn, int scan_variant, int nthreads,
                      int64_t *out_ids, float *out_d, int32_t *out_n,
                      double *diag)
{
    batch_args a;
    pthread_t th[256];
    int t, nt = nthreads < 1 ? 1 : (nthreads > 256 ? 256 : nthreads);
    a.queries = queries; a.nq = nq; a.d = d; a.m = m; a.codebooks = codebooks;
    a.rotation = rotation; a.cent = cent; a.K = K; a.ma = ma; a.blocks = blocks;
    a.blk_off = blk_off; a.ids = ids; a.count = count; a.R = R; a.init = init;
    a.lut_in = lut_in; a.cells_in = cells_in; a.scan_fn = scan_fn;
    a.scan_variant = scan_variant; a.out_ids = out_ids; a.out_d = out_d;
    a.out_n = out_n; a.diag = diag; a.next = 0;
    pthread_mutex_init(&a.mu, NULL);
    if (nt == 1) {
        batch_worker(&a);
    } else {
        for (t = 0; t < nt; t++)
            pthread_create(&th[t], NULL, batch_worker, &a);
        for (t = 0; t < nt; t++)
            pthread_join(th[t], NULL);
    }
    pthread_mutex_destroy(&a.mu);
}

/* ---------- sharded search: one shard of every list + global prefixes ----------
 *
 * a shard holds part of each inverted list (range sharding:
 * a contiguous id range of every list; list sharding: whole lists, the
 * rest empty). The reference heap's result over the FULL lists equals
 * the top-R by (mid, id) of {valid lanes with q < 255} U F_sat, where
 * F_sat = the saturated (q == 255) lanes among the first R valid lanes of
 * the probe-order stream (orc_qadc_scan above admits a
 * q == 255 lane only while the heap is not full). Lanes split over shards
 * therefore merge exactly if every shard computes qmax and F_sat from the
 * GLOBAL first codes of each list (pblocks / pblk_off / pids, pcount = the
 * global list lengths) and only one shard (with_fsat) contributes F_sat.
 * This is the order-free restatement of that semantics: tests check it
 * against the heap restatement (orc_search_batch) on unsharded indexes
 * and on merged shards. */
static void search_one_sharded(int qi, const float *queries, int d, int m,
                               const float *codebooks, const float *rotation,
                               const float *cent, int K, int ma,
                               const uint8_t *blocks, const int64_t *blk_off,
                               const int64_t *ids, const uint8_t *pblocks,
                               const int64_t *pblk_off, const int64_t *pids,
                               const int64_t *pcount, int R, int init,
                               int with_fsat, int64_t *out_ids, float *out_d,
                               int32_t *out_n)
{
    int dsub = d / m, mrows = m / 2, nslots = cent ? ma : 1, s, i, size = 0;
    int need = R;
    const float *q = queries + (size_t)qi * d;
    int64_t *cells = (int64_t *)malloc(sizeof(int64_t) * (size_t)nslots);
    float *res = (float *)malloc(sizeof(float) * (size_t)nslots * d);
    float *y = (float *)malloc(sizeof(float) * (size_t)d);
    float *hd = (float *)malloc(sizeof(float) * (size_t)R);
    int64_t *hi = (int64_t *)malloc(sizeof(int64_t) * (size_t)R);
    float tab[128 * 16];
    uint8_t qt[128 * 16], lane_d[16];
    double qmax = 0.0;

    if (!cent) {
        cells[0] = 0;
        memcpy(res, q, sizeof(float) * (size_t)d);
    } else {
        orc_probe(cent, K, d, q, ma, cells, res);
    }
    for (s = 0; s < nslots; s++) {
        int64_t c = cells[s], bi;
        const uint8_t *pb = pblocks + (size_t)pblk_off[c] * mrows * 16;
        const int64_t *pid = pids + (size_t)pblk_off[c] * 16;
        int64_t pnb = pblk_off[c + 1] - pblk_off[c];
        const uint8_t *cb = blocks + (size_t)blk_off[c] * mrows * 16;
        const int64_t *cid = ids + (size_t)blk_off[c] * 16;
        int64_t nb = blk_off[c + 1] - blk_off[c];
        const float *r = res + (size_t)s * d;
        float tmin, fqmin, fdelta;
        double qmin, delta;
        if (rotation) {
            orc_rotate(rotation, d, r, y);
            r = y;
        }
        orc_compute_tables(codebooks, m, dsub, r, tab);
        if (s == 0)
            qmax = (double)orc_find_qmax(tab, m, pb, pcount[c], R, init);
        tmin = tab[0];
        for (i = 1; i < m * 16; i++)
            if (tab[i] < tmin)
                tmin = tab[i];
        qmin = (double)tmin < qmax ? (double)tmin : qmax;
        delta = orc_quantize_tables(tab, m, qmin, qmax, qt);
        fqmin = (float)qmin;
        fdelta = (float)delta;
        /* F_sat: the first R valid lanes of the global stream */
        for (bi = 0; with_fsat && need > 0 && bi < pnb; bi++) {
            lane_sums(pb + (size_t)bi * mrows * 16, mrows, qt, lane_d);
            for (i = 0; i < 16 && need > 0; i++) {
                if (pid[bi * 16 + i] < 0)
                    continue;
                need--;
                if (lane_d[i] == 255)
                    size = heap_push(hd, hi, size, R,
                                     fqmin + (255.0f + 0.5f) * fdelta,
                                     pid[bi * 16 + i]);
            }
        }
        /* this shard's lanes of the cell */
        for (bi = 0; bi < nb; bi++) {
            lane_sums(cb + (size_t)bi * mrows * 16, mrows, qt, lane_d);
            for (i = 0; i < 16; i++) {
                if (cid[bi * 16 + i] < 0 || lane_d[i] == 255)
                    continue;
                size = heap_push(hd, hi, size, R,
                                 fqmin + ((float)lane_d[i] + 0.5f) * fdelta,
                                 cid[bi * 16 + i]);
            }
        }
    }
    orc_heap_extract(hd, hi, size);
    for (i = 0; i < R; i++) {
        out_ids[(size_t)qi * R + i] = i < size ? hi[i] : -1;
        out_d[(size_t)qi * R + i] = i < size ? hd[i] : INFINITY;
    }
    out_n[qi] = size;
    free(cells);
    free(res);
    free(y);
    free(hd);
    free(hi);
}

typedef struct {
    const float *queries; int nq, d, m; const float *codebooks, *rotation, *cent;
    int K, ma; const uint8_t *blocks; const int64_t *blk_off, *ids;
    const uint8_t *pblocks; const int64_t *pblk_off, *pids, *pcount;
    int R, init, with_fsat; int64_t *out_ids; float *out_d; int32_t *out_n;
    int next; pthread_mutex_t mu;
} sharded_args;

static void *sharded_worker(void *p)
{
    sharded_args *a = (sharded_args *)p;
    for (;;) {
        int qi;
        pthread_mutex_lock(&a->mu);
        qi = a->next++;
        pthread_mutex_unlock(&a->mu);
        if (qi >= a->nq)
            return NULL;
        search_one_sharded(qi, a->queries, a->d, a->m, a->codebooks, a->rotation,
                           a->cent, a->K, a->ma, a->blocks, a->blk_off, a->ids,
                           a->pblocks, a->pblk_off, a->pids, a->pcount, a->R,
                           a->init, a->with_fsat, a->out_ids, a->out_d,
                           a->out_n);
    }
}

void orc_search_batch_sharded(const float *queries, int nq, int d, int m,
                              const float *codebooks, const float *rotation,
                              const float *cent, int K, int ma,
                              const uint8_t *blocks, const int64_t *blk_off,
                              const int64_t *ids, const uint8_t *pblocks,
                              const int64_t *pblk_off, const int64_t *pids,
                              const int64_t *pcount, int R, int init,
                              int with_fsat, int nthreads, int64_t *out_ids,
                              float *out_d, int32_t *out_n)
{
    sharded_args a;
    pthread_t th[256];
    int t, nt = nthreads < 1 ? 1 : (nthreads > 256 ? 256 : nthreads);
    a.queries = queries; a.nq = nq; a.d = d; a.m = m; a.codebooks = codebooks;
    a.rotation = rotation; a.cent = cent; a.K = K; a.ma = ma; a.blocks = blocks;
    a.blk_off = blk_off; a.ids = ids; a.pblocks = pblocks; a.pblk_off = pblk_off;
    a.pids = pids; a.pcount = pcount; a.R = R; a.init = init;
    a.with_fsat = with_fsat; a.out_ids = out_ids; a.out_d = out_d;
    a.out_n = out_n; a.next = 0;
    pthread_mutex_init(&a.mu, NULL);
    if (nt == 1) {
        sharded_worker(&a);
    } else {
        for (t = 0; t < nt; t++)
            pthread_create(&th[t], NULL, sharded_worker, &a);
        for (t = 0; t < nt; t++)
            pthread_join(th[t], NULL);
    }
    pthread_mutex_destroy(&a.mu);
}
