// C ABI of libqadc_b200 (include/qadc_b200.h): the reference kernel ABI
// (scan_kernels.h:15-46) re-implemented on sm_100a, plus the batched
// device-resident search (adc.py:114-187 for many queries at once).
#include <cstdio>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "qadc_b200.h"
#include "internal.cuh"

namespace qadc {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char *where) {
  g_err = std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + where;
  return kErrCuda;
}

namespace {

int arg_error(const std::string &msg) {
  g_err = msg;
  return kErrArgs;
}

int device_sms() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

__global__ void k_transpose(const float *__restrict__ in, int rows, int cols, float *__restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)rows * cols;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(t / cols), c = (int)(t % cols);
    out[(size_t)c * rows + r] = in[t];
  }
}

__global__ void k_init_bounds(unsigned *M_bits, const unsigned *M_override, float *hist_w, int nq) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    unsigned mb = M_bits[q];
    if (M_override) mb = min(mb, M_override[q]);
    M_bits[q] = mb;
    const float M = __uint_as_float(mb);
    hist_w[q] = (isfinite(M) && M > 0.f) ? M / (float)kHistBins : 0.f;
  }
}

__global__ void k_scatter_out(const int64_t *__restrict__ ids, const float *__restrict__ d,
                              const int32_t *__restrict__ n, const int *__restrict__ rows, int cnt,
                              int R, int64_t *__restrict__ out_ids, float *__restrict__ out_d,
                              int32_t *__restrict__ out_n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)cnt * R;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / R), r = (int)(t % R);
    out_ids[(size_t)rows[i] * R + r] = ids[t];
    out_d[(size_t)rows[i] * R + r] = d[t];
    if (r == 0) out_n[rows[i]] = n[i];
  }
}

// ivf.py:181-182: residual = q - C[cell] in fp32.
__global__ void k_residuals(const float *__restrict__ queries, const float *__restrict__ coarse,
                            const int64_t *__restrict__ cells, int nq, int ma, int d,
                            float *__restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)nq * ma * d;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pair = t / d;
    const int c = (int)(t % d);
    out[t] = __fsub_rn(queries[(pair / ma) * d + c], coarse[cells[pair] * d + c]);
  }
}

// SURVEY 8d "codes scanned" = sum over (query, probed list) of len(list).
__global__ void k_count_codes(const int64_t *__restrict__ cells, int64_t npairs,
                              const int64_t *__restrict__ lanes, unsigned long long *out) {
  unsigned long long acc = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs;
       p += (int64_t)gridDim.x * blockDim.x)
    acc += (unsigned long long)lanes[cells ? cells[p] : 0];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

inline int gridn(int64_t n) {
  return (int)std::min<int64_t>(std::max<int64_t>((n + 255) / 256, 1), 148 * 16);
}

template <class T>
struct DevBuf {
  T *p = nullptr;
  cudaStream_t st = nullptr;
  int alloc(int64_t n, cudaStream_t s) {
    st = s;
    if (cudaMallocAsync(&p, (size_t)std::max<int64_t>(n, 1) * sizeof(T), s) != cudaSuccess)
      return kErrCuda;
    return kOk;
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

struct SearchStats {
  int64_t codes = 0, cands = 0, reruns = 0, scan_launches = 0, launches = 0;
  double scan_us = 0.0;
  int scan_tc = 0;  // the scan ran on the tensor cores
  int scan_tile_q = 0;  // queries per work item (per pass over a list) of the scan kernel
  // device time per phase of the first pass (adc.py:140-179's Index /
  // Tables / Scan split; the work list and the exact top-R are the GPU's
  // own phases), CUDA events on the search stream
  double probe_us = 0.0, tables_us = 0.0, work_us = 0.0, select_us = 0.0;
};

// Phase events of search_impl, created once per host thread.
enum { kEvStart, kEvProbe, kEvTables, kEvWork0, kEvScan0, kEvScan1, kEvSelect, kEvCount };
cudaEvent_t *phase_events() {
  static thread_local cudaEvent_t ev[kEvCount];
  static thread_local int dev_made = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev_made != dev) {
    for (auto &e : ev) cudaEventCreate(&e);
    dev_made = dev;
  }
  return ev;
}

// Keep stream-ordered workspace in the device pool between calls (the
// default release threshold of 0 returns it to the OS at every sync, which
// turns each search's workspace allocation into page mapping work).
void retain_pool_memory() {
  static thread_local int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}

// ivf.py:166-182 probe of the index's coarse quantizer: cells (nq, ma).
void index_probe(const qadc_b200_index *idx, const float *queries, int nq, int ma, int64_t *cells,
                 cudaStream_t st) {
  // 2 = fused tensor-core probe, 1 = FFMA pre-selection, 0 = exact scan
  static const int probe_kind = scan_env_int("QADC_B200_PROBE", 2);
  const bool done =
      (probe_kind >= 2 && idx->pcsplit &&
       launch_probe_tc(idx->coarse, idx->pmu, idx->pcsplit, idx->pcn2, idx->K, idx->d, queries,
                       nq, ma, cells, st)) ||
      (probe_kind >= 1 && idx->cnorm &&
       launch_probe_fast(idx->coarseT, idx->coarse, idx->cnorm, idx->K, idx->d, queries, nq, ma,
                         cells, st));
  if (!done) launch_probe(idx->coarseT, idx->K, idx->d, queries, nq, ma, cells, st);
}

// Per-query scan inputs produced by the Index + Tables phases
// (adc.py:140-174 for every query of the batch), device arrays.
struct Prep {
  const int64_t *cells = nullptr;   // [npairs] probe order (IVF) or null (flat)
  const uint32_t *qt = nullptr;     // [npairs][m][4] uint8 tables as words
  const float *qmin_f = nullptr;    // [npairs] fp32 casts the scan uses
  const float *delta_f = nullptr;   // [npairs]
  const uint8_t *depth = nullptr;   // [npairs] byte-sum depth of the pair's tables
  unsigned *M_bits = nullptr;       // [nq] running distance bound (the scan tightens it)
  const int *fsat_n = nullptr;      // [nq] saturated first-R lanes (F_sat)
  const float *fsat_mid = nullptr;  // [nq][R]
  const int64_t *fsat_id = nullptr; // [nq][R]
};

template <class T>
__global__ void k_gather(const T *__restrict__ src, const int *__restrict__ rows, int n, int width,
                         T *__restrict__ dst) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n * width;
       t += (int64_t)gridDim.x * blockDim.x)
    dst[t] = src[(size_t)rows[t / width] * width + t % width];
}

// Index + Tables phases: probe (IVF, unless cells_in), residual + rotation +
// float LUT (unless lut_in), qmax from the first probed cell, per-pair qmin /
// delta and uint8 tables (+ byte-sum depth), prefix facts (F_sat, initial
// bound). Outputs are caller-owned device arrays; cells_out may alias
// nothing (flat) and receives the probe order otherwise.
int prepare_impl(qadc_b200_index *idx, const float *queries, int nq, int R, int ma, int init,
                 const float *lut_in, const int64_t *cells_in, bool no_fsat, cudaStream_t st,
                 SearchStats &ss, int64_t *cells_out, uint32_t *qt, float *qmin_f, float *delta_f,
                 uint8_t *depth, float *qmax, unsigned *M_bits, int *fsat_n, float *fsat_mid,
                 int64_t *fsat_id) {
  if (nq == 0) return kOk;
  const int m = idx->m;
  const int nslots = idx->K ? ma : 1;
  const int64_t npairs = (int64_t)nq * nslots;
  cudaEvent_t *ev = phase_events();
  cudaEventRecord(ev[kEvStart], st);
  const int64_t *cells = nullptr;
  if (idx->K) {
    if (cells_in) {
      if (cells_out && cells_out != cells_in)
        QADC_CUDA(cudaMemcpyAsync(cells_out, cells_in, npairs * 8, cudaMemcpyDeviceToDevice, st));
      cells = cells_in;
    } else {
      index_probe(idx, queries, nq, ma, cells_out, st);
      QADC_CUDA(cudaGetLastError());
      ss.launches++;
      cells = cells_out;
    }
  }
  cudaEventRecord(ev[kEvProbe], st);
  DevBuf<float> lut_b;
  const float *lut = lut_in;
  if (!lut) {
    if (lut_b.alloc(npairs * m * 16, st)) return cuda_fail(cudaGetLastError(), "alloc lut");
    launch_residual_lut(idx, queries, cells, nq, nslots, lut_b.p, st);
    QADC_CUDA(cudaGetLastError());
    ss.launches++;
    lut = lut_b.p;
  }
  // tuning knob (default = measured best): byte-sum depth cap
  static const int max_depth = std::min(16, std::max(2, scan_env_int("QADC_B200_MAX_DEPTH", 16)));
  if (int rc = launch_qmax(idx, lut, cells, nq, nslots, R, init, qmax, st)) return rc;
  launch_quantize(lut, (int)npairs, m, qmax, nslots, nullptr, nullptr, qt, qmin_f, delta_f,
                  nullptr, nullptr, st, max_depth, depth);
  launch_prefix(idx, qt, qmin_f, delta_f, cells, nq, nslots, R, init, M_bits, fsat_n, fsat_mid,
                fsat_id, st);
  QADC_CUDA(cudaGetLastError());
  ss.launches += 3;
  if (no_fsat) QADC_CUDA(cudaMemsetAsync(fsat_n, 0, sizeof(int) * nq, st));
  cudaEventRecord(ev[kEvTables], st);
  return kOk;
}

// Work list, scan, exact top-R (and the rare overflow passes) over prepared
// per-query inputs. p.M_bits is tightened in place. level > 0: a rerun pass
// over a subset with a larger candidate capacity (no phase timing).
int scan_impl(qadc_b200_index *idx, const Prep &p, int nq, int R, int ma, int init,
              int64_t *out_ids, float *out_d, int32_t *out_n, cudaStream_t st, SearchStats &ss,
              int cap_g, int level, bool prmt, bool force_tc, bool one_sm, bool force_tcw) {
  if (nq == 0) return kOk;
  const int m = idx->m;
  const int nslots = idx->K ? ma : 1;
  const int64_t npairs = (int64_t)nq * nslots;
  const int64_t *cells = idx->K ? p.cells : nullptr;
  cudaEvent_t *ev = phase_events();
  if (level == 0) cudaEventRecord(ev[kEvWork0], st);
  // The tensor-core scan amortises each code's one-hot expansion over the
  // queries probing its list: with few (query, list) pairs per list (IVF
  // at small nprobe / large K) the PRMT kernel is faster (measured: cfg2
  // nprobe 16, ~40 pairs per list: 10.2 ms PRMT vs 25.6 ms tensor cores).
  static const int tc_min_pairs = scan_env_int("QADC_B200_TC_MIN_PAIRS", 64);
  // Inverted lists probed by a handful of queries each: the warpgroup-
  // pipelined tensor-core scan (k_scan_tcw, <= 32 queries per pass over a
  // list). Its cost per code is the one-hot expansion, whatever the number
  // of queries, so the PRMT kernel keeps the batches that put fewer than
  // ~4 queries on a probed list (expected probed lists under uniform
  // probing: nl (1 - exp(-npairs / nl))). QADC_B200_TCW=0 disables it.
  static const int tcw_env = scan_env_int("QADC_B200_TCW", 1);
  // (measured at configs[4] with smaller batches: Q = 2000 PRMT 10.2 ms vs
  // 15.1 ms, Q = 4000 16.9 vs 15.9 ms, Q = 6000 23.8 vs ~16.5 ms, Q = 10^4
  // 37.4 vs 17.9 ms: the kernels cross at ~3.8 by this estimate)
  static const int tcw_min = scan_env_int("QADC_B200_TCW_MIN_PAIRS", 4);
  static const int tcw_max = scan_env_int("QADC_B200_TCW_MAX_PAIRS", 1 << 20);
  const int nl = idx->nlists;
  int tcw = 0;
  if (!prmt && !force_tc && !one_sm && idx->K > 0 && scan_use_tc(m, false)) {
    const double load = (double)npairs / nl;
    const double per_probed = load / std::max(1e-9, 1.0 - std::exp(-load));
    // (a 2-warpgroup shape with <= 128 queries per pass was measured for the
    // lists of configs[2]: 32.2 / 23.7 ms at nprobe 16 / 64 against 5.9 /
    // 11.7 ms here: its survivor entries are 4x wider and two filter warps
    // do not keep up)
    if (force_tcw || (tcw_env && nl > 1 && per_probed >= 0.95 * tcw_min && load <= tcw_max)) tcw = 1;
    // the code-major copy (m / 2 more bytes per code) may not fit next to a
    // very large index: the heuristic choice then stays on the PRMT scan
    if (tcw && ensure_code_major(idx, st) != kOk) {
      if (force_tcw) return kErrCuda;
      cudaGetLastError();
      tcw = 0;
    }
  }
  if (!tcw && !force_tc && npairs < (int64_t)tc_min_pairs * std::max(idx->nlists, 1)) prmt = true;
  const int qt_tile = scan_tile_queries(m, prmt, tcw != 0);

  DevBuf<float> cand_mid, hist_w;
  DevBuf<unsigned> cand_n, hist;
  DevBuf<int> n_items, counter, scratch, overflow;
  DevBuf<unsigned long long> ncodes;
  DevBuf<int64_t> cand_id;
  DevBuf<int32_t> pair_q, pair_t;
  DevBuf<WorkItem> items, items_ord;
  DevBuf<unsigned> cls;
  int rc = 0;
  if (hist.alloc((int64_t)nq * kHistWords, st) || hist_w.alloc(nq, st) || cand_n.alloc(nq, st) ||
      cand_mid.alloc((int64_t)nq * cap_g, st) || cand_id.alloc((int64_t)nq * cap_g, st) ||
      pair_q.alloc(npairs, st) || pair_t.alloc(npairs, st) || n_items.alloc(1, st) ||
      counter.alloc(1, st) || scratch.alloc(build_work_scratch(nl, nslots), st) ||
      overflow.alloc(nq, st) || ncodes.alloc(1, st))
    return cuda_fail(cudaGetLastError(), "alloc workspace");
  // tuning knobs (defaults are the measured best): the half-tile loop for
  // tiles with <= QT/2 queries, item ordering, per-variant item counts
  static const int no_half = scan_env_int("QADC_B200_NO_HALF", 0);
  static const int variant_stats = scan_env_int("QADC_B200_VARIANT_STATS", 0);
  static const int no_order = scan_env_int("QADC_B200_NO_ORDER", 0);
  k_init_bounds<<<gridn(nq), 256, 0, st>>>(p.M_bits, nullptr, hist_w.p, nq);
  QADC_CUDA(cudaGetLastError());
  ss.launches++;

  // ---- work list ----
  const int nsm = device_sms();
  int64_t max_ranges = 0, sum_ranges = 0;
  const int64_t avg_chunks = std::max<int64_t>(1, idx->total_chunks / std::max(nl, 1));
  const int64_t work_chunks = ((npairs + qt_tile - 1) / qt_tile) * avg_chunks;
  // few, long items: each warp's local selection sees many codes before it
  // publishes (about 3 items per resident CTA, 4 CTAs per SM)
  int64_t range_chunks = work_chunks / ((int64_t)nsm * 12);
  int64_t rcp = 16;
  while (rcp < range_chunks && rcp < 16384) rcp <<= 1;
  range_chunks = rcp;
  const int cap_l = (std::max(R + 128, 256) + 31) / 32 * 32;
  const int linear = scan_env_int("QADC_B200_LINEAR", -1) >= 0 ? scan_env_int("QADC_B200_LINEAR", 0)
                                                                 : (avg_chunks >= 64 ? 1 : 0);
  // one exhaustive list on the tensor-core scan: CTA pairs (k_scan_tc2)
  static const int tc2_env = scan_env_int("QADC_B200_TC2", 1);
  // CTA-pair variant: flusher warps for long scans (>= 8K chunks per
  // list: the survivor burst of the loose initial bound is amortised),
  // inline survivor handling otherwise (QADC_B200_TC2=2 / 3 forces inline / rings)
  static const int tc2_rings_min = scan_env_int("QADC_B200_TC2_RINGS_MIN_CHUNKS", 8192);
  int pair_cta = (tc2_env && !one_sm && nl == 1 && scan_use_tc(m, prmt) && nsm >= 2) ? 1 : 0;
  if (pair_cta) pair_cta = tc2_env == 2 ? 2 : tc2_env == 3 ? 1 : (idx->total_chunks >= tc2_rings_min ? 1 : 2);
  if (nl == 1 && idx->total_chunks > 0) {
    // one exhaustive list: equal-size items, so the persistent CTAs finish
    // together only if the item count fills whole waves. Pick the range
    // count r minimising waves x (chunks per item + per-item overhead).
    const int64_t tiles = (npairs + qt_tile - 1) / qt_tile;
    const int64_t ctas = pair_cta ? nsm / 2 : scan_resident_ctas(m, cap_l, nsm, linear, prmt);
    const int64_t ch = idx->total_chunks;
    int64_t best_r = 1;
    double best = 1e300;
    for (int64_t r = 1; r <= std::min<int64_t>(ch, 4096); r++) {
      const int64_t per = (ch + r - 1) / r;
      if (per < 16 && r > 1) break;
      const int64_t waves = (tiles * r + ctas - 1) / ctas;
      // per-item overhead ~20 chunk-times (measured: prologue, end-of-item
      // barrier and flush)
      const double cost = (double)waves * (double)(per + 20);
      if (cost < best * 0.999) {
        best = cost;
        best_r = r;
      }
    }
    static const int r_env = scan_env_int("QADC_B200_RANGES", 0);
    if (r_env > 0) best_r = std::min<int64_t>(r_env, ch);
    range_chunks = (ch + best_r - 1) / best_r;
  }
  for (int L = 0; L < nl; L++) {
    const int64_t nch = idx->h_chunk_off[L + 1] - idx->h_chunk_off[L];
    const int64_t r = (nch + range_chunks - 1) / range_chunks;
    max_ranges = std::max(max_ranges, r);
    sum_ranges += r;
  }
  const int64_t max_items = (npairs / qt_tile + 1) * max_ranges + sum_ranges + 1;
  if (items.alloc(max_items, st)) return cuda_fail(cudaGetLastError(), "alloc items");
  build_work(idx, cells, nq, nslots, qt_tile, range_chunks, pair_q.p, pair_t.p, items.p, n_items.p,
             scratch.p, max_items, st);
  if (items_ord.alloc(max_items, st) || cls.alloc(order_items_scratch(max_items), st))
    return cuda_fail(cudaGetLastError(), "alloc items");
  order_items(items.p, n_items.p, max_items, pair_t.p, p.depth, no_half ? 0 : qt_tile / 2,
              nslots, cls.p, items_ord.p, st);
  ss.launches += 8;

  // ---- scan ----
  cudaMemsetAsync(cand_n.p, 0, sizeof(unsigned) * nq, st);
  cudaMemsetAsync(hist.p, 0, sizeof(unsigned) * (size_t)nq * kHistWords, st);
  cudaMemsetAsync(counter.p, 0, sizeof(int), st);
  cudaMemsetAsync(ncodes.p, 0, sizeof(unsigned long long), st);
  k_count_codes<<<gridn(npairs), 256, 0, st>>>(cells, npairs, idx->scan_count, ncodes.p);
  ScanArgs a;
  a.codes = idx->codes;
  a.codes_cm = nullptr;
  a.tcw = tcw;
  if (scan_use_tc(m, prmt) && !pair_cta) {  // k_scan_tc / k_scan_tcw expand from the code-major copy
    if ((rc = ensure_code_major(idx, st))) return rc;
    a.codes_cm = idx->codes_cm;
  }
  a.valid = idx->valid;
  a.ids = idx->ids;
  a.items = no_order ? items.p : items_ord.p;
  a.n_items = n_items.p;
  a.item_counter = counter.p;
  a.pair_q = pair_q.p;
  a.pair_t = pair_t.p;
  a.qt = p.qt;
  a.qmin_f = p.qmin_f;
  a.delta_f = p.delta_f;
  a.M_bits = p.M_bits;
  a.cand_n = cand_n.p;
  a.cand_mid = cand_mid.p;
  a.cand_id = cand_id.p;
  a.hist = hist.p;
  a.hist_w = hist_w.p;
  a.cap_g = cap_g;
  a.cap_l = cap_l;
  a.m = m;
  a.R = R;
  static const int bound_every = std::max(1, scan_env_int("QADC_B200_BOUND_EVERY", 32));
  a.bound_every = bound_every;
  a.linear = linear;  // long items (>= 64 chunks per list on average)
  static const int tc_dbg = scan_env_int("QADC_B200_TC_DEBUG", 0);
  a.dbg = tc_dbg;
  a.pair_cta = pair_cta;
  cudaEvent_t e0 = ev[kEvScan0], e1 = ev[kEvScan1];
  cudaEventRecord(e0, st);
  launch_scan(a, nsm, st, prmt);
  if (tc_dbg & 64) {
    cudaStreamSynchronize(st);
    tc_stats_dump();
  }
  ss.scan_tc = scan_use_tc(m, prmt) ? (tcw ? 2 : 1) : 0;
  if (level == 0) ss.scan_tile_q = qt_tile;
  QADC_CUDA(cudaGetLastError());
  cudaEventRecord(e1, st);
  ss.scan_launches++;
  ss.launches++;
  launch_select(nq, R, p.M_bits, cand_n.p, cand_mid.p, cand_id.p, cap_g, p.fsat_n, p.fsat_mid,
                p.fsat_id, out_ids, out_d, out_n, overflow.p, st);
  ss.launches++;
  QADC_CUDA(cudaGetLastError());
  cudaEventRecord(ev[kEvSelect], st);

  // ---- overflow handling (rare: massive ties or very loose early bounds) ----
  std::vector<int> h_over(nq);
  std::vector<unsigned> h_cn(nq);
  QADC_CUDA(cudaMemcpyAsync(h_over.data(), overflow.p, sizeof(int) * nq, cudaMemcpyDeviceToHost, st));
  QADC_CUDA(cudaMemcpyAsync(h_cn.data(), cand_n.p, sizeof(unsigned) * nq, cudaMemcpyDeviceToHost, st));
  unsigned long long h_codes = 0;
  QADC_CUDA(cudaMemcpyAsync(&h_codes, ncodes.p, sizeof(h_codes), cudaMemcpyDeviceToHost, st));
  QADC_CUDA(cudaStreamSynchronize(st));
  if (level == 0) ss.codes += (int64_t)h_codes;
  if (variant_stats) {
    unsigned v[8];
    cudaMemcpy(v, cls.p, sizeof(v), cudaMemcpyDeviceToHost);
    fprintf(stderr, "qadc_b200 scan items by variant (full D16 D8 D4 D2 | half D16 D8 D4 D2):"
            " %u %u %u %u | %u %u %u %u\n", v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]);
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  ss.scan_us += ms * 1e3;
  if (level == 0) {
    float t = 0.f;
    cudaEventElapsedTime(&t, ev[kEvWork0], e0);
    ss.work_us += t * 1e3;
    cudaEventElapsedTime(&t, e1, ev[kEvSelect]);
    ss.select_us += t * 1e3;
  }
  for (int q = 0; q < nq; q++) ss.cands += std::min<unsigned>(h_cn[q], (unsigned)cap_g);
  std::vector<int> rerun, big;
  unsigned need = 0;
  for (int q = 0; q < nq; q++) {
    if (!h_over[q]) continue;
    if (h_cn[q] > (unsigned)cap_g) {
      rerun.push_back(q);
      need = std::max(need, h_cn[q]);
    } else {
      big.push_back(q);
    }
  }
  for (int q : big) {
    if ((rc = select_large(q, R, p.M_bits, cand_n.p, cand_mid.p, cand_id.p, cap_g, p.fsat_n,
                           p.fsat_mid, p.fsat_id, out_ids, out_d, out_n, st)))
      return rc;
    ss.launches += 4;
  }
  if (!rerun.empty()) {
    // the dropped candidates are re-found by scanning the overflowed
    // queries again with their final (tight) bound and a larger capacity;
    // their prepared tables are gathered, not recomputed
    if (level > 4) return arg_error("candidate capacity could not be satisfied");
    ss.reruns += (int64_t)rerun.size();
    const int nr = (int)rerun.size();
    const int64_t w = (int64_t)nslots;
    DevBuf<int> rows, sub_fn;
    DevBuf<uint32_t> sub_qt;
    DevBuf<float> sub_qmin, sub_delta, sub_fm, sub_d;
    DevBuf<uint8_t> sub_depth;
    DevBuf<unsigned> sub_M;
    DevBuf<int64_t> sub_cells, sub_fi, sub_ids;
    DevBuf<int32_t> sub_n;
    if (rows.alloc(nr, st) || sub_qt.alloc(nr * w * m * 4, st) || sub_qmin.alloc(nr * w, st) ||
        sub_delta.alloc(nr * w, st) || sub_depth.alloc(nr * w, st) || sub_M.alloc(nr, st) ||
        sub_fn.alloc(nr, st) || sub_fm.alloc((int64_t)nr * R, st) ||
        sub_fi.alloc((int64_t)nr * R, st) || sub_ids.alloc((int64_t)nr * R, st) ||
        sub_d.alloc((int64_t)nr * R, st) || sub_n.alloc(nr, st) ||
        (cells && sub_cells.alloc(nr * w, st)))
      return cuda_fail(cudaGetLastError(), "alloc rerun");
    QADC_CUDA(cudaMemcpyAsync(rows.p, rerun.data(), sizeof(int) * nr, cudaMemcpyHostToDevice, st));
    k_gather<uint32_t><<<gridn(nr * w * m * 4), 256, 0, st>>>(p.qt, rows.p, nr, (int)(w * m * 4), sub_qt.p);
    k_gather<float><<<gridn(nr * w), 256, 0, st>>>(p.qmin_f, rows.p, nr, (int)w, sub_qmin.p);
    k_gather<float><<<gridn(nr * w), 256, 0, st>>>(p.delta_f, rows.p, nr, (int)w, sub_delta.p);
    k_gather<uint8_t><<<gridn(nr * w), 256, 0, st>>>(p.depth, rows.p, nr, (int)w, sub_depth.p);
    k_gather<unsigned><<<gridn(nr), 256, 0, st>>>(p.M_bits, rows.p, nr, 1, sub_M.p);
    k_gather<int><<<gridn(nr), 256, 0, st>>>(p.fsat_n, rows.p, nr, 1, sub_fn.p);
    k_gather<float><<<gridn((int64_t)nr * R), 256, 0, st>>>(p.fsat_mid, rows.p, nr, R, sub_fm.p);
    k_gather<int64_t><<<gridn((int64_t)nr * R), 256, 0, st>>>(p.fsat_id, rows.p, nr, R, sub_fi.p);
    if (cells)
      k_gather<int64_t><<<gridn(nr * w), 256, 0, st>>>(cells, rows.p, nr, (int)w, sub_cells.p);
    QADC_CUDA(cudaGetLastError());
    Prep sp;
    sp.cells = cells ? sub_cells.p : nullptr;
    sp.qt = sub_qt.p;
    sp.qmin_f = sub_qmin.p;
    sp.delta_f = sub_delta.p;
    sp.depth = sub_depth.p;
    sp.M_bits = sub_M.p;
    sp.fsat_n = sub_fn.p;
    sp.fsat_mid = sub_fm.p;
    sp.fsat_id = sub_fi.p;
    const int cap2 = (int)std::min<int64_t>(std::max<int64_t>((int64_t)need + 1024, 2LL * cap_g),
                                            (int64_t)1 << 28);
    rc = scan_impl(idx, sp, nr, R, ma, init, sub_ids.p, sub_d.p, sub_n.p, st, ss, cap2, level + 1,
                   prmt, force_tc, one_sm, force_tcw);
    if (rc) return rc;
    k_scatter_out<<<gridn((int64_t)nr * R), 256, 0, st>>>(sub_ids.p, sub_d.p, sub_n.p, rows.p, nr,
                                                          R, out_ids, out_d, out_n);
  }
  QADC_CUDA(cudaGetLastError());
  return kOk;
}

// Whole search: prepare into stream-ordered buffers, then scan.
int search_impl(qadc_b200_index *idx, const float *queries, int nq, int R, int ma, int init,
                const float *lut_in, const int64_t *cells_in, int64_t *out_ids, float *out_d,
                int32_t *out_n, cudaStream_t st, SearchStats &ss, int cap_g, bool no_fsat,
                bool prmt, bool force_tc, bool one_sm, bool force_tcw) {
  if (nq == 0) return kOk;
  const int m = idx->m;
  const int nslots = idx->K ? ma : 1;
  const int64_t npairs = (int64_t)nq * nslots;
  DevBuf<int64_t> cells_b, fsat_id;
  DevBuf<float> qmax_b, qmin_f, delta_f, fsat_mid;
  DevBuf<uint32_t> qt_b;
  DevBuf<unsigned> M_bits;
  DevBuf<int> fsat_n;
  DevBuf<uint8_t> depth;
  if (qmax_b.alloc(nq, st) || qt_b.alloc(npairs * m * 4, st) || qmin_f.alloc(npairs, st) ||
      delta_f.alloc(npairs, st) || M_bits.alloc(nq, st) || fsat_n.alloc(nq, st) ||
      fsat_mid.alloc((int64_t)nq * R, st) || fsat_id.alloc((int64_t)nq * R, st) ||
      depth.alloc(npairs, st) || (idx->K && !cells_in && cells_b.alloc(npairs, st)))
    return cuda_fail(cudaGetLastError(), "alloc workspace");
  int rc = prepare_impl(idx, queries, nq, R, ma, init, lut_in, cells_in, no_fsat, st, ss,
                        cells_in ? nullptr : cells_b.p, qt_b.p, qmin_f.p, delta_f.p, depth.p,
                        qmax_b.p, M_bits.p, fsat_n.p, fsat_mid.p, fsat_id.p);
  if (rc) return rc;
  Prep p;
  p.cells = idx->K ? (cells_in ? cells_in : cells_b.p) : nullptr;
  p.qt = qt_b.p;
  p.qmin_f = qmin_f.p;
  p.delta_f = delta_f.p;
  p.depth = depth.p;
  p.M_bits = M_bits.p;
  p.fsat_n = fsat_n.p;
  p.fsat_mid = fsat_mid.p;
  p.fsat_id = fsat_id.p;
  rc = scan_impl(idx, p, nq, R, ma, init, out_ids, out_d, out_n, st, ss, cap_g, 0, prmt, force_tc,
                 one_sm, force_tcw);
  if (rc) return rc;
  float t = 0.f;
  cudaEvent_t *ev = phase_events();
  cudaEventElapsedTime(&t, ev[kEvStart], ev[kEvProbe]);
  ss.probe_us += t * 1e3;
  cudaEventElapsedTime(&t, ev[kEvProbe], ev[kEvTables]);
  ss.tables_us += t * 1e3;
  return kOk;
}

int candidate_capacity(int nq, int R) {
  // per-query candidate capacity: at least 8192 / 8R, and up to 64K while
  // the lists stay within ~512 MB (small batches with heavy ties at the
  // boundary level then never need the rerun pass)
  const int64_t cap_mem = (512LL << 20) / 12 / std::max(nq, 1);
  return (int)std::min<int64_t>(
      std::max<int64_t>({8192, 8LL * R, std::min<int64_t>(65536, cap_mem)}), 1 << 20);
}

void write_stats(const SearchStats &ss, int64_t *stats) {
  if (!stats) return;
  stats[0] = ss.codes;
  stats[1] = ss.cands;
  stats[2] = ss.reruns;
  stats[3] = ss.scan_launches;
  stats[4] = ss.launches;
  stats[5] = (int64_t)llround(ss.scan_us);
  stats[6] = ss.scan_tc;  // scan kernel: 0 = PRMT, 1 = int8 tensor-core, 2 = warpgroup-pipelined int8 tensor-core
  stats[7] = (int64_t)llround(ss.probe_us);
  stats[8] = (int64_t)llround(ss.tables_us);
  stats[9] = (int64_t)llround(ss.work_us);
  stats[10] = (int64_t)llround(ss.select_us);
  stats[11] = ss.scan_tile_q;
  for (int i = 12; i < 16; i++) stats[i] = 0;
}

}  // namespace
}  // namespace qadc

using namespace qadc;

// ============================ Part 1 ============================

extern "C" int qadc_simd_level(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    set_error("no CUDA device");
    return -1;
  }
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) {
    set_error("device is not sm_100 (Blackwell B200)");
    return -1;
  }
  return QADC_KERNEL_B200;
}

extern "C" const char *qadc_b200_last_error(void) { return g_err.c_str(); }

namespace {
template <class T>
int upload(T **d, const T *h, int64_t n) {
  QADC_CUDA(cudaMalloc(d, (size_t)std::max<int64_t>(n, 1) * sizeof(T)));
  if (n > 0) QADC_CUDA(cudaMemcpy(*d, h, (size_t)n * sizeof(T), cudaMemcpyHostToDevice));
  return kOk;
}

// Heap arrays leave in descending (dist, id) order: a valid max-heap layout
// (heap.py:95-98 relies on the same fact).
void write_heap_desc(const std::vector<float> &d, const std::vector<int64_t> &i, int n, float *hd,
                     int64_t *hi) {
  for (int k = 0; k < n; k++) {
    hd[k] = d[n - 1 - k];
    hi[k] = i[n - 1 - k];
  }
}

int check_heap(int size, int R) {
  if (R < 1) return arg_error("heap capacity must be positive");
  if (size < 0 || size > R) return arg_error("heap size out of range");
  return kOk;
}
}  // namespace

extern "C" int adc_scan_f32(const uint8_t *codes, int64_t n, const int64_t *ids, int m, int b,
                            const float *tables, float *hd, int64_t *hi, int size, int R) {
  g_err.clear();
  if (check_heap(size, R)) return -1;
  if (b != 4 && b != 8 && b != 16) return (arg_error("b must be 4, 8 or 16"), -1);
  if (m < 1 || m > QADC_MAX_M || (b == 4 && m % 2)) return (arg_error("unsupported m"), -1);
  if (n <= 0) return size;
  const int64_t row = b == 4 ? m / 2 : (b == 8 ? m : 2 * m);
  uint8_t *dc = nullptr;
  int64_t *di = nullptr, *dhi = nullptr, *oi = nullptr;
  float *dt = nullptr, *dhd = nullptr, *od = nullptr;
  int out = -1;
  if (!upload(&dc, codes, n * row) && !upload(&di, ids, n) &&
      !upload(&dt, tables, (int64_t)m << b) && !upload(&dhd, hd, size) && !upload(&dhi, hi, size) &&
      cudaMalloc(&od, (size_t)R * 4) == cudaSuccess && cudaMalloc(&oi, (size_t)R * 8) == cudaSuccess) {
    out = adc_f32_device(dc, n, di, m, b, dt, dhd, dhi, size, R, od, oi, 0);
    if (out >= 0) {
      std::vector<float> vd(out);
      std::vector<int64_t> vi(out);
      if (cudaMemcpy(vd.data(), od, out * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
          cudaMemcpy(vi.data(), oi, out * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
        cuda_fail(cudaGetLastError(), "adc_scan_f32 D2H");
        out = -1;
      } else {
        write_heap_desc(vd, vi, out, hd, hi);
      }
    } else {
      out = -1;
    }
  }
  cudaFree(dc); cudaFree(di); cudaFree(dt); cudaFree(dhd); cudaFree(dhi); cudaFree(od); cudaFree(oi);
  return out;
}

extern "C" int qadc_scan_u8(const uint8_t *blocks, int64_t nblocks, const int64_t *ids, int mrows,
                            const uint8_t *qt, float qmin, float delta, float *hd, int64_t *hi,
                            int size, int R, int variant) {
  g_err.clear();
  (void)variant;
  if (check_heap(size, R)) return -1;
  if (mrows < 1 || 2 * mrows > QADC_MAX_M) return (arg_error("unsupported row count"), -1);
  if (nblocks <= 0) return size;
  uint8_t *db = nullptr, *dq = nullptr;
  int64_t *di = nullptr, *dhi = nullptr, *oi = nullptr;
  float *dhd = nullptr, *od = nullptr;
  int out = -1;
  if (!upload(&db, blocks, nblocks * mrows * 16) && !upload(&di, ids, nblocks * 16) &&
      !upload(&dq, qt, (int64_t)mrows * 32) && !upload(&dhd, hd, size) && !upload(&dhi, hi, size) &&
      cudaMalloc(&od, (size_t)R * 4) == cudaSuccess && cudaMalloc(&oi, (size_t)R * 8) == cudaSuccess) {
    out = scan_u8_device(db, nblocks, di, mrows, dq, qmin, delta, dhd, dhi, size, R, od, oi, 0);
    if (out >= 0) {
      std::vector<float> vd(out);
      std::vector<int64_t> vi(out);
      if (cudaMemcpy(vd.data(), od, out * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
          cudaMemcpy(vi.data(), oi, out * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
        cuda_fail(cudaGetLastError(), "qadc_scan_u8 D2H");
        out = -1;
      } else {
        write_heap_desc(vd, vi, out, hd, hi);
      }
    } else {
      out = -1;
    }
  }
  cudaFree(db); cudaFree(dq); cudaFree(di); cudaFree(dhd); cudaFree(dhi); cudaFree(od); cudaFree(oi);
  return out;
}

extern "C" void qadc_block_dists(const uint8_t *blocks, int64_t nblocks, int mrows,
                                 const uint8_t *qt, int per_block, uint8_t *out, int variant) {
  g_err.clear();
  (void)variant;
  if (nblocks <= 0 || mrows < 1 || 2 * mrows > QADC_MAX_M) return;
  uint8_t *db = nullptr, *dq = nullptr, *dout = nullptr;
  const int64_t qn = per_block ? nblocks * mrows * 32 : (int64_t)mrows * 32;
  if (!upload(&db, blocks, nblocks * mrows * 16) && !upload(&dq, qt, qn) &&
      cudaMalloc(&dout, (size_t)nblocks * 16) == cudaSuccess) {
    launch_block_dists(db, nblocks, mrows, dq, per_block, dout, 0);
    if (cudaMemcpy(out, dout, (size_t)nblocks * 16, cudaMemcpyDeviceToHost) != cudaSuccess)
      cuda_fail(cudaGetLastError(), "qadc_block_dists D2H");
  }
  cudaFree(db); cudaFree(dq); cudaFree(dout);
}

// ============================ Part 2 ============================

namespace {
void alias_prefix(qadc_b200_index *idx) {
  idx->pcodes = idx->codes;
  idx->pids = idx->ids;
  idx->pchunk_off = idx->chunk_off;
  idx->planes = idx->lanes;
  idx->own_prefix = false;
}

int index_common(int d, int m, int nlists, const float *coarse, bool coarse_dev,
                 const float *codebooks, const float *rotation, bool model_dev,
                 const std::vector<int64_t> &lanes, const std::vector<int64_t> &count,
                 qadc_b200_index *idx) {
  if (d < 1 || m < 2 || m > QADC_MAX_M || m % 2 || d % m) return arg_error("invalid d / m geometry");
  if (nlists < 1) return arg_error("index needs at least one list");
  if (!coarse && nlists != 1) return arg_error("a flat index has exactly one list");
  idx->d = d;
  idx->m = m;
  idx->dsub = d / m;
  idx->nlists = nlists;
  idx->K = coarse ? nlists : 0;
  idx->h_lanes = lanes;
  idx->h_count = count;
  idx->h_chunk_off.assign(nlists + 1, 0);
  for (int L = 0; L < nlists; L++) {
    const int64_t nch = (lanes[L] + kChunkCodes - 1) / kChunkCodes;
    idx->h_chunk_off[L + 1] = idx->h_chunk_off[L] + nch;
    idx->max_list_chunks = std::max(idx->max_list_chunks, nch);
  }
  idx->total_chunks = idx->h_chunk_off[nlists];
  const cudaMemcpyKind ck = coarse_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  const cudaMemcpyKind mk = model_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (coarse) {
    const size_t cb = (size_t)nlists * d * 4;
    QADC_CUDA(cudaMalloc(&idx->coarse, cb));
    QADC_CUDA(cudaMalloc(&idx->coarseT, cb));
    QADC_CUDA(cudaMemcpy(idx->coarse, coarse, cb, ck));
    k_transpose<<<gridn((int64_t)nlists * d), 256>>>(idx->coarse, nlists, d, idx->coarseT);
    QADC_CUDA(cudaMalloc(&idx->cnorm, (size_t)nlists * 4));
    launch_cnorm(idx->coarse, nlists, d, idx->cnorm, 0);
    if (probe_tc_supported(nlists, d, 1)) {
      if (int rc = probe_tc_prepare(idx->coarse, nlists, d, &idx->pmu, &idx->pcsplit, &idx->pcn2, 0))
        return rc;
      idx->bytes += (int64_t)(nlists + 255) / 256 * 256 * 3 * d * 2 + (int64_t)nlists * 4 + d * 4;
    }
    idx->bytes += 2 * (int64_t)cb + (int64_t)nlists * 4;
  }
  const size_t bb = (size_t)m * 16 * (d / m) * 4;
  QADC_CUDA(cudaMalloc(&idx->codebooks, bb));
  QADC_CUDA(cudaMemcpy(idx->codebooks, codebooks, bb, mk));
  if (rotation) {
    QADC_CUDA(cudaMalloc(&idx->rotation, (size_t)d * d * 4));
    QADC_CUDA(cudaMemcpy(idx->rotation, rotation, (size_t)d * d * 4, mk));
    QADC_CUDA(cudaMalloc(&idx->rotationT, (size_t)d * d * 4));
    k_transpose<<<gridn((int64_t)d * d), 256>>>(idx->rotation, d, d, idx->rotationT);
    QADC_CUDA(cudaGetLastError());
  }
  QADC_CUDA(cudaMalloc(&idx->chunk_off, (nlists + 1) * 8));
  QADC_CUDA(cudaMalloc(&idx->lanes, nlists * 8));
  QADC_CUDA(cudaMalloc(&idx->count, nlists * 8));
  QADC_CUDA(cudaMalloc(&idx->scan_count, nlists * 8));
  QADC_CUDA(cudaMemcpy(idx->scan_count, count.data(), nlists * 8, cudaMemcpyHostToDevice));
  QADC_CUDA(cudaMemcpy(idx->chunk_off, idx->h_chunk_off.data(), (nlists + 1) * 8, cudaMemcpyHostToDevice));
  QADC_CUDA(cudaMemcpy(idx->lanes, lanes.data(), nlists * 8, cudaMemcpyHostToDevice));
  QADC_CUDA(cudaMemcpy(idx->count, count.data(), nlists * 8, cudaMemcpyHostToDevice));
  return kOk;
}
}  // namespace

extern "C" void qadc_b200_index_destroy(qadc_b200_index *idx) {
  if (!idx) return;
  if (idx->own_prefix) {
    cudaFree(idx->pcodes); cudaFree(idx->pids); cudaFree(idx->pchunk_off); cudaFree(idx->planes);
  }
  cudaFree(idx->coarse); cudaFree(idx->coarseT); cudaFree(idx->cnorm); cudaFree(idx->pmu); cudaFree(idx->pcsplit); cudaFree(idx->pcn2); cudaFree(idx->codebooks); cudaFree(idx->rotation); cudaFree(idx->rotationT);
  cudaFree(idx->codes); cudaFree(idx->codes_cm); cudaFree(idx->valid); cudaFree(idx->ids); cudaFree(idx->chunk_list);
  cudaFree(idx->chunk_off); cudaFree(idx->lanes); cudaFree(idx->count); cudaFree(idx->scan_count);
  delete idx;
}

extern "C" int64_t qadc_b200_index_bytes(const qadc_b200_index *idx) { return idx ? idx->bytes : 0; }

extern "C" int qadc_b200_index_create(int d, int m, int nlists, const float *coarse,
                                      const uint8_t *blocks, const int64_t *blk_off,
                                      const int64_t *ids, const int64_t *count,
                                      const float *codebooks, const float *rotation,
                                      qadc_b200_index **out) {
  g_err.clear();
  if (!out || !blk_off || !count || !codebooks) return arg_error("null argument");
  *out = nullptr;
  std::vector<int64_t> lanes(nlists > 0 ? nlists : 0), cnt(nlists > 0 ? nlists : 0);
  for (int L = 0; L < nlists; L++) {
    lanes[L] = 16 * (blk_off[L + 1] - blk_off[L]);
    cnt[L] = count[L];
    if (lanes[L] < 0 || cnt[L] < 0 || cnt[L] > lanes[L]) return arg_error("invalid list geometry");
  }
  qadc_b200_index *idx = new qadc_b200_index();
  int rc = index_common(d, m, nlists, coarse, false, codebooks, rotation, false, lanes, cnt, idx);
  uint8_t *db = nullptr;
  int64_t *doff = nullptr, *dids = nullptr;
  const int64_t nb = nlists > 0 ? blk_off[nlists] : 0;
  if (!rc) rc = upload(&db, blocks, nb * (m / 2) * 16);
  if (!rc) rc = upload(&doff, blk_off, (int64_t)nlists + 1);
  if (!rc) rc = upload(&dids, ids, nb * 16);
  if (!rc) rc = pack_from_blocks(idx, db, doff, dids, 0);
  if (!rc) alias_prefix(idx);
  if (!rc) rc = cudaDeviceSynchronize() == cudaSuccess ? kOk : cuda_fail(cudaGetLastError(), "pack");
  cudaFree(db);
  cudaFree(doff);
  cudaFree(dids);
  if (rc) {
    qadc_b200_index_destroy(idx);
    return rc;
  }
  *out = idx;
  return kOk;
}

extern "C" int qadc_b200_index_create_device(int d, int m, int nlists, const float *coarse,
                                             const uint8_t *codes, const int64_t *row_off,
                                             const int64_t *ids, const float *codebooks,
                                             const float *rotation, qadc_b200_index **out) {
  g_err.clear();
  if (!out || !row_off || !codebooks) return arg_error("null argument");
  *out = nullptr;
  if (nlists < 1) return arg_error("index needs at least one list");
  std::vector<int64_t> h_off(nlists + 1);
  QADC_CUDA(cudaMemcpy(h_off.data(), row_off, (nlists + 1) * 8, cudaMemcpyDeviceToHost));
  std::vector<int64_t> lanes(nlists), cnt(nlists);
  for (int L = 0; L < nlists; L++) {
    lanes[L] = cnt[L] = h_off[L + 1] - h_off[L];
    if (lanes[L] < 0) return arg_error("row offsets must be non-decreasing");
  }
  qadc_b200_index *idx = new qadc_b200_index();
  int rc = index_common(d, m, nlists, coarse, true, codebooks, rotation, true, lanes, cnt, idx);
  if (!rc) rc = pack_from_rows(idx, codes, row_off, ids, 0);
  if (!rc) alias_prefix(idx);
  if (!rc) rc = cudaDeviceSynchronize() == cudaSuccess ? kOk : cuda_fail(cudaGetLastError(), "pack");
  if (rc) {
    qadc_b200_index_destroy(idx);
    return rc;
  }
  *out = idx;
  return kOk;
}

extern "C" int qadc_b200_index_set_prefix_device(qadc_b200_index *idx, const uint8_t *rows,
                                                 const int64_t *row_off, const int64_t *ids,
                                                 const int64_t *full_count) {
  g_err.clear();
  if (!idx || !row_off || !full_count) return arg_error("null argument");
  const int nl = idx->nlists;
  std::vector<int64_t> h_off(nl + 1);
  QADC_CUDA(cudaMemcpy(h_off.data(), row_off, (nl + 1) * 8, cudaMemcpyDeviceToHost));
  qadc_b200_index tmp;
  tmp.d = idx->d;
  tmp.m = idx->m;
  tmp.nlists = nl;
  std::vector<int64_t> lanes(nl);
  tmp.h_chunk_off.assign(nl + 1, 0);
  for (int L = 0; L < nl; L++) {
    lanes[L] = h_off[L + 1] - h_off[L];
    if (lanes[L] < 0) return arg_error("prefix row offsets must be non-decreasing");
    if (full_count[L] < lanes[L]) return arg_error("prefix longer than the list");
    tmp.h_chunk_off[L + 1] = tmp.h_chunk_off[L] + (lanes[L] + kChunkCodes - 1) / kChunkCodes;
  }
  tmp.total_chunks = tmp.h_chunk_off[nl];
  QADC_CUDA(cudaMalloc(&tmp.chunk_off, (nl + 1) * 8));
  QADC_CUDA(cudaMalloc(&tmp.lanes, nl * 8));
  QADC_CUDA(cudaMemcpy(tmp.chunk_off, tmp.h_chunk_off.data(), (nl + 1) * 8, cudaMemcpyHostToDevice));
  QADC_CUDA(cudaMemcpy(tmp.lanes, lanes.data(), nl * 8, cudaMemcpyHostToDevice));
  int rc = pack_from_rows(&tmp, rows, row_off, ids, 0);
  if (!rc) rc = cudaDeviceSynchronize() == cudaSuccess ? kOk : cuda_fail(cudaGetLastError(), "pack prefix");
  cudaFree(tmp.valid);
  cudaFree(tmp.chunk_list);
  if (rc) {
    cudaFree(tmp.codes); cudaFree(tmp.ids); cudaFree(tmp.chunk_off); cudaFree(tmp.lanes);
    return rc;
  }
  if (idx->own_prefix) {
    cudaFree(idx->pcodes); cudaFree(idx->pids); cudaFree(idx->pchunk_off); cudaFree(idx->planes);
  }
  idx->pcodes = tmp.codes;
  idx->pids = tmp.ids;
  idx->pchunk_off = tmp.chunk_off;
  idx->planes = tmp.lanes;
  idx->own_prefix = true;
  idx->h_count.assign(full_count, full_count + nl);
  QADC_CUDA(cudaMemcpy(idx->count, full_count, nl * 8, cudaMemcpyHostToDevice));
  return kOk;
}

extern "C" int qadc_b200_search_batch(qadc_b200_index *idx, const float *queries, int nq, int R,
                                      int ma, int init, unsigned flags, const float *lut_in,
                                      const int64_t *cells_in, int64_t *out_ids, float *out_d,
                                      int32_t *out_n, void *stream, int64_t *stats) {
  g_err.clear();
  if (!idx) return arg_error("null index");
  if (R < 1) return arg_error("R must be positive");
  if (init < 1) return arg_error("init must be positive");
  if (nq < 0) return arg_error("nq must be non-negative");
  if (idx->K) {
    if (ma < 1) return arg_error("ma must be positive");
    if (ma > idx->K) return arg_error("ma exceeds the cell count K");
  }
  if ((flags & QADC_B200_LUT_IN) && (!lut_in || (idx->K && !cells_in)))
    return arg_error("LUT injection needs lut_in (and cells_in for an IVF index)");
  if (R > 1 << 20) return arg_error("R too large");
  cudaStream_t st = (cudaStream_t)stream;
  retain_pool_memory();
  const int nslots = idx->K ? ma : 1;
  const bool host = flags & QADC_B200_HOST_IO;
  DevBuf<float> dq, dd, dl;
  DevBuf<int64_t> di, dc;
  DevBuf<int32_t> dn;
  const float *q = queries, *lin = (flags & QADC_B200_LUT_IN) ? lut_in : nullptr;
  const int64_t *cin = (flags & QADC_B200_LUT_IN) ? cells_in : nullptr;
  int64_t *oi = out_ids;
  float *od = out_d;
  int32_t *on = out_n;
  if (host) {
    if (dq.alloc((int64_t)nq * idx->d, st) || di.alloc((int64_t)nq * R, st) ||
        dd.alloc((int64_t)nq * R, st) || dn.alloc(nq, st))
      return cuda_fail(cudaGetLastError(), "alloc host io");
    QADC_CUDA(cudaMemcpyAsync(dq.p, queries, (size_t)nq * idx->d * 4, cudaMemcpyHostToDevice, st));
    q = dq.p;
    if (lin) {
      if (dl.alloc((int64_t)nq * nslots * idx->m * 16, st)) return kErrCuda;
      QADC_CUDA(cudaMemcpyAsync(dl.p, lut_in, (size_t)nq * nslots * idx->m * 64, cudaMemcpyHostToDevice, st));
      lin = dl.p;
      if (cin) {
        if (dc.alloc((int64_t)nq * nslots, st)) return kErrCuda;
        QADC_CUDA(cudaMemcpyAsync(dc.p, cells_in, (size_t)nq * nslots * 8, cudaMemcpyHostToDevice, st));
        cin = dc.p;
      }
    }
    oi = di.p;
    od = dd.p;
    on = dn.p;
  }
  SearchStats ss;
  int rc = search_impl(idx, q, nq, R, ma, init, lin, cin, oi, od, on, st, ss,
                       candidate_capacity(nq, R), (flags & QADC_B200_NO_FSAT) != 0,
                       (flags & QADC_B200_SCAN_PRMT) != 0, (flags & QADC_B200_SCAN_TC) != 0,
                       (flags & QADC_B200_SCAN_TC1) != 0, (flags & QADC_B200_SCAN_TCW) != 0);
  if (rc) return rc;
  if (host) {
    QADC_CUDA(cudaMemcpyAsync(out_ids, oi, (size_t)nq * R * 8, cudaMemcpyDeviceToHost, st));
    QADC_CUDA(cudaMemcpyAsync(out_d, od, (size_t)nq * R * 4, cudaMemcpyDeviceToHost, st));
    QADC_CUDA(cudaMemcpyAsync(out_n, on, (size_t)nq * 4, cudaMemcpyDeviceToHost, st));
    QADC_CUDA(cudaStreamSynchronize(st));
  }
  write_stats(ss, stats);
  return kOk;
}

namespace {
int check_search_args(const qadc_b200_index *idx, int nq, int R, int ma, int init) {
  if (!idx) return arg_error("null index");
  if (R < 1) return arg_error("R must be positive");
  if (init < 1) return arg_error("init must be positive");
  if (nq < 0) return arg_error("nq must be non-negative");
  if (idx->K && (ma < 1 || ma > idx->K)) return arg_error("ma must be in 1..K");
  if (R > 1 << 20) return arg_error("R too large");
  return kOk;
}
}  // namespace

extern "C" int qadc_b200_search_prepare(qadc_b200_index *idx, const float *queries, int nq, int R,
                                        int ma, int init, unsigned flags, const float *lut_in,
                                        const int64_t *cells_in, int64_t *cells, uint32_t *qt,
                                        float *qmin_f, float *delta_f, uint8_t *depth,
                                        float *qmax, uint32_t *M_bits, int32_t *fsat_n,
                                        float *fsat_mid, int64_t *fsat_id, void *stream,
                                        int64_t *stats) {
  g_err.clear();
  if (int rc = check_search_args(idx, nq, R, ma, init)) return rc;
  const bool inj = flags & QADC_B200_LUT_IN;
  if (inj && (!lut_in || (idx->K && !cells_in)))
    return arg_error("LUT injection needs lut_in (and cells_in for an IVF index)");
  if (!qt || !qmin_f || !delta_f || !depth || !qmax || !M_bits || !fsat_n || !fsat_mid ||
      !fsat_id || (idx->K && !cells) || (nq > 0 && !queries && !inj))
    return arg_error("null argument");
  if (flags & QADC_B200_HOST_IO) return arg_error("search_prepare takes device pointers only");
  cudaStream_t st = (cudaStream_t)stream;
  retain_pool_memory();
  SearchStats ss;
  int rc = prepare_impl(idx, queries, nq, R, ma, init, inj ? lut_in : nullptr,
                        inj ? cells_in : nullptr, (flags & QADC_B200_NO_FSAT) != 0, st, ss,
                        idx->K ? cells : nullptr, qt, qmin_f, delta_f, depth, qmax,
                        (unsigned *)M_bits, fsat_n, fsat_mid, fsat_id);
  if (rc) return rc;
  if (stats) {
    QADC_CUDA(cudaStreamSynchronize(st));
    float t = 0.f;
    cudaEvent_t *ev = phase_events();
    cudaEventElapsedTime(&t, ev[kEvStart], ev[kEvProbe]);
    ss.probe_us += t * 1e3;
    cudaEventElapsedTime(&t, ev[kEvProbe], ev[kEvTables]);
    ss.tables_us += t * 1e3;
    write_stats(ss, stats);
  }
  return kOk;
}

extern "C" int qadc_b200_search_scan(qadc_b200_index *idx, int nq, int R, int ma, int init,
                                     unsigned flags, const int64_t *cells, const uint32_t *qt,
                                     const float *qmin_f, const float *delta_f,
                                     const uint8_t *depth, uint32_t *M_bits,
                                     const int32_t *fsat_n, const float *fsat_mid,
                                     const int64_t *fsat_id, int64_t *out_ids, float *out_d,
                                     int32_t *out_n, void *stream, int64_t *stats) {
  g_err.clear();
  if (int rc = check_search_args(idx, nq, R, ma, init)) return rc;
  if (!qt || !qmin_f || !delta_f || !depth || !M_bits || !fsat_n || !fsat_mid || !fsat_id ||
      (idx->K && !cells) || !out_ids || !out_d || !out_n)
    return arg_error("null argument");
  if (flags & QADC_B200_HOST_IO) return arg_error("search_scan takes device pointers only");
  cudaStream_t st = (cudaStream_t)stream;
  retain_pool_memory();
  Prep p;
  p.cells = idx->K ? cells : nullptr;
  p.qt = qt;
  p.qmin_f = qmin_f;
  p.delta_f = delta_f;
  p.depth = depth;
  p.M_bits = (unsigned *)M_bits;
  p.fsat_n = fsat_n;
  p.fsat_mid = fsat_mid;
  p.fsat_id = fsat_id;
  SearchStats ss;
  int rc = scan_impl(idx, p, nq, R, ma, init, out_ids, out_d, out_n, st, ss,
                     candidate_capacity(nq, R), 0, (flags & QADC_B200_SCAN_PRMT) != 0,
                     (flags & QADC_B200_SCAN_TC) != 0, (flags & QADC_B200_SCAN_TC1) != 0,
                     (flags & QADC_B200_SCAN_TCW) != 0);
  if (rc) return rc;
  write_stats(ss, stats);
  return kOk;
}

extern "C" int qadc_b200_search_tables(qadc_b200_index *idx, const float *queries, int nq,
                                       int R, int ma, int init, int64_t *cells_out,
                                       float *lut_out, float *qmax_out, uint8_t *qt_out,
                                       float *qmin_out, float *delta_out, void *stream) {
  g_err.clear();
  if (!idx || !queries || !lut_out || !qmax_out || !qt_out || !qmin_out || !delta_out)
    return arg_error("null argument");
  if (R < 1 || init < 1 || nq < 0) return arg_error("invalid R / init / nq");
  if (idx->K && (ma < 1 || ma > idx->K)) return arg_error("ma must be in 1..K");
  if (idx->K && !cells_out) return arg_error("an IVF index needs cells_out");
  cudaStream_t st = (cudaStream_t)stream;
  retain_pool_memory();
  if (nq == 0) return kOk;
  const int nslots = idx->K ? ma : 1;
  const int64_t *cells = nullptr;
  if (idx->K) {
    index_probe(idx, queries, nq, ma, cells_out, st);
    cells = cells_out;
  }
  launch_residual_lut(idx, queries, cells, nq, nslots, lut_out, st);
  if (int rc = launch_qmax(idx, lut_out, cells, nq, nslots, R, init, qmax_out, st)) return rc;
  launch_quantize(lut_out, nq * nslots, idx->m, qmax_out, nslots, nullptr, nullptr, nullptr,
                  qmin_out, delta_out, nullptr, qt_out, st);
  QADC_CUDA(cudaGetLastError());
  return kOk;
}

extern "C" int qadc_b200_compute_tables(const float *codebooks, int m, int dsub, const float *y,
                                        int npairs, float *out, void *stream) {
  g_err.clear();
  if (m < 1 || m > QADC_MAX_M || dsub < 1 || npairs < 0) return arg_error("invalid geometry");
  launch_compute_tables(codebooks, m, dsub, y, npairs, out, (cudaStream_t)stream);
  QADC_CUDA(cudaGetLastError());
  return kOk;
}

extern "C" int qadc_b200_probe(const float *coarse, int K, int d, const float *queries, int nq,
                               int ma, int64_t *cells, float *residuals, void *stream) {
  g_err.clear();
  if (K < 1 || d < 1 || ma < 1 || ma > K || nq < 0) return arg_error("invalid probe geometry");
  cudaStream_t st = (cudaStream_t)stream;
  float *cT = nullptr;
  QADC_CUDA(cudaMallocAsync(&cT, (size_t)K * d * 4, st));
  k_transpose<<<gridn((int64_t)K * d), 256, 0, st>>>(coarse, K, d, cT);
  float *cn = nullptr;
  QADC_CUDA(cudaMallocAsync(&cn, (size_t)K * 4, st));
  launch_cnorm(coarse, K, d, cn, st);
  static const int probe_kind = scan_env_int("QADC_B200_PROBE", 2);
  bool done = false;
  if (probe_kind >= 2 && probe_tc_supported(K, d, ma)) {
    float *mu = nullptr, *cn2 = nullptr;
    void *cs = nullptr;
    if (probe_tc_prepare(coarse, K, d, &mu, &cs, &cn2, st) == kOk)
      done = launch_probe_tc(coarse, mu, cs, cn2, K, d, queries, nq, ma, cells, st);
    cudaStreamSynchronize(st);
    cudaFree(mu);
    cudaFree(cs);
    cudaFree(cn2);
  }
  if (!done && probe_kind >= 1) done = launch_probe_fast(cT, coarse, cn, K, d, queries, nq, ma, cells, st);
  if (!done) launch_probe(cT, K, d, queries, nq, ma, cells, st);
  cudaFreeAsync(cn, st);
  cudaFreeAsync(cT, st);
  if (residuals)
    k_residuals<<<gridn((int64_t)nq * ma * d), 256, 0, st>>>(queries, coarse, cells, nq, ma, d,
                                                             residuals);
  QADC_CUDA(cudaGetLastError());
  return kOk;
}

extern "C" int qadc_b200_quantize_tables(const float *tables, int npairs, int m, const double *qmin,
                                         const double *qmax, uint8_t *out, double *delta,
                                         void *stream) {
  g_err.clear();
  if (m < 1 || m > QADC_MAX_M || npairs < 0) return arg_error("invalid geometry");
  launch_quantize(tables, npairs, m, nullptr, 1, qmin, qmax, nullptr, nullptr, nullptr, delta, out,
                  (cudaStream_t)stream);
  QADC_CUDA(cudaGetLastError());
  return kOk;
}
