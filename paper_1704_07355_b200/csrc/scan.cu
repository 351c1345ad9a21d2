// Scan phase of adc.py:114-187 (qadc branch), batched: the B200 analogue of
// qadc_scan_u8 (scan_kernels.c:318-382) plus the bounded heap
// (scan_kernels.c:22-74, 279-308), restructured for a GPU:
//
//  * one CTA = 4 warps works on a (list, query tile, chunk range) item
//    pulled from a global counter (persistent grid, 148 SMs x occupancy);
//  * a warp owns one 256-code chunk at a time, a lane one octet of codes;
//    per sub-quantizer pair the lane turns its two code words into PRMT
//    selectors once and reuses them for every query of the tile;
//  * lookups: PRMT on the two register halves of a 16-entry byte table
//    (entries <= 127, so PRMT's sign-replicate mode zeroes the wrong half),
//    byte sums of two sub-quantizers (<= 254, carry-free), widened into
//    16-bit lanes via acc_a = sum(s) and acc_o = sum(odd bytes of s):
//    even lanes = acc_a - (acc_o << 8). The adds run on the FMA pipe
//    (IMAD) and the lookups on the ALU pipe (PRMT) so both pipes issue;
//  * exact lane distance min(255, sum) (scan_kernels.c:137-167);
//  * selection: a lane survives if its sum is <= the tile's threshold for
//    that query, derived from a running per-query distance bound M (a
//    midpoint value with >= R candidates at or below it). Survivors go to
//    per-warp shared-memory buffers; a full buffer is tightened to its
//    R-th smallest value (which also lowers the global M with atomicMin)
//    and compacted. At the end of the item survivors with midpoint <= M
//    are appended to a per-query global candidate list; select.cu picks
//    the exact top-R by (midpoint, id).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "internal.cuh"

namespace qadc {
namespace {

constexpr int kWarps = 4;
constexpr unsigned kFull = 0xffffffffu;

struct Smem {
  int item;
  int pair_count;
  int64_t chunk_begin;
  int query[16];
  float qmin[16];
  float delta[16];
  float hinv[16];  // 1 / histogram bucket width of the query (0: no histogram)
  int thr[kWarps][16];
  unsigned kbias[kWarps][16];
  unsigned mc[kWarps][16];
  int bn[kWarps][16];
  int pend[kWarps][16];  // appended since this warp last read the global histogram
};

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// Code-word prefetch that stays where it is written: volatile asm is not
// reordered across the (volatile) table loads, so the next iteration's
// words are requested at the top of the current one instead of being sunk
// next to their first use (ncu: the sunk loads left ~25 % of the PRMT
// scan's warp samples on long_scoreboard).
__device__ __forceinline__ uint32_t ldg_early(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Bulk L2 prefetch of a contiguous range (one instruction for a whole code
// chunk): a warp asks for its next chunk while it scans the current one, so
// the register prefetch of the scan loop hits L2 instead of waiting on HBM
// (configs[4] scan 39.7 -> 38.7 ms). Staging the words through cp.async
// into shared memory instead measured slower (39.9 ms: the 4 KB of slots
// per CTA cost occupancy), and so did a two-iteration register lead
// (41.6 ms).
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ unsigned kbias_of(int thr) {
  return (0x8000u - (unsigned)(thr + 1)) * 0x10001u;
}

// Every candidate a warp appends to its buffer is counted once in a
// per-query two-level histogram of midpoints (bucket b = floor(mid / w),
// 32 coarse x 32 fine bins). Lanes are tested exactly once, so the counts
// are of distinct members of the candidate set, and the R-th smallest
// bucket bounds the R-th best candidate seen by ANY warp so far:
// M = (b + 2) * w (one bucket of slack absorbs fp32 rounding of b). The
// global bound therefore tracks the union of all warps' scans, not only
// the best single warp.
__device__ __forceinline__ unsigned hist_bound(const ScanArgs &a, int query) {
  const int lane = threadIdx.x & 31;
  const float hw = a.hist_w[query];
  if (!(hw > 0.f)) return 0x7f800000u;
  // lane l reads fine bins 32 l .. 32 l + 31 (8 independent 16-byte L2
  // reads: one round trip per refresh; counts read early only make the
  // bound looser)
  const uint4 *h = (const uint4 *)(a.hist + (size_t)query * kHistWords) + lane * 8;
  uint4 r[8];
#pragma unroll
  for (int i = 0; i < 8; i++) r[i] = __ldcg(h + i);
  unsigned c = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) c += r[i].x + r[i].y + r[i].z + r[i].w;
  unsigned incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  const unsigned R = (unsigned)a.R;
  const unsigned hit = __ballot_sync(kFull, incl >= R);
  if (!hit) return 0x7f800000u;
  const int k = __ffs(hit) - 1;
  int b = 31;
  if (lane == k) {  // this lane's bins, from its exclusive prefix
    unsigned cum = incl - c;
    bool found = false;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const unsigned w4[4] = {r[i].x, r[i].y, r[i].z, r[i].w};
#pragma unroll
      for (int j = 0; j < 4; j++) {
        cum += w4[j];
        if (!found && cum >= R) {
          b = 4 * i + j;
          found = true;
        }
      }
    }
  }
  b = k * 32 + __shfl_sync(kFull, b, k);
  return fbits(__fmul_rn((float)(b + 2), hw));
}

// Two-level variant for the PRMT scan, whose compute warps refresh the
// bound inline: 2 x 128 bytes (coarse sums, then one row of fine bins)
// instead of the whole histogram. Needs the coarse sums kept by that
// kernel's appends (h[kHistBins + b / 32]).
__device__ __forceinline__ unsigned hist_bound2(const ScanArgs &a, int query) {
  const int lane = threadIdx.x & 31;
  const float hw = a.hist_w[query];
  if (!(hw > 0.f)) return 0x7f800000u;
  const unsigned *h = a.hist + (size_t)query * kHistWords;
  const unsigned c = *(volatile const unsigned *)&h[kHistBins + lane];
  unsigned incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  const unsigned R = (unsigned)a.R;
  const unsigned hit = __ballot_sync(kFull, incl >= R);
  if (!hit) return 0x7f800000u;
  const int k = __ffs(hit) - 1;
  const unsigned base = __shfl_sync(kFull, incl - c, k);
  const unsigned f = *(volatile const unsigned *)&h[k * 32 + lane];
  unsigned fi = f;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, fi, o);
    if (lane >= o) fi += y;
  }
  const unsigned hit2 = __ballot_sync(kFull, base + fi >= R);
  const int b = k * 32 + (hit2 ? __ffs(hit2) - 1 : 31);
  return fbits(__fmul_rn((float)(b + 2), hw));
}

// Global append of every buffered entry of (warp, q) whose midpoint is <=
// the query's current bound; empties the buffer.
__device__ __noinline__ void flush_buffer(const ScanArgs &a, Smem &s, uint32_t *buf, int w, int q) {
  const int lane = threadIdx.x & 31;
  const int n = s.bn[w][q];
  const int query = s.query[q];
  const float qmin = s.qmin[q], delta = s.delta[q];
  const float Mg = __uint_as_float(*(volatile unsigned *)&a.M_bits[query]);
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    bool keep = false;
    float mid = 0.f;
    uint32_t e = 0;
    if (i < n) {
      e = buf[i];
      mid = midpoint(qmin, delta, (int)(e >> 24));
      keep = mid <= Mg;
    }
    const unsigned bal = __ballot_sync(kFull, keep);
    if (!bal) continue;
    unsigned pos = 0;
    if (lane == 0) pos = atomicAdd(&a.cand_n[query], (unsigned)__popc(bal));
    pos = __shfl_sync(kFull, pos, 0);
    if (keep) {
      const unsigned slot = pos + __popc(bal & ((1u << lane) - 1));
      if (slot < (unsigned)a.cap_g) {
        const size_t o = (size_t)query * a.cap_g + slot;
        a.cand_mid[o] = mid;
        a.cand_id[o] = a.ids[s.chunk_begin * kChunkCodes + (e & 0xffffffu)];
      }
    }
  }
  __syncwarp();
  if (lane == 0) s.bn[w][q] = 0;
  __syncwarp();
}

// End-of-item flush of all of this warp's buffers (one per tile query):
// the queries' bounds are read in parallel (lane q), the survivors are
// counted per query, ONE atomicAdd per query claims their slots (lanes in
// parallel), then the entries are written. Two global round trips per
// item instead of two per query.
__device__ __noinline__ void flush_all(const ScanArgs &a, Smem &s, uint32_t *wbuf, int w,
                                       int nq_tile) {
  const int lane = threadIdx.x & 31;
  float Ml = 0.f;
  if (lane < nq_tile) Ml = __uint_as_float(*(volatile unsigned *)&a.M_bits[s.query[lane]]);
  unsigned mycnt = 0;
  for (int q = 0; q < nq_tile; q++) {
    const int n = s.bn[w][q];
    if (n == 0) continue;
    const uint32_t *buf = wbuf + q * a.cap_l;
    const float Mg = __shfl_sync(kFull, Ml, q);
    const float qmin = s.qmin[q], delta = s.delta[q];
    unsigned c = 0;
    for (int i = lane; i < n; i += 32) c += midpoint(qmin, delta, (int)(buf[i] >> 24)) <= Mg;
    c = __reduce_add_sync(kFull, c);
    if (lane == q) mycnt = c;
  }
  unsigned pos = 0;
  if (lane < nq_tile && mycnt) pos = atomicAdd(&a.cand_n[s.query[lane]], mycnt);
  for (int q = 0; q < nq_tile; q++) {
    const int n = s.bn[w][q];
    if (n == 0) continue;
    const uint32_t *buf = wbuf + q * a.cap_l;
    const float Mg = __shfl_sync(kFull, Ml, q);
    unsigned base = __shfl_sync(kFull, pos, q);
    const int query = s.query[q];
    const float qmin = s.qmin[q], delta = s.delta[q];
    for (int b0 = 0; b0 < n; b0 += 32) {
      const int i = b0 + lane;
      bool keep = false;
      float mid = 0.f;
      uint32_t e = 0;
      if (i < n) {
        e = buf[i];
        mid = midpoint(qmin, delta, (int)(e >> 24));
        keep = mid <= Mg;
      }
      const unsigned bal = __ballot_sync(kFull, keep);
      if (keep) {
        const unsigned slot = base + __popc(bal & ((1u << lane) - 1));
        if (slot < (unsigned)a.cap_g) {
          const size_t o = (size_t)query * a.cap_g + slot;
          a.cand_mid[o] = mid;
          a.cand_id[o] = a.ids[s.chunk_begin * kChunkCodes + (e & 0xffffffu)];
        }
      }
      base += __popc(bal);
    }
  }
  __syncwarp();
  if (lane < nq_tile) s.bn[w][lane] = 0;
  __syncwarp();
}

// Tighten (warp, q)'s threshold to the R-th smallest buffered value and
// drop entries above it. Requires bn >= R.
__device__ __noinline__ void compact_buffer(const ScanArgs &a, Smem &s, uint32_t *buf, int w, int q) {
  const int lane = threadIdx.x & 31;
  const int n = s.bn[w][q];
  // every buffered value is <= 254; n >= R, so the search is well founded
  // even if the threshold dropped after some entries were buffered
  int lo = 0, hi = 254;
  while (lo < hi) {  // smallest t with count(value <= t) >= R
    const int mid = (lo + hi) >> 1;
    int c = 0;
    for (int i = lane; i < n; i += 32) c += (int)(buf[i] >> 24) <= mid;
    c = __reduce_add_sync(kFull, c);
    if (c >= a.R) hi = mid; else lo = mid + 1;
  }
  const float qmin = s.qmin[q], delta = s.delta[q];
  const float Mt = midpoint(qmin, delta, lo);
  const int t_ext = q_threshold(Mt, qmin, delta);  // >= lo; covers midpoint ties
  const int thr = min(s.thr[w][q], t_ext);
  if (lane == 0) {
    atomicMin(&a.M_bits[s.query[q]], fbits(Mt));
    s.thr[w][q] = thr;
    s.kbias[w][q] = kbias_of(thr);
  }
  int out = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    uint32_t e = 0;
    bool keep = false;
    if (i < n) {
      e = buf[i];
      keep = (int)(e >> 24) <= thr;
    }
    const unsigned bal = __ballot_sync(kFull, keep);
    if (keep) buf[out + __popc(bal & ((1u << lane) - 1))] = e;
    out += __popc(bal);
  }
  __syncwarp();
  if (lane == 0) s.bn[w][q] = out;
  __syncwarp();
}

// Warp-wide count of the set bits of every lane's K-bit mask: codes in
// lanes below this one, and in the whole warp.
template <int K>
__device__ __forceinline__ void count_bits(uint32_t mk, int &before, int &total) {
  const unsigned lt = (1u << (threadIdx.x & 31)) - 1;
  before = 0;
  total = 0;
#pragma unroll
  for (int k = 0; k < K; k++) {
    const unsigned b = __ballot_sync(kFull, (mk >> k) & 1u);
    before += __popc(b & lt);
    total += __popc(b);
  }
}

// Append this lane's surviving codes (mask bit k = code base_idx + k of
// the item; byte k of v0:v1 = its lane distance) to (warp, q)'s buffer.
// K = 8: the caller checked that the buffer has room; K = 4: at most 128
// codes, the buffer keeps R + 128 slots (compact / flush when full).
template <int K>
__device__ __noinline__ void append(const ScanArgs &a, Smem &s, uint32_t *buf, int w, int q,
                                    uint32_t mask4, uint32_t vals, uint32_t vals_hi,
                                    uint32_t base_idx, int before, int total) {
  const int lane = threadIdx.x & 31;
  int n = s.bn[w][q];
  if (K == 4 && n + total > a.cap_l) {  // n > cap_l - 128 >= R
    if (n >= a.R) compact_buffer(a, s, buf, w, q);
    // re-filter with the (possibly) tightened threshold
    const int thr = s.thr[w][q];
#pragma unroll
    for (int k = 0; k < 4; k++)
      if ((int)((vals >> (8 * k)) & 255u) > thr) mask4 &= ~(1u << k);
    count_bits<4>(mask4, before, total);
    n = s.bn[w][q];
    if (n + total > a.cap_l) {
      flush_buffer(a, s, buf, w, q);
      n = 0;
    }
  }
  int off = n + before;
  const int query = s.query[q];
  const float hinv = s.hinv[q], qmin = s.qmin[q], delta = s.delta[q];
  unsigned *h = a.hist + (size_t)query * kHistWords;
#pragma unroll
  for (int k = 0; k < K; k++) {
    if (mask4 & (1u << k)) {
      const uint32_t v = ((k < 4 ? vals : vals_hi) >> (8 * (k & 3))) & 255u;
      buf[off++] = (v << 24) | (base_idx + k);
      if (hinv > 0.f) {
        // bucket floor(mid / w) up to one bucket either way (hist_bound's
        // (b + 2) * w keeps one bucket of slack)
        const int b = min((int)__fmul_rn(midpoint(qmin, delta, (int)v), hinv), kHistBins - 1);
        atomicAdd(&h[b], 1u);
        atomicAdd(&h[kHistBins + (b >> 5)], 1u);  // coarse sums for hist_bound2
      }
    }
  }
  const int pend = s.pend[w][q] + total;
  __syncwarp();
  if (lane == 0) {
    s.bn[w][q] = n + total;
    s.pend[w][q] = pend >= a.bound_every ? 0 : pend;
  }
  // the union of all warps' candidates may now bound the query tighter
  // (read once per bound_every appended candidates: the histogram read and
  // its two warp scans cost more than the appends themselves)
  if (pend >= a.bound_every) {
    const unsigned mb = hist_bound2(a, query);
    if (lane == 0 && mb < s.mc[w][q]) {
      atomicMin(&a.M_bits[query], mb);
      s.mc[w][q] = mb;
      const int t = q_threshold(__uint_as_float(mb), qmin, delta);
      if (t < s.thr[w][q]) {
        s.thr[w][q] = t;
        s.kbias[w][q] = kbias_of(t);
      }
    }
  }
  __syncwarp();
}

// Rare path of the per-chunk test: some lane of (warp, q) may qualify.
__device__ __noinline__ void candidates(const ScanArgs &a, Smem &s, uint32_t *buf, int w, int q,
                                        uint32_t E0, uint32_t O0, uint32_t E1, uint32_t O1,
                                        uint32_t valid8, int chunk_local) {
  const unsigned kb = s.kbias[w][q];
  const uint32_t pe0 = ~(E0 + kb) & 0x80008000u, po0 = ~(O0 + kb) & 0x80008000u;
  const uint32_t pe1 = ~(E1 + kb) & 0x80008000u, po1 = ~(O1 + kb) & 0x80008000u;
  uint32_t mask8 = ((pe0 >> 15) & 1u) | ((po0 >> 14) & 2u) | ((pe0 >> 29) & 4u) |
                   ((po0 >> 28) & 8u);
  mask8 |= (((pe1 >> 15) & 1u) | ((po1 >> 14) & 2u) | ((pe1 >> 29) & 4u) | ((po1 >> 28) & 8u))
           << 4;
  mask8 &= valid8;
  const uint32_t v0 = prmt(E0, O0, 0x6240), v1 = prmt(E1, O1, 0x6240);  // low bytes
  const uint32_t base_idx = (uint32_t)chunk_local * kChunkCodes + 8u * (threadIdx.x & 31);
  int before, total;
  count_bits<8>(mask8, before, total);
  if (s.bn[w][q] + total <= a.cap_l) {  // common case: all 8 codes per lane at once
    if (total) append<8>(a, s, buf, w, q, mask8, v0, v1, base_idx, before, total);
    return;
  }
  // at most 4 codes per lane per append: the buffer needs R + 128 slots
  count_bits<4>(mask8 & 0x0fu, before, total);
  if (total) append<4>(a, s, buf, w, q, mask8 & 0x0fu, v0, 0, base_idx, before, total);
  count_bits<4>(mask8 >> 4, before, total);
  if (total) append<4>(a, s, buf, w, q, mask8 >> 4, v1, 0, base_idx + 4, before, total);
}

// Refresh each query's threshold from the global bound (lanes in parallel).
__device__ __forceinline__ void refresh(const ScanArgs &a, Smem &s, int w, int nq_tile) {
  const int lane = threadIdx.x & 31;
  if (lane < nq_tile) {
    const unsigned mb = *(volatile unsigned *)&a.M_bits[s.query[lane]];
    if (mb != s.mc[w][lane]) {
      s.mc[w][lane] = mb;
      const int t = q_threshold(__uint_as_float(mb), s.qmin[lane], s.delta[lane]);
      if (t < s.thr[w][lane]) {
        s.thr[w][lane] = t;
        s.kbias[w][lane] = kbias_of(t);
      }
    }
  }
  __syncwarp();
}

// Exact lane sums of one chunk for QT queries: lane `lane` owns the octet
// of codes 8*lane .. 8*lane+7. Per sub-quantizer pair the two code words
// become PRMT selectors (low / high 16 bits; XOR 0x8888 flips bit 3 so the
// 8-15 half of the table answers), reused for every query. Lookups of D
// consecutive sub-quantizers are summed in bytes (sacc; carry-free because
// the tile's tables satisfy sum of D row maxima <= 255), then widened into
// 16-bit lanes: acc_a += sacc, acc_o += odd bytes of sacc; the even lanes
// are acc_a - (acc_o << 8). Adds run on the FMA pipe (IMAD), lookups on the
// ALU pipe (PRMT). Two pairs per iteration keep the body inside the
// instruction cache; code words are prefetched one pair ahead.
// One sub-quantizer pair (j, j+1) of the octet for every query of the tile.
template <int QT>
__device__ __forceinline__ void pair_lookups(uint32_t w0, uint32_t w1, int j, int m,
                                             uint32_t tab_sa, uint32_t one,
                                             uint32_t (&sacc)[QT][2]) {
  const uint32_t a0 = w0, a1 = w0 >> 16, a0x = w0 ^ 0x88888888u, a1x = a0x >> 16;
  const uint32_t b0 = w1, b1 = w1 >> 16, b0x = w1 ^ 0x88888888u, b1x = b0x >> 16;
#pragma unroll
  for (int q = 0; q < QT; q++) {
    const uint4 t = lds128(tab_sa + (uint32_t)((q * m + j) * 16));
    const uint4 u = lds128(tab_sa + (uint32_t)((q * m + j + 1) * 16));
    // codes 0-3 of the octet: sub-quantizers j and j+1, both table halves
    sacc[q][0] = imad(prmt(t.x, t.y, a0), one,
                 imad(prmt(t.z, t.w, a0x), one,
                 imad(prmt(u.x, u.y, b0), one,
                 imad(prmt(u.z, u.w, b0x), one, sacc[q][0]))));
    // codes 4-7
    sacc[q][1] = imad(prmt(t.x, t.y, a1), one,
                 imad(prmt(t.z, t.w, a1x), one,
                 imad(prmt(u.x, u.y, b1), one,
                 imad(prmt(u.z, u.w, b1x), one, sacc[q][1]))));
  }
}

template <int QT>
__device__ __forceinline__ void widen(uint32_t one, uint32_t (&sacc)[QT][2],
                                      uint32_t (&acc_a)[QT][2], uint32_t (&acc_o)[QT][2]) {
#pragma unroll
  for (int q = 0; q < QT; q++) {
#pragma unroll
    for (int h = 0; h < 2; h++) {
      acc_a[q][h] = imad(sacc[q][h], one, acc_a[q][h]);
      acc_o[q][h] = imad(prmt(sacc[q][h], 0, 0x4341), one, acc_o[q][h]);
      sacc[q][h] = 0;
    }
  }
}

// Lane sums of one chunk, two sub-quantizer pairs per iteration. The code
// words of the NEXT iteration's two pairs (possibly the first pairs of the
// warp's next chunk, cw_next) are loaded at the top of the iteration and
// moved into place at its end, ~170 instructions later, so no L2 latency
// is exposed and no register move waits on an in-flight load. Groups of D
// sub-quantizers are summed in bytes (sacc), then widened.
template <int D, int MC, int QT>
__device__ __forceinline__ void lane_sums(const uint32_t *__restrict__ cw,
                                          const uint32_t *__restrict__ cw_next, int m,
                                          uint32_t tab_sa, uint32_t one, uint32_t (&c)[4],
                                          uint32_t (&acc_a)[QT][2], uint32_t (&acc_o)[QT][2]) {
  uint32_t sacc[QT][2];
#pragma unroll
  for (int q = 0; q < QT; q++)
    acc_a[q][0] = acc_a[q][1] = acc_o[q][0] = acc_o[q][1] = sacc[q][0] = sacc[q][1] = 0;
  if (!MC && m < 4) {  // a single pair per chunk
    pair_lookups<QT>(__ldg(cw), __ldg(cw + 32), 0, m, tab_sa, one, sacc);
    widen<QT>(one, sacc, acc_a, acc_o);
    return;
  }
#pragma unroll 1
  for (int j = 0; j < m; j += 4) {
    // next iteration: pairs (jn, jn + 2) of this chunk, or of the next one
    const bool same = j + 4 < m;
    const uint32_t *base = same ? cw : cw_next;
    const int jn = same ? j + 4 : 0;
    const int jn2 = jn + 2 < m ? jn + 2 : jn;  // absent second pair: any valid row
    const uint32_t n0 = ldg_early(base + jn * 32), n1 = ldg_early(base + (jn + 1) * 32);
    const uint32_t n2 = ldg_early(base + jn2 * 32), n3 = ldg_early(base + (jn2 + 1) * 32);
    pair_lookups<QT>(c[0], c[1], j, m, tab_sa, one, sacc);
    if (D == 2) widen<QT>(one, sacc, acc_a, acc_o);
    const bool second = (MC && MC % 4 == 0) || j + 2 < m;
    if (second) pair_lookups<QT>(c[2], c[3], j + 2, m, tab_sa, one, sacc);
    if ((D == 2 && second) || (D != 2 && (((j + 4) % D) == 0 || j + 4 >= m)))
      widen<QT>(one, sacc, acc_a, acc_o);
    c[0] = n0;
    c[1] = n1;
    c[2] = n2;
    c[3] = n3;
  }
}

// The chunk loop of one work item for a fixed byte-sum depth D: lane sums,
// then one combined threshold test per query and ONE warp reduction for
// the whole tile; the per-lane candidate masks are built only for the
// queries that have a qualifying lane (rare once the bound has converged).
template <int D, int MC, int QT>
__device__ __forceinline__ void chunk_loop(const ScanArgs &a, Smem &s, const WorkItem &it,
                                           uint32_t *wbuf, int m, uint32_t tab_sa,
                                           uint32_t one, int nq_tile) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int iter = 0;
  uint32_t ring[4] = {0, 0, 0, 0};  // words of pairs 0 and 1 of the next chunk
  if (m >= 4 && it.chunk_begin + w < it.chunk_end) {
    const uint32_t *c0 = a.codes + (size_t)(it.chunk_begin + w) * m * 32 + lane;
    ring[0] = __ldg(c0);
    ring[1] = __ldg(c0 + 32);
    ring[2] = __ldg(c0 + 64);
    ring[3] = __ldg(c0 + 96);
  }
  for (int64_t g = it.chunk_begin + w; g < it.chunk_end; g += kWarps, iter++) {
    if ((iter & 3) == 3) refresh(a, s, w, nq_tile);
    if (lane == 0 && g + kWarps < it.chunk_end)
      prefetch_l2(a.codes + (size_t)(g + kWarps) * m * 32, (uint32_t)m * 128);
    const uint32_t valid8 = a.valid[g * 32 + lane];
    const uint32_t *cw = a.codes + (size_t)g * m * 32 + lane;
    // no next chunk: prefetch reads this chunk again (valid memory, unused)
    const uint32_t *cw_next = g + kWarps < it.chunk_end ? cw + (size_t)kWarps * m * 32 : cw;
    uint32_t acc_a[QT][2], acc_o[QT][2];
    lane_sums<D, MC, QT>(cw, cw_next, m, tab_sa, one, ring, acc_a, acc_o);
    // ---- threshold test: 16-bit lanes, bit 15 clear <=> lane <= thr ----
    uint32_t hitq = 0;
#pragma unroll
    for (int q = 0; q < QT; q++) {
      const unsigned kb = s.kbias[w][q];
      const uint32_t O0 = acc_o[q][0], E0 = acc_a[q][0] - (O0 << 8);
      const uint32_t O1 = acc_o[q][1], E1 = acc_a[q][1] - (O1 << 8);
      const uint32_t all = (E0 + kb) & (O0 + kb) & (E1 + kb) & (O1 + kb);
      hitq |= ((all & 0x80008000u) != 0x80008000u) ? (1u << q) : 0u;
    }
    hitq = __reduce_or_sync(kFull, hitq);
    if (hitq) {
      const int chunk_local = (int)(g - it.chunk_begin);
#pragma unroll
      for (int q = 0; q < QT; q++) {
        if (hitq & (1u << q)) {
          const uint32_t O0 = acc_o[q][0], E0 = acc_a[q][0] - (O0 << 8);
          const uint32_t O1 = acc_o[q][1], E1 = acc_a[q][1] - (O1 << 8);
          candidates(a, s, wbuf + q * a.cap_l, w, q, E0, O0, E1, O1, valid8, chunk_local);
        }
      }
    }
  }
}

// Fixed-m chunk loop (MC % 8 == 0, byte-sum depth D >= 8): each warp takes
// a CONTIGUOUS run of the item's chunks, so its code words form one linear
// stream of 32-word rows. The body covers 8 sub-quantizers with two
// register sets in ping-pong (A: rows r..r+3, B: rows r+4..r+7), each
// loaded half a body before use; no register moves, no per-row address
// selection, one pointer increment per 8 rows. The prefetch runs up to 12
// rows past the warp's last chunk (the code array keeps one chunk of
// padding).
template <int D, int MC, int QT>
__device__ __forceinline__ void chunk_loop_lin(const ScanArgs &a, Smem &s, const WorkItem &it,
                                               uint32_t *wbuf, uint32_t tab_sa, uint32_t one,
                                               int nq_tile) {
  static_assert(MC % 8 == 0 && D >= 8 && MC % D == 0, "linear loop shape");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t n = it.chunk_end - it.chunk_begin;
  const int64_t per = (n + kWarps - 1) / kWarps;
  const int64_t g0 = it.chunk_begin + min(n, w * per);
  const int64_t g1 = it.chunk_begin + min(n, (w + 1) * per);
  if (g0 >= g1) return;
  const uint32_t *p = a.codes + (size_t)g0 * MC * 32 + lane;
  uint32_t A[4] = {__ldg(p), __ldg(p + 32), __ldg(p + 64), __ldg(p + 96)};
  uint32_t B[4];
  int iter = 0;
  for (int64_t g = g0; g < g1; g++, iter++) {
    if ((iter & 3) == 3) refresh(a, s, w, nq_tile);
    if (lane == 0 && g + 2 < g1) prefetch_l2(a.codes + (size_t)(g + 2) * MC * 32, MC * 128u);
    const uint32_t valid8 = a.valid[g * 32 + lane];
    uint32_t acc_a[QT][2], acc_o[QT][2], sacc[QT][2];
#pragma unroll
    for (int q = 0; q < QT; q++)
      acc_a[q][0] = acc_a[q][1] = acc_o[q][0] = acc_o[q][1] = sacc[q][0] = sacc[q][1] = 0;
#pragma unroll 1
    for (int j = 0; j < MC; j += 8) {
#pragma unroll
      for (int r = 0; r < 4; r++) B[r] = ldg_early(p + 128 + 32 * r);
      pair_lookups<QT>(A[0], A[1], j, MC, tab_sa, one, sacc);
      pair_lookups<QT>(A[2], A[3], j + 2, MC, tab_sa, one, sacc);
#pragma unroll
      for (int r = 0; r < 4; r++) A[r] = ldg_early(p + 256 + 32 * r);
      pair_lookups<QT>(B[0], B[1], j + 4, MC, tab_sa, one, sacc);
      pair_lookups<QT>(B[2], B[3], j + 6, MC, tab_sa, one, sacc);
      p += 256;
      if ((j + 8) % D == 0) widen<QT>(one, sacc, acc_a, acc_o);
    }
    // ---- threshold test: 16-bit lanes, bit 15 clear <=> lane <= thr ----
    uint32_t hitq = 0;
#pragma unroll
    for (int q = 0; q < QT; q++) {
      const unsigned kb = s.kbias[w][q];
      const uint32_t O0 = acc_o[q][0], E0 = acc_a[q][0] - (O0 << 8);
      const uint32_t O1 = acc_o[q][1], E1 = acc_a[q][1] - (O1 << 8);
      const uint32_t all = (E0 + kb) & (O0 + kb) & (E1 + kb) & (O1 + kb);
      hitq |= ((all & 0x80008000u) != 0x80008000u) ? (1u << q) : 0u;
    }
    hitq = __reduce_or_sync(kFull, hitq);
    if (hitq) {
      const int chunk_local = (int)(g - it.chunk_begin);
#pragma unroll
      for (int q = 0; q < QT; q++) {
        if (hitq & (1u << q)) {
          const uint32_t O0 = acc_o[q][0], E0 = acc_a[q][0] - (O0 << 8);
          const uint32_t O1 = acc_o[q][1], E1 = acc_a[q][1] - (O1 << 8);
          candidates(a, s, wbuf + q * a.cap_l, w, q, E0, O0, E1, O1, valid8, chunk_local);
        }
      }
    }
  }
}

// Loop variant of one tile: the linear fixed-m loop where it applies.
template <int D, int MC, int QT, bool LIN>
__device__ __forceinline__ void run_chunks(const ScanArgs &a, Smem &s, const WorkItem &it,
                                           uint32_t *wbuf, int m, uint32_t tab_sa, uint32_t one,
                                           int nq_tile) {
  if constexpr (LIN && MC > 0 && MC % 8 == 0 && D >= 8)
    chunk_loop_lin<D, MC, QT>(a, s, it, wbuf, tab_sa, one, nq_tile);
  else
    chunk_loop<D, MC, QT>(a, s, it, wbuf, m, tab_sa, one, nq_tile);
}

// Occupancy: 4 CTAs per SM for 8-query tiles (128 registers): with the
// 96-register cap of 5 CTAs ptxas sank the code-word prefetch of the hot
// loop next to its use (ncu: the scan's top stall) and spilled; the wider
// budget keeps the loads at the top of the iteration (configs[4] scan
// 38.6 -> 37.8 ms).
template <int MC, int QT, bool LIN>
__global__ void __launch_bounds__(kWarps * 32, QT >= 16 ? 3 : (QT >= 8 ? 4 : 6))
k_scan(const __grid_constant__ ScanArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ Smem s;
  const int m = MC ? MC : a.m;
  uint4 *s_tab = (uint4 *)dsm;                                      // [QT][m]
  uint32_t *s_buf = (uint32_t *)(dsm + (size_t)QT * m * 16);        // [W][QT][cap_l]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t *wbuf = s_buf + (size_t)w * QT * a.cap_l;
  const uint32_t tab_sa = (uint32_t)__cvta_generic_to_shared(s_tab);
  const uint32_t one = (uint32_t)(a.R > 0);  // runtime 1 (keeps IMAD on the FMA pipe)
  const int n_items = *a.n_items;
  if (threadIdx.x == 0) s.item = atomicAdd(a.item_counter, 1);
  for (;;) {
    __syncthreads();
    const int item = s.item;
    if (item >= n_items) break;
    const WorkItem it = a.items[item];
    // ---- stage the tile's byte tables and per-query state ----
    for (int e = threadIdx.x; e < QT * m; e += blockDim.x) {
      const int q = e / m, j = e - q * m;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (q < it.pair_count) {
        const int t = a.pair_t[it.pair_begin + q];
        v = ((const uint4 *)a.qt)[(size_t)t * m + j];
      }
      s_tab[e] = v;
    }
    if (threadIdx.x < QT) {
      const int q = threadIdx.x;
      int thr = -1;
      unsigned mb = 0;
      if (q < it.pair_count) {
        const int pi = it.pair_begin + q;
        const int query = a.pair_q[pi], t = a.pair_t[pi];
        s.query[q] = query;
        s.qmin[q] = a.qmin_f[t];
        s.delta[q] = a.delta_f[t];
        const float hw = a.hist_w[query];
        s.hinv[q] = hw > 0.f ? __frcp_rn(hw) : 0.f;
        mb = *(volatile unsigned *)&a.M_bits[query];
        thr = q_threshold(__uint_as_float(mb), s.qmin[q], s.delta[q]);
      } else {
        s.query[q] = 0;
        s.qmin[q] = 0.f;
        s.delta[q] = 0.f;
        s.hinv[q] = 0.f;
      }
      for (int ww = 0; ww < kWarps; ww++) {
        s.thr[ww][q] = thr;
        s.kbias[ww][q] = kbias_of(thr);
        s.mc[ww][q] = mb;
        s.bn[ww][q] = 0;
        s.pend[ww][q] = 0;
      }
    }
    if (threadIdx.x == 0) {
      s.pair_count = it.pair_count;
      s.chunk_begin = it.chunk_begin;
    }
    __syncthreads();
    // claim the next item now: the atomic's latency hides behind this item
    if (threadIdx.x == 0) s.item = atomicAdd(a.item_counter, 1);
    const int nq_tile = s.pair_count;
    const int depth = it.variant & 255;  // order_items: min pair depth of the tile
    // ---- warp loop over chunks (one specialization per byte-sum depth) ----
    // tiles with at most half the query slots in use (the last tile of an
    // inverted list) run the QT/2 loop instead of computing empty slots
    constexpr int QH = QT / 2 > 0 ? QT / 2 : 1;
    const bool half = QH < QT && ((it.variant >> 8) & 1);
    if (half) {
      switch (depth) {
        case 16: run_chunks<16, MC, QH, LIN>(a, s, it, wbuf, m, tab_sa, one, nq_tile); break;
        case 8: run_chunks<8, MC, QH, LIN>(a, s, it, wbuf, m, tab_sa, one, nq_tile); break;
        case 4: run_chunks<4, MC, QH, LIN>(a, s, it, wbuf, m, tab_sa, one, nq_tile); break;
        default: run_chunks<2, MC, QH, LIN>(a, s, it, wbuf, m, tab_sa, one, nq_tile); break;
      }
    } else {
      switch (depth) {
        case 16: run_chunks<16, MC, QT, LIN>(a, s, it, wbuf, m, tab_sa, one, nq_tile); break;
        case 8: run_chunks<8, MC, QT, LIN>(a, s, it, wbuf, m, tab_sa, one, nq_tile); break;
        case 4: run_chunks<4, MC, QT, LIN>(a, s, it, wbuf, m, tab_sa, one, nq_tile); break;
        default: run_chunks<2, MC, QT, LIN>(a, s, it, wbuf, m, tab_sa, one, nq_tile); break;
      }
    }
    // ---- end of item: CTA-level bound per query (the R-th smallest value
    // over all four warps' buffers lowers the global M), all queries of the
    // tile in one pass: 256 bins as packed 16-bit pairs (<= 4 * cap_l
    // entries per query), then one warp per query scans them ----
    __syncthreads();
    {
      uint32_t *s_h = s_buf + (size_t)kWarps * QT * a.cap_l;  // [QT][128]
      for (int i = threadIdx.x; i < QT * 128; i += blockDim.x) s_h[i] = 0;
      __syncthreads();
      for (int q = 0; q < nq_tile; q++) {
        int tot = 0;
        for (int ww = 0; ww < kWarps; ww++) tot += s.bn[ww][q];
        if (tot < a.R) continue;  // uniform: s.bn is stable after the barrier
        for (int ww = 0; ww < kWarps; ww++) {
          const int n = s.bn[ww][q];
          const uint32_t *b = s_buf + ((size_t)ww * QT + q) * a.cap_l;
          for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const uint32_t v = b[i] >> 24;
            atomicAdd(&s_h[q * 128 + (v >> 1)], 1u << ((v & 1u) * 16));
          }
        }
      }
      __syncthreads();
      for (int q = w; q < nq_tile; q += kWarps) {
        int tot = 0;
        for (int ww = 0; ww < kWarps; ww++) tot += s.bn[ww][q];
        if (tot < a.R) continue;
        const uint4 h4 = *(const uint4 *)&s_h[q * 128 + lane * 4];  // bins 8*lane .. +7
        const uint32_t hw[4] = {h4.x, h4.y, h4.z, h4.w};
        unsigned c = 0;
#pragma unroll
        for (int i = 0; i < 4; i++) c += (hw[i] & 0xffffu) + (hw[i] >> 16);
        unsigned incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += y;
        }
        const unsigned hit = __ballot_sync(kFull, incl >= (unsigned)a.R);
        if (lane == __ffs(hit) - 1) {
          unsigned cum = incl - c;
          int t = lane * 8;
          for (int i = 0; i < 8; i++, t++) {
            cum += (hw[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
            if (cum >= (unsigned)a.R) break;
          }
          atomicMin(&a.M_bits[s.query[q]], fbits(midpoint(s.qmin[q], s.delta[q], t)));
        }
      }
    }
    flush_all(a, s, wbuf, w, nq_tile);
    __syncthreads();
  }
}

template <int MC, int QT, bool LIN>
void launch_t(const ScanArgs &a, int nsm, cudaStream_t st) {
  const int m = MC ? MC : a.m;
  const size_t smem = (size_t)QT * m * 16 + (size_t)kWarps * QT * a.cap_l * 4 + (size_t)QT * 512;
  cudaFuncSetAttribute(k_scan<MC, QT, LIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_scan<MC, QT, LIN>, kWarps * 32, smem);
  per_sm = std::max(per_sm, 1);
  k_scan<MC, QT, LIN><<<nsm * per_sm, kWarps * 32, smem, st>>>(a);
}

template <int MC, int QT, bool LIN>
int resident_t(int m_rt, int cap_l, int nsm) {
  const int m = MC ? MC : m_rt;
  const size_t smem = (size_t)QT * m * 16 + (size_t)kWarps * QT * cap_l * 4 + (size_t)QT * 512;
  cudaFuncSetAttribute(k_scan<MC, QT, LIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_scan<MC, QT, LIN>, kWarps * 32, smem);
  return nsm * std::max(per_sm, 1);
}

// Long items (exhaustive lists) run the linear fixed-m loop for depths
// >= 8; short items (inverted lists) keep the interleaved loop, which
// measured faster there.
template <int MC, int QT>
void launch_t(const ScanArgs &a, int nsm, cudaStream_t st) {
  if (MC > 0 && a.linear) launch_t<MC, QT, true>(a, nsm, st);
  else launch_t<MC, QT, false>(a, nsm, st);
}

// ---- tensor-core scan (int8 tcgen05.mma) ----
//
// The lane sum of a code for a query is a dot product with a one-hot code:
//   sum_j T_q[j][c_j] = onehot(c) . T_q,   onehot(c)[16 j + c_j] = 1,
// exact in int32 (entries <= 127, m <= 32), and min(255, .) of it is the
// reference's saturating byte sum (all entries are >= 0). A tile of 128 codes
// is expanded by its threads into the A operand, written straight to TMEM
// with tcgen05.st (128 lanes x 16m bytes, K-major: no shared-memory traffic
// for the 16x-inflated one-hot operand); the uint8 tables of the item's NQ
// queries are the resident B operand (NQ x 16m, K-major, SMEM); one elected
// thread issues m/2 tcgen05.mma.kind::i8 (K = 32 each, A from TMEM) into a
// TMEM accumulator (128 lanes x NQ int32 columns) and commits to an mbarrier; every thread then reads its
// code's NQ sums with tcgen05.ld and tests them against the queries'
// thresholds. Survivors go straight to the per-query global candidate lists
// (midpoint <= the global bound M), counted in the per-query midpoint
// histogram whose R-th bucket tightens M (hist_bound) — the same selection
// contract as k_scan. B's SMEM layout: canonical K-major, no swizzle: row
// r, 16-byte column j at (r / 8) * 8K + 128 j + 16 (r % 8) (LBO = 128 B,
// SBO = 8K B).
constexpr int kTcCodes = 128;  // codes per tile (MMA M)
constexpr int kTcNQ = 256;     // queries per item (max MMA N)
constexpr int kRing = 1024;    // survivor ring between the compute warps and the flusher warp

__device__ __forceinline__ uint64_t tc_smem_desc(uint32_t saddr, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__device__ __forceinline__ void tc_wait(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tTC_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra TC_DONE;\n\tbra TC_WAIT;\n\tTC_DONE:\n\t}" ::"r"(mbar),
      "r"(phase), "n"(1000000)  // suspend-time hint (ns): the warp sleeps instead of spinning
      : "memory");
}

// One elected lane of the (converged) warp.
__device__ __forceinline__ bool tc_elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
               : "=r"(pred));
  return pred != 0;
}

// As tc_wait without the suspend-time hint (short tiles: the wake-up must be prompt).
__device__ __forceinline__ void tc_wait_spin(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tTCS_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra TCS_DONE;\n\tbra TCS_WAIT;\n\tTCS_DONE:\n\t}" ::"r"(mbar),
      "r"(phase)
      : "memory");
}

// Non-blocking probe of an mbarrier phase (warp-uniform: lane 0 decides).
__device__ __forceinline__ bool tc_try_warp(uint32_t mbar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(mbar), "r"(phase)
      : "memory");
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

// 64 accumulator columns of the thread's TMEM lane, low 16 bits of each,
// two adjacent columns per register (column 2i in the low half of v[i]).
// Sums are < 2^13, so the 16-bit halves are exact. No wait: the caller
// issues tcgen05.wait::ld once for all its loads.
__device__ __forceinline__ void tc_ld64p(uint32_t taddr, uint32_t *v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
      "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

struct TcEntry {
  float mid;
  int query;     // -1: slot free
  int64_t pos;   // code position (chunk * 256 + code)
};

struct TcSmem {
  uint64_t mbar[2];
  uint32_t tmem;
  int item;
  int done;
  unsigned head;  // ring slots reserved (monotone)
  unsigned tail;  // ring slots consumed by the flusher (monotone)
  int query[kTcNQ];
  float qmin[kTcNQ];
  float delta[kTcNQ];
  // per-query threshold t as t + 0x8000 (t in [-1, 254]); read as packed
  // pairs by the epilogue's SWAR test
  __align__(16) uint16_t thr16[kTcNQ];
  unsigned mc[kTcNQ];  // cached global bound M (bits)
  __align__(16) uint32_t xfer[16][4][32];  // per compute warp: up to 4 lanes' packed sums
  int64_t stash_pos[16][4];                 // (k_scan_tc2i: survivors stashed until the warp idles)
  TcEntry ring[kRing];
};
// debug counters (QADC_B200_TC_DEBUG bit 64): slow-path entries, hits, ring
// pushes, direct appends
__device__ unsigned long long g_tc_stats[4];
// one instance per CTA of k_scan_tc (file-scope: direct shared addressing
// from every helper)
__shared__ TcSmem g_tc;

// Global append of one candidate (its slot already claimed).
__device__ __forceinline__ void tc_put(const ScanArgs &a, int query, float mid, int64_t pos,
                                       unsigned slot) {
  if (slot < (unsigned)a.cap_g) {
    const size_t o = (size_t)query * a.cap_g + slot;
    a.cand_mid[o] = mid;
    a.cand_id[o] = a.ids[pos];
  }
  const float hw = a.hist_w[query];
  if (hw > 0.f) {
    unsigned *h = a.hist + (size_t)query * kHistWords;
    const int b = min((int)__fmul_rn(mid, __frcp_rn(hw)), kHistBins - 1);
    atomicAdd(&h[b], 1u);
  }
}

// Survivors of the epilogue, one candidate per lane (want = the lane has
// one): pushed to the shared-memory ring drained by the flusher warp (no
// global round trip on the tile's critical path). Warp-converged: one slot
// claim per warp. Each warp checks the ring's room before reserving and has
// at most one reservation (<= 32 slots) in flight, so 16 x 32 = 512 slots of
// slack make the reservation safe; a full ring falls back to direct appends.
// (slack: slots kept free for reservations in flight — every warp that can
// push may hold one of up to 64 slots between its check and its claim;
// k_scan_tcw passes 640 = 12 compute warps x 32 + 3 filter warps x 64 + a
// margin, which makes its ring overflow-free by construction.)
__device__ __forceinline__ void tc_hit_warp(const ScanArgs &a, bool w0, bool w1, int q,
                                            uint32_t vv, int64_t pos, unsigned slack = 512) {
  const int lane = threadIdx.x & 31;
  float mid0 = 0.f, mid1 = 0.f;
  if (w0) {
    mid0 = midpoint(g_tc.qmin[q], g_tc.delta[q], (int)(vv & 0xffffu));
    w0 = mid0 <= __uint_as_float(g_tc.mc[q]) && !(a.dbg & 32);
  }
  if (w1) {
    mid1 = midpoint(g_tc.qmin[q + 1], g_tc.delta[q + 1], (int)(vv >> 16));
    w1 = mid1 <= __uint_as_float(g_tc.mc[q + 1]) && !(a.dbg & 32);
  }
  const unsigned b0 = __ballot_sync(kFull, w0), b1 = __ballot_sync(kFull, w1);
  if (!(b0 | b1)) return;
  const int leader = __ffs(b0 | b1) - 1;
  unsigned base = 0xffffffffu;
  if (lane == leader) {
    const unsigned h = *(volatile unsigned *)&g_tc.head, t = *(volatile unsigned *)&g_tc.tail;
    if (h - t < (unsigned)kRing - slack)
      base = atomicAdd(&g_tc.head, (unsigned)(__popc(b0) + __popc(b1)));
  }
  base = __shfl_sync(kFull, base, leader);
  if (!(w0 || w1)) return;
  if (a.dbg & 64) atomicAdd(&g_tc_stats[1], (unsigned long long)(w0 + w1));
  if (base != 0xffffffffu) {
    const unsigned lt = (1u << lane) - 1u;
    const unsigned k = base + __popc(b0 & lt) + __popc(b1 & lt);
    TcEntry &e0 = g_tc.ring[k % kRing];
    TcEntry &e1 = g_tc.ring[(k + (w0 ? 1u : 0u)) % kRing];
    if (w0) {
      e0.mid = mid0;
      e0.pos = pos;
    }
    if (w1) {
      e1.mid = mid1;
      e1.pos = pos;
    }
    if (!(a.dbg & 16)) __threadfence_block();
    if (w0) *(volatile int *)&e0.query = g_tc.query[q];
    if (w1) *(volatile int *)&e1.query = g_tc.query[q + 1];
    if (a.dbg & 64) atomicAdd(&g_tc_stats[2], (unsigned long long)(w0 + w1));
    return;
  }
  if (a.dbg & 64) atomicAdd(&g_tc_stats[3], (unsigned long long)(w0 + w1));
  if (w0) tc_put(a, g_tc.query[q], mid0, pos, atomicAdd(&a.cand_n[g_tc.query[q]], 1u));
  if (w1) tc_put(a, g_tc.query[q + 1], mid1, pos, atomicAdd(&a.cand_n[g_tc.query[q + 1]], 1u));
}

// Flusher warp: drains the ring into the global candidate lists (4 entries
// per lane per round, their slot claims in flight together) and tightens the
// global bound M of a query from the histogram every bound_every appends.
__device__ __forceinline__ void tc_flusher(const ScanArgs &a, int done_target = 1) {
  const int lane = threadIdx.x & 31;
  unsigned tail = 0;
  for (;;) {
    const unsigned head = *(volatile unsigned *)&g_tc.head;
    if (head == tail) {
      if (*(volatile int *)&g_tc.done >= done_target && *(volatile unsigned *)&g_tc.head == tail) break;
      __nanosleep(200);
      continue;
    }
    const unsigned n = min(head - tail, 128u);
    TcEntry e[4];
    unsigned slot[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
      e[r].query = -1;
      const unsigned i = (unsigned)(r * 32 + lane);
      if (i < n) {
        volatile TcEntry *ve = &g_tc.ring[(tail + i) % kRing];
        int qy;
        while ((qy = ve->query) < 0) __nanosleep(64);  // writer between its claim and its publish: yield the issue slots
        __threadfence_block();
        e[r].query = qy;
        e[r].mid = ve->mid;
        e[r].pos = ve->pos;
      }
    }
#pragma unroll
    for (int r = 0; r < 4; r++)
      if (e[r].query >= 0) slot[r] = atomicAdd(&a.cand_n[e[r].query], 1u);
    unsigned bound_lanes = 0;
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const bool has = e[r].query >= 0;
      if (has) {
        tc_put(a, e[r].query, e[r].mid, e[r].pos, slot[r]);
        g_tc.ring[(tail + r * 32 + lane) % kRing].query = -1;
      }
      const bool bnd = has && (slot[r] + 1) % (unsigned)a.bound_every == 0;
      bound_lanes |= __ballot_sync(kFull, bnd) ? (1u << r) : 0u;
    }
    __syncwarp();
    __threadfence_block();  // freed slots (query = -1) visible before the new tail
    tail += n;
    if (lane == 0) *(volatile unsigned *)&g_tc.tail = tail;
    // bound refresh for the queries that crossed a multiple of bound_every
#pragma unroll
    for (int r = 0; r < 4; r++) {
      if (!(bound_lanes >> r & 1u)) continue;
      unsigned mq = __ballot_sync(kFull, e[r].query >= 0 && (slot[r] + 1) % (unsigned)a.bound_every == 0);
      while (mq) {
        const int src = __ffs(mq) - 1;
        mq &= mq - 1;
        const int query = __shfl_sync(kFull, e[r].query, src);
        const unsigned mb = hist_bound(a, query);
        if (lane == 0) atomicMin(&a.M_bits[query], mb);
      }
    }
  }
}

// Expand MH sub-quantizers of one code into the A operand in TMEM: the
// thread's own lane (= A row, the code's position in the tile), 16 columns
// per group of four sub-quantizers, from column a_col. The source is the
// code-major copy of the codes (qadc_b200_index::codes_cm): 16 bits = the
// four sub-codes of one group, i.e. a ready PRMT selector. Word e of a group
// is PRMT(pool_e, selector): byte i = 1 iff sub-code i of the group equals e
// (pool_e = the 8-byte constant with byte e & 7 set to 1; entries 8..15 use
// the selector with bit 3 of every nibble flipped, and a nibble >= 8 reads
// the sign of a pool byte = 0). One PRMT per 32-bit TMEM cell, against ~2.4
// shift / add instructions per cell when the one-hot bytes are built from
// the interleaved words. The K order this produces — byte (16 (4 g) + 4 e +
// i) = entry e of sub-quantizer 4 g + i — is matched by the B staging.
// (mode: timing experiments of k_scan_tcw only: 1 = stores without the PRMTs,
// 2 = PRMTs without the stores)
template <int MH>
__device__ __forceinline__ void tc_expand_cm(uint32_t a_col, const uint32_t (&cw)[(MH + 7) / 8],
                                             int mode = 0) {
#pragma unroll
  for (int gi = 0; gi < MH / 4; gi++) {
    // The pool constant sits in PRMT's second source (bytes 4..7), where SASS
    // takes an immediate; as first source ptxas re-materialises it from a
    // uniform register before every PRMT (64 extra moves per code). Entries
    // whose pool byte would be 0..3 flip bit 2 of every selector nibble
    // instead, so four selector variants serve the 16 entries.
    const uint32_t sel = (gi & 1) ? (cw[gi / 2] >> 16) : cw[gi / 2];
    const uint32_t sv[4] = {sel ^ 0x4444u, sel, sel ^ 0xccccu, sel ^ 0x8888u};
    uint32_t r[16];
#pragma unroll
    for (int e = 0; e < 16; e++) r[e] = mode == 1 ? sv[e >> 2] : prmt(0u, 1u << (8 * (e & 3)), sv[e >> 2]);
    if (mode == 2) {
      uint32_t x = 0;
#pragma unroll
      for (int e = 0; e < 16; e++) asm volatile("" ::"r"(r[e]));
      (void)x;
      continue;
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16};" ::"r"(a_col + 16 * gi),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
  }
}

// The code-major words of sub-quantizers [j0, j0 + MH) of code c of chunk g
// (MH = 4: the group's 16 bits moved to the low half).
template <int MC, int MH>
__device__ __forceinline__ void tc_load_cm(const ScanArgs &a, int64_t g, int c, int j0,
                                           uint32_t (&cw)[(MH + 7) / 8]) {
  if (a.dbg & 4) g = 0;  // timing experiment: every tile reads chunk 0 (L1/L2 resident)
  const uint32_t *p = a.codes_cm + ((size_t)g * kChunkCodes + c) * (MC / 8) + j0 / 8;
#pragma unroll
  for (int i = 0; i < (MH + 7) / 8; i++) cw[i] = __ldg(p + i);
  if (MH == 4) cw[0] >>= (j0 & 4) * 4;
}

// 4 x 4 byte transpose: o[ee] byte i = a[i] byte ee.
__device__ __forceinline__ void tc_transpose4(const uint32_t (&a)[4], uint32_t (&o)[4]) {
  const uint32_t t0 = prmt(a[0], a[1], 0x5140u), t1 = prmt(a[0], a[1], 0x7362u);
  const uint32_t u0 = prmt(a[2], a[3], 0x5140u), u1 = prmt(a[2], a[3], 0x7362u);
  o[0] = prmt(t0, u0, 0x5410u);
  o[1] = prmt(t0, u0, 0x7632u);
  o[2] = prmt(t1, u1, 0x5410u);
  o[3] = prmt(t1, u1, 0x7632u);
}

// nr packed registers (2 accumulator columns each, 16-bit halves) of the
// thread's TMEM lane from column taddr: only the item's query columns are
// read (TMEM reads cost ~64 B / cycle per SM: with the few queries of an
// inverted list, reading all 64 columns of a part was the tile's longest
// step). Registers past nr are zero.
__device__ __forceinline__ void tc_ldp(uint32_t taddr, int nr, uint32_t *v) {
  if (nr > 16) {
    tc_ld64p(taddr, v);
  } else if (nr > 8) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
        "%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 16; i < 32; i++) v[i] = 0;
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7])
        : "r"(taddr));
#pragma unroll
    for (int i = 8; i < 32; i++) v[i] = 0;
  }
}

// (k_scan_tc2 / k_scan_tc2i: interleaved source)
// Word w of sub-code x is 1 << (8 x - 32 w) when 0 <= 8 x - 32 w < 32, else
// 0: PTX shl clamps shift amounts >= 32 to a zero result.
__device__ __forceinline__ uint32_t tc_shl(uint32_t s) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(1u), "r"(s));
  return r;
}

template <int MC, int MH>
__device__ __forceinline__ void tc_load(const ScanArgs &a, int64_t g, int c, int j0,
                                        uint32_t (&cw)[MH]) {
  if (a.dbg & 4) g = 0;  // timing experiment: every tile reads chunk 0 (L1/L2 resident)
  const uint32_t *p = a.codes + ((size_t)g * MC + j0) * 32 + (c >> 3);
#pragma unroll
  for (int j = 0; j < MH; j++) cw[j] = __ldg(p + j * 32);
}

// Named barriers over the compute warps and the MMA warp (NB threads).
template <int NB>
__device__ __forceinline__ void tc_bar_all() { asm volatile("bar.sync 1, %0;" ::"n"(NB) : "memory"); }
template <int NB>
__device__ __forceinline__ void tc_arrive(int t) {
  if (t & 1) asm volatile("bar.arrive 3, %0;" ::"n"(NB) : "memory");
  else asm volatile("bar.arrive 2, %0;" ::"n"(NB) : "memory");
}
template <int NB>
__device__ __forceinline__ void tc_sync(int t) {
  if (t & 1) asm volatile("bar.sync 3, %0;" ::"n"(NB) : "memory");
  else asm volatile("bar.sync 2, %0;" ::"n"(NB) : "memory");
}

// 4G + 2 warps, specialised (G = 4 by default):
//  * warps 0 .. 4G-1 (compute): warps w, w + 4, ... share TMEM lane quarter
//    w % 4 (codes 32 (w % 4) .. + 31 of the tile); warp part p = w / 4
//    expands sub-quantizers [p m/G, (p + 1) m/G) and reads query columns
//    32 k with k % G == p. Per tile: expand tile t + 1 into A[(t + 1) & 1]
//    while MMA(t) runs, wait for MMA(t), read its sums, then arrive on tile
//    t + 1's named barrier (2 / 3 alternating). They never wait for each
//    other inside an item;
//  * warps 4G + 1 .. 4G + kMmaWarps (MMA): per tile, bar.sync on the tile's
//    named barrier (all compute threads expanded it, finished reading D and
//    zeroed it), then one elected lane per warp issues its share of the m/2
//    MMAs (k-steps mw, mw + kMmaWarps, ...; N = the item's queries, up to
//    256) and commits to the mbarrier (one arrival per MMA warp). As compiled
//    here an issuing warp spends ~70 cycles per MMA (its operands are moved
//    from vector to uniform registers for every instruction), which matters
//    only below N = 128 (the tensor pipe needs N / 2 cycles): four issuing
//    warps hide it. (k_scan_tcw, the kernel for lists with few queries,
//    issues from ONE warp with loop-invariant uniform operands at the pipe's
//    own rate: tools/tc_kind_bench.) The MMAs of a tile come from several
//    warps in no fixed order, so all of them ACCUMULATE into a D the compute
//    threads zeroed after reading the previous tile (int32 sums:
//    order-independent).
//  D is single-buffered at N = 256: one MMA instruction costs ~77 cycles of
//  issue for any N <= 128 but 128 cycles of execution at N = 256
//  (tools/tc_mma_bench: 3.79 vs 4.59 POP/s back to back), so 256 queries per
//  instruction beat double-buffering two 128-query accumulators;
//  * warp 4G (flusher): drains the survivor ring (tc_flusher).
constexpr int kMmaWarps = 4;
template <int MC, int G>
__global__ void __launch_bounds__(128 * G + 32 + 32 * kMmaWarps, 1)
k_scan_tc(const __grid_constant__ ScanArgs a) {
  constexpr int K = 16 * MC, SBO = 8 * K, MH = MC / G;
  constexpr int NT = 128 * G, NB = NT + 32 * kMmaWarps;  // compute threads; + the MMA warps
  constexpr int kCPT = kTcNQ / G;             // accumulator columns per compute thread
  static_assert(kCPT % 64 == 0, "64-column packed TMEM loads");
  static_assert(MH % 4 == 0 && kTcNQ % (32 * G) == 0 && 4 * G <= 16, "tile split");
  // TMEM columns: D (kTcNQ, single-buffered), then A[0], A[1] (K / 4 each)
  constexpr uint32_t kCols = 512, kACols = K / 4, kA0 = kTcNQ;
  static_assert(kA0 + 2 * kACols <= kCols, "TMEM budget");
  extern __shared__ __align__(16) unsigned char dsm[];  // no-swizzle operands: 16 B alignment
  TcSmem &s = g_tc;
  uint8_t *sB = dsm;                       // [kTcNQ][K]
  const int tid = threadIdx.x, w = tid >> 5;
  const int row = tid & 127, part = tid >> 7, j0 = part * MH, col0 = part * kCPT;
  const uint32_t sB_a = (uint32_t)__cvta_generic_to_shared(sB);
  const uint32_t mbar0 = (uint32_t)__cvta_generic_to_shared(&s.mbar[0]);
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s.tmem)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar0), "n"(kMmaWarps));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar0 + 8));
    asm volatile("fence.mbarrier_init.release.cluster;");
    s.item = atomicAdd(a.item_counter, 1);
    s.done = 0;
    s.head = 0;
    s.tail = 0;
  }
  for (int i = tid; i < kRing; i += blockDim.x) s.ring[i].query = -1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w == 4 * G) {
    tc_flusher(a);
  } else {
  const bool mma_warp = w > 4 * G;
  const int mw = w - (4 * G + 1);  // MMA warp index
  const uint32_t tmem = s.tmem;
  const uint32_t t_row = tmem + ((uint32_t)((w & 3) * 32) << 16);
  const int n_items = *a.n_items;
  uint32_t ph0 = 0;
  if (!mma_warp) {
    // zero this thread's accumulator columns: every MMA accumulates, and a
    // thread zeroes the columns it read again before the next tile's MMAs
    // are released; columns an item's MMAs do not write (>= its N) stay 0,
    // which the SWAR test compares against t = -1
    const uint32_t z[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < kCPT; c += 16)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
          "%13,%14,%15,%16};" ::"r"(t_row + col0 + c),
          "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]),
          "r"(z[8]), "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]),
          "r"(z[15])
          : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  for (;;) {
    const int item = s.item;
    if (item >= n_items) break;
    const WorkItem it = a.items[item];
    const int nq = it.pair_count;
    const int64_t c0g = it.chunk_begin;
    const int64_t ntiles = 2 * (it.chunk_end - it.chunk_begin);
    const int n_mma = max(16, (nq + 15) & ~15);  // MMA N: the item's queries, rounded to 16
    if (!mma_warp) {
      // ---- stage the item's tables (B operand) and per-query state ----
      // K order of tc_expand: per group of four sub-quantizers, entry-major
      // (a 4 x 4 byte transpose of the group's tables); only the rows the
      // MMAs read (< n_mma) are written
      for (int e = tid; e < n_mma * (MC / 4); e += NT) {
        const int q = e / (MC / 4), g4 = e - q * (MC / 4);
        uint4 in[4];
#pragma unroll
        for (int i = 0; i < 4; i++) in[i] = make_uint4(0, 0, 0, 0);
        if (q < nq) {
          const uint4 *src = (const uint4 *)a.qt + (size_t)a.pair_t[it.pair_begin + q] * MC + 4 * g4;
#pragma unroll
          for (int i = 0; i < 4; i++) in[i] = src[i];
        }
        const uint32_t ax[4] = {in[0].x, in[1].x, in[2].x, in[3].x};
        const uint32_t ay[4] = {in[0].y, in[1].y, in[2].y, in[3].y};
        const uint32_t az[4] = {in[0].z, in[1].z, in[2].z, in[3].z};
        const uint32_t aw[4] = {in[0].w, in[1].w, in[2].w, in[3].w};
        uint32_t o[4];
        uint8_t *dst = sB + (q >> 3) * SBO + (4 * g4) * 128 + (q & 7) * 16;
        tc_transpose4(ax, o);
        *(uint4 *)(dst) = make_uint4(o[0], o[1], o[2], o[3]);
        tc_transpose4(ay, o);
        *(uint4 *)(dst + 128) = make_uint4(o[0], o[1], o[2], o[3]);
        tc_transpose4(az, o);
        *(uint4 *)(dst + 256) = make_uint4(o[0], o[1], o[2], o[3]);
        tc_transpose4(aw, o);
        *(uint4 *)(dst + 384) = make_uint4(o[0], o[1], o[2], o[3]);
      }
      if (tid < kTcNQ) {
        const int q = tid;
        int thr = -1;
        unsigned mb = 0;
        if (q < nq) {
          const int pi = it.pair_begin + q;
          const int query = a.pair_q[pi], t = a.pair_t[pi];
          s.query[q] = query;
          s.qmin[q] = a.qmin_f[t];
          s.delta[q] = a.delta_f[t];
          mb = *(volatile unsigned *)&a.M_bits[query];
          thr = q_threshold(__uint_as_float(mb), s.qmin[q], s.delta[q]);
        } else {
          s.query[q] = 0;
          s.qmin[q] = 0.f;
          s.delta[q] = 0.f;
        }
        s.thr16[q] = (uint16_t)(thr + 0x8000);
        s.mc[q] = mb;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    tc_bar_all<NB>();  // B and the query state are staged
    if (tid == 0) s.item = atomicAdd(a.item_counter, 1);  // claimed ahead (read after the item's end barrier)
    if (mma_warp) {
      const uint32_t idesc =
          (2u << 4) | ((uint32_t)(n_mma >> 3) << 17) | ((uint32_t)(kTcCodes >> 4) << 24);
      for (int64_t t = 0; t < ntiles; t++) {
        tc_sync<NB>((int)t);
        const int buf = (int)(t & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if ((tid & 31) == 0) {
#pragma unroll
          for (int ks = 0; ks < K / 32; ks++) {
            if (ks % kMmaWarps != mw) continue;
            const uint32_t ta = tmem + kA0 + buf * kACols + ks * 8;  // A from TMEM (K = 32 bytes = 8 columns)
            const uint64_t db = tc_smem_desc(sB_a + ks * 256, SBO);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                "r"(ta), "l"(db), "r"(idesc), "r"(1u));
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                  mbar0)
              : "memory");
        }
        __syncwarp();
      }
    } else {
      uint32_t cw[(MH + 7) / 8];
      // this thread's A columns (its lane quarter, its part of the K range)
      const uint32_t a_lane = tmem + ((uint32_t)((w & 3) * 32) << 16) + kA0 + (uint32_t)(j0 * 4);
      // prologue: expand tile 0 into A[0], load tile 1's words
      tc_load_cm<MC, MH>(a, c0g, row, j0, cw);
      tc_expand_cm<MH>(a_lane, cw);
      if (ntiles > 1) tc_load_cm<MC, MH>(a, c0g, kTcCodes + row, j0, cw);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      tc_arrive<NB>(0);
      for (int64_t t = 0; t < ntiles; t++) {
        unsigned mpre = 0;
        if (tid < nq) mpre = *(volatile unsigned *)&a.M_bits[s.query[tid]];  // lands during the wait
        // valid byte of this thread's code in tile t (lands during the wait;
        // read only by the survivor path)
        const int c_t = (int)(t & 1) * kTcCodes + row;
        const int64_t g_t = c0g + (t >> 1);
        const uint32_t vb_t = __ldg(a.valid + g_t * 32 + (c_t >> 3));
        // ---- expand tile t + 1 into A[(t + 1) & 1] while MMA(t) runs
        // (MMA(t - 1), its last reader, completed before this warp read
        // tile t - 1) ----
        if (t + 1 < ntiles) {
          if (!(a.dbg & 2)) tc_expand_cm<MH>(a_lane + (uint32_t)((t + 1) & 1) * kACols, cw);
          if (t + 2 < ntiles)
            tc_load_cm<MC, MH>(a, c0g + ((t + 2) >> 1), (int)((t + 2) & 1) * kTcCodes + row, j0, cw);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        // ---- tile t: copy this thread's sums out of TMEM and release D
        // (MMA(t + 1) waits for every compute thread's arrive), then test
        // them from registers while MMA(t + 1) runs ----
        tc_wait(mbar0, ph0);
        ph0 ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;");
        // (columns >= the MMA's N hold earlier items' sums: see the zeroing
        // above)
        // (warps whose query columns lie past the item's N have nothing to
        // read: with few queries per list only part 0 runs the epilogue)
        const bool has_cols = col0 < n_mma;
        uint32_t v[kCPT / 2];
        if (has_cols) {
#pragma unroll
          for (int l = 0; l < kCPT / 64; l++)
            tc_ldp(t_row + col0 + 64 * l, min(64, max(0, n_mma - col0 - 64 * l)) / 2, v + 32 * l);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          // zero the columns just read (the next tile's MMAs accumulate)
          const uint32_t z = 0;
#pragma unroll
          for (int c = 0; c < kCPT; c += 16)
            if (col0 + c < n_mma)
              asm volatile(
                  "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
                  "%1,%1,%1,%1};" ::"r"(t_row + col0 + c), "r"(z)
                  : "memory");
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        if (t + 1 < ntiles) tc_arrive<NB>((int)(t + 1));  // A(t + 1) written, D read and zeroed
        // SWAR survivor test on packed pairs: (t + 0x8000) - s keeps bit
        // 15 of its half iff s <= t (halves never borrow: s < 2^13 and
        // t + 0x8000 in [0x7fff, 0x80fe])
        const uint4 *T = (const uint4 *)&s.thr16[col0];
        uint32_t any = 0;
        if (has_cols) {
#pragma unroll
          for (int i = 0; i < kCPT / 2 && !(a.dbg & 8); i += 4) {
            if (2 * i >= n_mma - col0) break;
            const uint4 tt = T[i / 4];
            any |= (tt.x - v[i]) | (tt.y - v[i + 1]) | (tt.z - v[i + 2]) | (tt.w - v[i + 3]);
          }
        }
        // survivors (rare once the bounds converge): the warp handles its
        // lanes with survivors one at a time, each of the lane's packed
        // sum registers passed through shared memory to a lane of its own
        unsigned todo = has_cols ? __ballot_sync(kFull, (any & 0x80008000u) &&
                                                            ((vb_t >> (c_t & 7)) & 1u) && !(a.dbg & 1))
                                 : 0u;
        if (todo) {
          const int lane = tid & 31;
          uint32_t *xf = s.xfer[w][0];
          const int64_t pos0 = g_t * kChunkCodes + (int64_t)(c_t - lane);
          while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            if (a.dbg & 64 && lane == src) atomicAdd(&g_tc_stats[0], 1ull);
#pragma unroll
            for (int r = 0; r < kCPT / 64; r++) {
              if (lane == src) {
#pragma unroll
                for (int i = 0; i < 32; i += 4)
                  *(uint4 *)&xf[i] = make_uint4(v[32 * r + i], v[32 * r + i + 1], v[32 * r + i + 2],
                                                v[32 * r + i + 3]);
              }
              __syncwarp();
              const uint32_t vv = xf[lane];
              const int q = col0 + 64 * r + 2 * lane;
              const uint32_t x = *(const uint32_t *)&s.thr16[q] - vv;
              __syncwarp();
              tc_hit_warp(a, (x & 0x8000u) != 0, (x & 0x80000000u) != 0, q, vv, pos0 + src);
            }
          }
        }
        if (tid < nq && mpre < s.mc[tid]) {  // bounds tightened by the flusher or other CTAs
          s.mc[tid] = mpre;
          const int th = q_threshold(__uint_as_float(mpre), s.qmin[tid], s.delta[tid]);
          if (th + 0x8000 < (int)s.thr16[tid]) s.thr16[tid] = (uint16_t)(th + 0x8000);
        }
      }
    }
    tc_bar_all<NB>();  // end of item: every tile read, s.item holds the next item
  }
  if (tid == 0) *(volatile int *)&s.done = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s.tmem), "n"(kCols));
}


// ---- tensor-core scan for inverted lists with few queries (k_scan_tcw) ----
//
// IVF batches put 10-40 (query, list) pairs on a list (configs[4]: 93 % of
// the scanned codes sit in lists probed by <= 32 queries of the batch), so
// the MMA itself is short (N = 16 or 32: 8-16 cycles per K = 32 step) and a
// tile's cost is the one-hot expansion of its codes on the ALU pipe plus the
// latency of the expand -> MMA -> read chain. k_scan_tc runs ONE tile at a
// time on all its warps, so every thread repeats the tile's fixed work
// (addresses, barriers, bound refresh) for a quarter of a code; here a CTA
// holds kWG independent warpgroups, each scanning its own work item (list,
// <= 32 queries, chunk range) tile by tile:
//   * thread = one code of the 128-code tile: ONE 16-byte load of its
//     code-major row (coalesced 512 B per warp, requested two tiles ahead),
//     m / 4 x 16 PRMT one-hot words written to its TMEM lane (tc_expand_cm);
//   * the tile is expanded and multiplied in two halves of m / 2
//     sub-quantizers: warp 0 of the warpgroup waits on the half's named
//     barrier (the others only arrive and go on), issues its m / 4 MMAs from
//     loop-invariant uniform operands (the first MMA of a tile overwrites D,
//     the rest accumulate) and commits to the half's mbarrier. The MMAs of
//     half 0 run while half 1 is expanded, those of half 1 while half 0 of
//     the NEXT tile is expanded, so no thread waits for an MMA just issued;
//   * every thread reads its code's N sums (16-bit packed) and runs the SWAR
//     threshold test after the next tile's first half has been issued;
//     a code with survivors is handed (its packed sums) through the warp's
//     own ring to the warpgroup's filter warp, which runs the per-pair test,
//     midpoints and the push to the candidate ring (tc_hit_warp) drained by
//     the flusher warp (tc_flusher, as k_scan_tc).
// While one warpgroup waits (barrier, MMA) the others expand: the ALU pipe
// (PRMT), the tensor pipe and the survivor path overlap without any
// cross-warpgroup barrier. TMEM per warpgroup: D (32 columns) + A (4 m
// columns), single-buffered.
constexpr int kWG = 3;        // warpgroups per CTA (3 x (32 + 128) <= 512 TMEM columns)
constexpr int kTcwNQ = 32;    // queries per item (MMA N = 16 or 32)
constexpr int kTcwSlots = 8;  // survivor slots per compute warp
// timing experiments (QADC_B200_TC_DEBUG bits 1 / 2 / 128: no survivors / no
// expansion / no MMAs) are compiled in only with -DQADC_TCW_DEBUG=1
#ifndef QADC_TCW_DEBUG
#define QADC_TCW_DEBUG 0
#endif
constexpr bool kTcwDbg = QADC_TCW_DEBUG != 0;
// A code with at least one surviving (query, code) pair: its packed sums go
// through the compute warp's own single-producer ring to the filter warp,
// which runs the per-pair test, midpoints and the push to the candidate ring
// (tc_hit_warp). A compute warp spends ~25 instructions on a survivor
// instead of the per-pair path (configs[4]: ~10^7 survivors per batch cost
// 5.5 of 21.9 ms while compute warps handled them inline).
struct __align__(16) TcwEnt {
  uint32_t sums[kTcwNQ / 2];  // packed pairs: query 2 i (low half), 2 i + 1 (high)
  int64_t pos;                // code position (chunk * 256 + code)
};
struct TcwSmem {
  uint64_t mbar[kWG][2];         // MMAs of half 0 / half 1 of the warpgroup's tile
  int item[kWG];
  int nm2[kWG];                  // packed sum registers of the warpgroup's current item (N / 2)
  unsigned head[4 * kWG];        // slots published by compute warp w (monotone)
  unsigned tail[4 * kWG];        // slots consumed by the filter warp
  __align__(16) TcwEnt ent[4 * kWG][kTcwSlots];
};
__shared__ TcwSmem g_tcw;

// Filter warp f of k_scan_tcw serves the four compute warps of warpgroup f:
// two ring entries per round (lanes 0-15 / 16-31 take one packed pair each),
// the entries' tails released once per round.
__device__ __forceinline__ void tcw_filter(const ScanArgs &a, int f) {
  const int lane = threadIdx.x & 31;
  const int qb = f * kTcwNQ;
  unsigned tail = 0;  // lane l < 4: of ring 4 f + l
  for (;;) {
    unsigned head = 0;
    if (lane < 4) head = *(volatile unsigned *)&g_tcw.head[4 * f + lane];
    const unsigned busy = __ballot_sync(kFull, head != tail);
    if (!busy) {
      // a compute warp publishes its entries before it reports done: re-check once
      if (*(volatile int *)&g_tc.done >= kWG) {
        if (lane < 4) head = *(volatile unsigned *)&g_tcw.head[4 * f + lane];
        if (!__ballot_sync(kFull, head != tail)) break;
        continue;
      }
      __nanosleep(100);
      continue;
    }
    __threadfence_block();  // entries written before the heads read above
    const int rl = __ffs(busy) - 1, r = 4 * f + rl;
    const unsigned h = __shfl_sync(kFull, head, rl), t0 = __shfl_sync(kFull, tail, rl);
    const unsigned n = min(h - t0, 2u);
    const int nm2 = *(volatile int *)&g_tcw.nm2[f];
    const int half = lane >> 4, pl = lane & 15;
    const TcwEnt &e = g_tcw.ent[r][(t0 + (unsigned)half) % kTcwSlots];
    const bool on = (unsigned)half < n && pl < nm2;
    const uint32_t vv = on ? e.sums[pl] : 0u;
    const int64_t pos = e.pos;
    const int q = qb + 2 * pl;
    const uint32_t x = *(const uint32_t *)&g_tc.thr16[q] - vv;
    tc_hit_warp(a, on && (x & 0x8000u) != 0, on && (x & 0x80000000u) != 0, q, vv, pos, 640u);
    if (lane == rl) {
      tail = t0 + n;
      __threadfence_block();  // the entries were read before their slots are released
      *(volatile unsigned *)&g_tcw.tail[r] = tail;
    }
    __syncwarp();
  }
}

template <int MC>
__global__ void __launch_bounds__(128 * kWG + 32 + 32 * kWG, 1) k_scan_tcw(const __grid_constant__ ScanArgs a) {
  constexpr int K = 16 * MC, SBO = 8 * K, WPC = MC / 8;
  constexpr uint32_t kCols = 512, kWgCols = kTcwNQ + K / 4;
  static_assert(kWG * kWgCols <= kCols, "TMEM budget");
  extern __shared__ __align__(16) unsigned char dsm[];  // B: [kWG][kTcwNQ rows][K]
  TcSmem &s = g_tc;
  const int tid = threadIdx.x, lane = tid & 31;
  const int w = __shfl_sync(kFull, tid >> 5, 0);  // warp-uniform for the compiler
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s.tmem)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int g = 0; g < 2 * kWG; g++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&g_tcw.mbar[g >> 1][g & 1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    s.done = 0;
    s.head = 0;
    s.tail = 0;
  }
  if (tid < 4 * kWG) {
    g_tcw.head[tid] = 0;
    g_tcw.tail[tid] = 0;
  }
  for (int i = tid; i < kRing; i += blockDim.x) s.ring[i].query = -1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w == 4 * kWG) {
    tc_flusher(a, 2 * kWG);
  } else if (w > 4 * kWG) {
    tcw_filter(a, w - (4 * kWG + 1));
    if (lane == 0) atomicAdd(&s.done, 1);  // this filter's survivors are in the candidate ring
  } else {
    const int wg = w >> 2, wt = tid & 127, wq = w & 3;  // warpgroup, thread in it, warp in it
    const int qb = wg * kTcwNQ;                          // the warpgroup's slice of the query-state arrays
    uint8_t *sB = dsm + (size_t)wg * kTcwNQ * K;
    const uint32_t sB_a = (uint32_t)__cvta_generic_to_shared(sB);
    const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&g_tcw.mbar[wg][0]);
    const uint32_t tmem = s.tmem;
    const uint32_t t_d = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)wg * kWgCols;  // this thread's D row
    const uint32_t t_a = t_d + kTcwNQ;                                                  // its A row
    const uint32_t d_mma = tmem + (uint32_t)wg * kWgCols, a_mma = d_mma + kTcwNQ;
    const int n_items = *a.n_items;
    uint32_t ph = 0;
    unsigned rh = 0;  // this warp's survivor ring: slots published
    auto wg_sync = [&]() { asm volatile("bar.sync %0, 128;" ::"r"(3 * wg + 1) : "memory"); };
    if (wt == 0) g_tcw.item[wg] = atomicAdd(a.item_counter, 1);
    wg_sync();
    for (;;) {
      const int item = g_tcw.item[wg];
      if (item >= n_items) break;
      const WorkItem it = a.items[item];
      const int nq = it.pair_count;
      const int64_t c0g = it.chunk_begin;
      const int64_t ntiles = 2 * (it.chunk_end - it.chunk_begin);
      const int n_mma = nq > 16 ? 32 : 16;
      // ---- stage the item's tables (B operand, tc_expand_cm's K order) and query state ----
      for (int e = wt; e < n_mma * (MC / 4); e += 128) {
        const int q = e / (MC / 4), g4 = e - q * (MC / 4);
        uint4 in[4];
#pragma unroll
        for (int i = 0; i < 4; i++) in[i] = make_uint4(0, 0, 0, 0);
        if (q < nq) {
          const uint4 *src = (const uint4 *)a.qt + (size_t)a.pair_t[it.pair_begin + q] * MC + 4 * g4;
#pragma unroll
          for (int i = 0; i < 4; i++) in[i] = src[i];
        }
        const uint32_t ax[4] = {in[0].x, in[1].x, in[2].x, in[3].x};
        const uint32_t ay[4] = {in[0].y, in[1].y, in[2].y, in[3].y};
        const uint32_t az[4] = {in[0].z, in[1].z, in[2].z, in[3].z};
        const uint32_t aw[4] = {in[0].w, in[1].w, in[2].w, in[3].w};
        uint32_t o[4];
        uint8_t *dst = sB + (q >> 3) * SBO + (4 * g4) * 128 + (q & 7) * 16;
        tc_transpose4(ax, o);
        *(uint4 *)(dst) = make_uint4(o[0], o[1], o[2], o[3]);
        tc_transpose4(ay, o);
        *(uint4 *)(dst + 128) = make_uint4(o[0], o[1], o[2], o[3]);
        tc_transpose4(az, o);
        *(uint4 *)(dst + 256) = make_uint4(o[0], o[1], o[2], o[3]);
        tc_transpose4(aw, o);
        *(uint4 *)(dst + 384) = make_uint4(o[0], o[1], o[2], o[3]);
      }
      if (wt < kTcwNQ) {
        const int q = wt;
        int thr = -1;
        unsigned mb = 0;
        if (q < nq) {
          const int pi = it.pair_begin + q;
          const int query = a.pair_q[pi], t = a.pair_t[pi];
          s.query[qb + q] = query;
          s.qmin[qb + q] = a.qmin_f[t];
          s.delta[qb + q] = a.delta_f[t];
          mb = *(volatile unsigned *)&a.M_bits[query];
          thr = q_threshold(__uint_as_float(mb), s.qmin[qb + q], s.delta[qb + q]);
        } else {
          s.query[qb + q] = 0;
          s.qmin[qb + q] = 0.f;
          s.delta[qb + q] = 0.f;
        }
        s.thr16[qb + q] = (uint16_t)(thr + 0x8000);
        s.mc[qb + q] = mb;
        if (q == 0) g_tcw.nm2[wg] = n_mma / 2;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      wg_sync();  // B and the query state are staged; everyone has read g_tcw.item
      if (wt == 0) g_tcw.item[wg] = atomicAdd(a.item_counter, 1);  // claimed ahead (read after the item's last barrier)
      const uint32_t idesc =
          (2u << 4) | ((uint32_t)(n_mma >> 3) << 17) | ((uint32_t)(kTcCodes >> 4) << 24);
      // operands of k-step i = the step-0 operands plus compile-time offsets
      // (A from TMEM: 8 columns per step; B: 256 bytes per step): no
      // per-MMA register-to-uniform moves, so ONE warp issues at the tensor
      // pipe's own rate (N / 2 cycles per MMA, tools/tc_kind_bench)
      const uint64_t db_0 = tc_smem_desc(sB_a, SBO);
      const uint32_t *pc = a.codes_cm + ((size_t)c0g * kChunkCodes + wt) * WPC;  // this thread's row of tile 0
      const uint8_t *pv = a.valid + c0g * 32 + (wt >> 3);
      const int64_t pos_w = c0g * kChunkCodes + (wt - lane);  // position of the warp's first code in tile 0
      uint32_t vb_next = __ldg(pv);  // valid byte of this thread's code, one tile ahead
      // code-major rows of tiles t, t + 1 and t + 2 (the row of tile t + 2 is
      // requested a whole tile before its first use)
      uint32_t cw[WPC], cn[WPC], cf[WPC];
      auto load_row = [&](const uint32_t *p, uint32_t (&dst)[WPC]) {
        if (WPC == 4) {
          const uint4 v4 = __ldg((const uint4 *)p);
          dst[0] = v4.x; dst[1] = v4.y; dst[WPC - 2] = v4.z; dst[WPC - 1] = v4.w;
        } else {
          const uint2 v2 = __ldg((const uint2 *)p);
          dst[0] = v2.x; dst[WPC - 1] = v2.y;
        }
      };
      load_row(pc, cw);
      if (ntiles > 1) load_row(pc + kTcCodes * WPC, cn);
      // Half h of a tile = sub-quantizers [h m / 2, (h + 1) m / 2): its own A
      // columns and its own MMAs (k-steps [h m / 4, (h + 1) m / 4), this warp:
      // wq, wq + 4, ... of them), committed to mbarrier h.
      constexpr int HW = WPC / 2, HCOLS = 2 * MC, HK = K / 64;  // words, A columns, MMAs (K = 32 steps) of a half
      auto expand_half = [&](int h, const uint32_t (&row)[WPC]) {
        if (kTcwDbg && (a.dbg & 2)) return;
        uint32_t hw[HW];
#pragma unroll
        for (int i = 0; i < HW; i++) hw[i] = row[h * HW + i];
        tc_expand_cm<MC / 2>(t_a + (uint32_t)(h * HCOLS), hw,
                             kTcwDbg ? ((a.dbg >> 9) & 3) : 0);
      };
      auto issue_half = [&](int h) {
        // this thread's A row half is written (and, for half 0, its D row read)
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        if (wq != 0) {  // only the issuing warp waits for the warpgroup
          asm volatile("bar.arrive %0, 128;" ::"r"(3 * wg + 2 + h) : "memory");
          return;
        }
        asm volatile("bar.sync %0, 128;" ::"r"(3 * wg + 2 + h) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (kTcwDbg && (a.dbg & 128)) return;
        if (tc_elect_one()) {
#pragma unroll
          for (int i = 0; i < HK; i++) {
            // the tile's first MMA overwrites D, the others accumulate
            if (h == 0 && i == 0)
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_mma),
                  "r"(a_mma), "l"(db_0), "r"(idesc), "r"(0u));
            else
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_mma),
                  "r"(a_mma + 8u * (uint32_t)(h * HK + i)), "l"(db_0 + 16ull * (uint64_t)(h * HK + i)),
                  "r"(idesc), "r"(1u));
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                  mbar + 8u * (uint32_t)h)
              : "memory");
        }
        __syncwarp();
      };
      // Software pipeline of one warpgroup (A and D single-buffered, A in two
      // halves): the MMAs of half 0 run while half 1 is expanded, those of
      // half 1 while half 0 of the NEXT tile is expanded, and the threshold
      // test of tile t runs after half 0 of tile t + 1 has been issued: the
      // warpgroup never waits for an MMA it has just issued.
      expand_half(0, cw);
      issue_half(0);
      auto run = [&](auto nm_c) {
        constexpr int NM = decltype(nm_c)::value;  // MMA N: 16 or 32 query columns
        for (int t = 0; t < (int)ntiles; t++) {
          const bool more = t + 1 < (int)ntiles;
          unsigned mpre = 0;
          if (wt < nq) mpre = *(volatile unsigned *)&a.M_bits[s.query[qb + wt]];  // lands during the tile
          const uint32_t vb_t = vb_next;  // read only by the survivor path
          pv += kTcCodes / 8;
          if (more) vb_next = __ldg(pv);
          // ---- half 1 of tile t ----
          expand_half(1, cw);
          pc += kTcCodes * WPC;  // row of tile t + 1
          if (t + 2 < (int)ntiles) {
            load_row(pc + kTcCodes * WPC, cf);
            if (lane == 0 && t + 5 < (int)ntiles)  // the warp's 32 rows of tile t + 5 into L2
              prefetch_l2(pc + 4 * kTcCodes * WPC, 128u * WPC);
          }
          issue_half(1);
          // ---- half 0 of tile t + 1 (its A columns are free once the MMAs of half 0 of tile t are done) ----
          if (!(kTcwDbg && (a.dbg & 128))) tc_wait_spin(mbar, ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (more) expand_half(0, cn);
          // ---- tile t: read this code's sums, zero them ----
          if (!(kTcwDbg && (a.dbg & 128))) tc_wait_spin(mbar + 8, ph);
          ph ^= 1;
          asm volatile("tcgen05.fence::after_thread_sync;");
          uint32_t v[NM / 2];
          if (NM == 32) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
                "%12,%13,%14,%15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                  "=r"(v[7]), "=r"(v[NM / 2 - 8]), "=r"(v[NM / 2 - 7]), "=r"(v[NM / 2 - 6]),
                  "=r"(v[NM / 2 - 5]), "=r"(v[NM / 2 - 4]), "=r"(v[NM / 2 - 3]), "=r"(v[NM / 2 - 2]),
                  "=r"(v[NM / 2 - 1])
                : "r"(t_d));
          } else {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                  "=r"(v[7])
                : "r"(t_d));
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (more) issue_half(0);  // tile t + 1 starts on the tensor pipe before tile t is tested
          // ---- tile t: threshold test ----
          const uint4 *T = (const uint4 *)&s.thr16[qb];
          uint32_t any = 0;
#pragma unroll
          for (int i = 0; i < NM / 2; i += 4) {
            const uint4 tt = T[i / 4];
            any |= (tt.x - v[i]) | (tt.y - v[i + 1]) | (tt.z - v[i + 2]) | (tt.w - v[i + 3]);
          }
          const int c_t = (t & 1) * kTcCodes + wt;
          unsigned todo = __ballot_sync(kFull, (any & 0x80008000u) && ((vb_t >> (c_t & 7)) & 1u) &&
                                                   !(kTcwDbg && (a.dbg & 1)));
          if (todo) {
            const int64_t pos0 = pos_w + (int64_t)t * kTcCodes;
            while (todo) {
              const int src = __ffs(todo) - 1;
              todo &= todo - 1;
              if (rh - *(volatile unsigned *)&g_tcw.tail[w] >= (unsigned)kTcwSlots) {
                // ring full (a burst under a still loose bound): this warp
                // runs the per-pair path itself instead of waiting
                uint32_t *xf = s.xfer[w][0];
                if (lane == src) {
#pragma unroll
                  for (int i = 0; i < NM / 2; i += 4)
                    *(uint4 *)&xf[i] = make_uint4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                }
                __syncwarp();
                const bool on = lane < NM / 2;
                const uint32_t vv = on ? xf[lane] : 0u;
                const int q = qb + 2 * (lane & (NM / 2 - 1));
                const uint32_t x = *(const uint32_t *)&s.thr16[q] - vv;
                __syncwarp();
                tc_hit_warp(a, on && (x & 0x8000u) != 0, on && (x & 0x80000000u) != 0, q, vv, pos0 + src, 640u);
                continue;
              }
              if (lane == src) {
                // No fence between the entry and its publication: one
                // thread's shared-memory stores are performed in program
                // order (in-order LSU, nothing cached between an SM's warps
                // and its shared memory); the volatile accesses and the asm
                // barrier keep the compiler from reordering them.
                volatile TcwEnt &e = g_tcw.ent[w][rh % kTcwSlots];
#pragma unroll
                for (int i = 0; i < NM / 2; i++) e.sums[i] = v[i];
                e.pos = pos0 + src;
                asm volatile("" ::: "memory");
                *(volatile unsigned *)&g_tcw.head[w] = rh + 1;
              }
              rh++;
            }
          }
          if (wt < nq && mpre < s.mc[qb + wt]) {  // bounds tightened by the flusher or other CTAs
            s.mc[qb + wt] = mpre;
            const int th = q_threshold(__uint_as_float(mpre), s.qmin[qb + wt], s.delta[qb + wt]);
            if (th + 0x8000 < (int)s.thr16[qb + wt]) s.thr16[qb + wt] = (uint16_t)(th + 0x8000);
          }
#pragma unroll
          for (int i = 0; i < WPC; i++) {
            cw[i] = cn[i];
            cn[i] = cf[i];
          }
        }
      };
      if (n_mma == 16) run(std::integral_constant<int, 16>{});
      else run(std::integral_constant<int, 32>{});
      // the filter warp reads this item's thresholds and query state: drain
      // the warp's ring before the next item is staged
      while (*(volatile unsigned *)&g_tcw.tail[w] != rh) __nanosleep(40);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      wg_sync();  // end of item: every tile read, g_tcw.item holds the next item
    }
    if (wt == 0) atomicAdd(&s.done, 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s.tmem), "n"(kCols));
}

template <int MC>
void launch_tcw(const ScanArgs &a, int nsm, cudaStream_t st) {
  const size_t smem = (size_t)kWG * kTcwNQ * 16 * MC;
  cudaFuncSetAttribute(k_scan_tcw<MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_scan_tcw<MC><<<nsm, 128 * kWG + 32 + 32 * kWG, smem, st>>>(a);
}


// ---- survivors of the two-SM scan: per-warp rings drained by 4 flushers ----
// A compute warp hands the packed sums of its codes with survivors to a
// flusher warp through its own single-producer ring (slots claimed
// warp-synchronously: no atomics, one fence and one head store per tile).
// The flusher re-runs the SWAR test per query column, computes midpoints,
// filters by the cached bound and appends (compacted, up to 32 candidates'
// slot claims and id reads in flight together). Compute warps, on whose
// timeliness every MMA depends, never run the per-pair survivor path.
constexpr int kWRing = 10;      // slots per compute warp
constexpr int kFlushers = 4;    // flusher warps (flusher f serves compute warps kPerF f .. kPerF f + kPerF - 1)
constexpr int kPerF = 16 / kFlushers;
struct Tc2Ent {
  uint32_t sums[32];  // packed pairs: columns col0 + 2 i (low half), + 1 (high)
  int64_t pos;        // code position (chunk * 256 + code)
  int col0;
  int pad;
};
struct Tc2Cand {
  int query;
  float mid;
  int64_t pos;
};
struct Tc2Smem {
  uint32_t tmem;
  int done;
  unsigned whead[16];  // per compute warp: slots published (monotone)
  unsigned wtail[16];  // per compute warp: slots consumed by its flusher
  int query[kTcNQ];
  float qmin[kTcNQ];
  float delta[kTcNQ];
  __align__(16) uint16_t thr16[kTcNQ];
  unsigned mc[kTcNQ];
  __align__(16) Tc2Ent ent[16][kWRing];
  Tc2Cand clist[kFlushers][96];
};
__shared__ Tc2Smem g_tc2;

// Bound of one query per lane (lane-parallel: all crossing queries of an
// append batch refresh in two L2 round trips): coarse sums, then the fine
// bins of the coarse bucket holding the R-th candidate.
__device__ __forceinline__ unsigned hist_bound_lane(const ScanArgs &a, int query) {
  const float hw = a.hist_w[query];
  if (!(hw > 0.f)) return 0x7f800000u;
  const unsigned *h = a.hist + (size_t)query * kHistWords;
  const unsigned R = (unsigned)a.R;
  uint4 c4[8];
#pragma unroll
  for (int i = 0; i < 8; i++) c4[i] = __ldcg((const uint4 *)(h + kHistBins) + i);
  unsigned cum = 0;
  int k = -1;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const unsigned w4[4] = {c4[i].x, c4[i].y, c4[i].z, c4[i].w};
#pragma unroll
    for (int j = 0; j < 4; j++)
      if (k < 0) {
        if (cum + w4[j] >= R) k = 4 * i + j;
        else cum += w4[j];
      }
  }
  if (k < 0) return 0x7f800000u;
  uint4 f4[8];
#pragma unroll
  for (int i = 0; i < 8; i++) f4[i] = __ldcg((const uint4 *)(h + 32 * k) + i);
  int b = 31;
  bool found = false;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const unsigned w4[4] = {f4[i].x, f4[i].y, f4[i].z, f4[i].w};
#pragma unroll
    for (int j = 0; j < 4; j++) {
      cum += w4[j];
      if (!found && cum >= R) {
        b = 4 * i + j;
        found = true;
      }
    }
  }
  return fbits(__fmul_rn((float)(k * 32 + b + 2), hw));
}

// Appends the compacted candidates cl[0, cnt) (one per lane per pass) and
// refreshes the bound of queries crossing a multiple of bound_every.
__device__ __forceinline__ void tc2_append(const ScanArgs &a, const Tc2Cand *cl, int cnt) {
  const int lane = threadIdx.x & 31;
  for (int base = 0; base < cnt; base += 32) {
    const int i = base + lane;
    const bool has = i < cnt;
    int qy = 0;
    unsigned slot = 0;
    if (has) {
      qy = cl[i].query;
      const float mid = cl[i].mid;
      const int64_t id = a.ids[cl[i].pos];  // in flight with the slot claim
      slot = atomicAdd(&a.cand_n[qy], 1u);
      if (slot < (unsigned)a.cap_g) {
        const size_t o = (size_t)qy * a.cap_g + slot;
        a.cand_mid[o] = mid;
        a.cand_id[o] = id;
      }
      const float hw = a.hist_w[qy];
      if (hw > 0.f) {
        unsigned *h = a.hist + (size_t)qy * kHistWords;
        const int b = min((int)__fmul_rn(mid, __frcp_rn(hw)), kHistBins - 1);
        atomicAdd(&h[b], 1u);
        atomicAdd(&h[kHistBins + (b >> 5)], 1u);  // coarse sums (hist_bound_lane)
      }
    }
    if (has && (slot + 1) % (unsigned)a.bound_every == 0)
      atomicMin(&a.M_bits[qy], hist_bound_lane(a, qy));
  }
}

__device__ __forceinline__ void tc2_flusher(const ScanArgs &a, int f) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  Tc2Cand *cl = g_tc2.clist[f];
  unsigned tail[kPerF] = {};
  for (;;) {
    bool busy = false;
#pragma unroll
    for (int r = 0; r < kPerF; r++) {
      const int cwi = kPerF * f + r;
      const unsigned head = *(volatile unsigned *)&g_tc2.whead[cwi];
      if (head == tail[r]) continue;
      busy = true;
      __threadfence_block();  // the entries' contents before their head
      int cnt = 0;
      for (unsigned k = tail[r]; k != head; k++) {
        const Tc2Ent &e = g_tc2.ent[cwi][k % kWRing];
        const uint32_t vv = e.sums[lane];
        const int64_t pos = e.pos;
        const int q = e.col0 + 2 * lane;
        __syncwarp();  // the slot is free once every lane holds its part
        if (lane == 0) *(volatile unsigned *)&g_tc2.wtail[cwi] = k + 1;
        const uint32_t x = *(const uint32_t *)&g_tc2.thr16[q] - vv;
        bool c[2];
        float md[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          c[h] = false;
          md[h] = 0.f;
          if (x & (0x8000u << (16 * h))) {
            md[h] = midpoint(g_tc2.qmin[q + h], g_tc2.delta[q + h], (int)((vv >> (16 * h)) & 0xffffu));
            c[h] = md[h] <= __uint_as_float(g_tc2.mc[q + h]);
          }
        }
        const unsigned b0 = __ballot_sync(kFull, c[0]), b1 = __ballot_sync(kFull, c[1]);
        if (c[0]) cl[cnt + __popc(b0 & lt)] = {g_tc2.query[q], md[0], pos};
        if (c[1]) cl[cnt + __popc(b0) + __popc(b1 & lt)] = {g_tc2.query[q + 1], md[1], pos};
        cnt += __popc(b0) + __popc(b1);
        if (cnt > 32) {  // room for the next entry's up to 64
          __syncwarp();
          tc2_append(a, cl, cnt);
          __syncwarp();
          cnt = 0;
        }
      }
      __syncwarp();
      tail[r] = head;
      if (cnt) tc2_append(a, cl, cnt);
      __syncwarp();
    }
    if (!busy) {
      if (*(volatile int *)&g_tc2.done) {
        bool empty = true;
#pragma unroll
        for (int r = 0; r < kPerF; r++)
          empty = empty && *(volatile unsigned *)&g_tc2.whead[kPerF * f + r] == tail[r];
        if (empty) break;
      }
      __nanosleep(64);
    }
  }
}

// ---- two-SM variant (cta_group::2): one tile = one 256-code chunk ----
// A CTA pair (cluster of 2) shares every MMA: M = 256 codes (CTA r expands
// codes 128 r .. 128 r + 127 of the chunk into its own shared memory), N =
// the item's queries (CTA r holds B rows r N/2 .. (r + 1) N/2 - 1), D = 128
// codes x N sums in each CTA's TMEM. Halving B per CTA frees the shared
// memory for a double-buffered A, so TMEM holds a double-buffered D
// (2 x 256 columns): the MMA of tile t + 1 runs while the compute warps
// read and test tile t, and the tensor pipe no longer waits for the
// epilogue. CTA 0's MMA warp issues for both; the compute warps of both
// CTAs arrive (remotely for CTA 1) on CTA 0's ready[t & 1] barrier once
// A(t) is written and D(t & 1) is free; the MMA commit is multicast to
// done[t & 1] in both CTAs. Items are assigned statically (pair p takes
// items p, p + P, ...): both CTAs walk the same sequence without
// communicating.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <int MH>
__device__ __forceinline__ void tc2_expand(uint32_t a_row, const uint32_t (&cw)[MH], int c) {
  const int sh = 4 * (c & 7);
#pragma unroll
  for (int j = 0; j < MH; j++) {
    const uint32_t s8 = ((cw[j] >> sh) << 3) & 0x78u;
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a_row + 128 * j),
                 "r"(tc_shl(s8)), "r"(tc_shl(s8 - 32u)), "r"(tc_shl(s8 - 64u)),
                 "r"(tc_shl(s8 - 96u))
                 : "memory");
  }
}

template <int MC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128 * 4 + 32 * (kFlushers + 1), 1)
    k_scan_tc2(const __grid_constant__ ScanArgs a) {
  constexpr int G = 4;
  constexpr int K = 16 * MC, SBO = 8 * K, MH = MC / G;
  constexpr int NT = 128 * G;           // compute threads
  constexpr int kCPT = kTcNQ / G;       // accumulator columns per compute thread
  constexpr int kATile = kTcCodes * K;  // bytes of one A buffer
  constexpr uint32_t kCols = 512;
  static_assert(MH >= 1 && kCPT == 64, "tile split");
  extern __shared__ __align__(16) unsigned char dsm[];
  Tc2Smem &s = g_tc2;
  uint8_t *sB = dsm;                           // [kTcNQ / 2][K]
  uint8_t *sA = dsm + (size_t)(kTcNQ / 2) * K; // [2][kTcCodes][K]
  __shared__ __align__(8) uint64_t ready[2], done[2];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const int row = tid & 127, part = tid >> 7, j0 = part * MH, col0 = part * kCPT;
  const uint32_t sB_a = (uint32_t)__cvta_generic_to_shared(sB);
  const uint32_t sA_a = (uint32_t)__cvta_generic_to_shared(sA);
  const uint32_t ready_a = (uint32_t)__cvta_generic_to_shared(&ready[0]);
  const uint32_t done_a = (uint32_t)__cvta_generic_to_shared(&done[0]);
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s.tmem)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ready_a), "n"(2 * 4 * G));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ready_a + 8), "n"(2 * 4 * G));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(done_a));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(done_a + 8));
    asm volatile("fence.mbarrier_init.release.cluster;");
    s.done = 0;
  }
  if (tid < 16) {
    s.whead[tid] = 0;
    s.wtail[tid] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s.tmem;
  const int n_items = *a.n_items;
  const int pair = blockIdx.x >> 1, npair = gridDim.x >> 1;
  if (w >= 4 * G && w < 4 * G + kFlushers) {
    tc2_flusher(a, w - 4 * G);
  } else if (w == 4 * G + kFlushers) {
    // ---- MMA issuer (CTA 0 only) ----
    if (rank == 0) {
      uint32_t gt = 0;
      for (int item = pair; item < n_items; item += npair) {
        const WorkItem it = a.items[item];
        const int nq = it.pair_count;
        const int n_mma = max(16, (nq + 15) & ~15);
        const uint32_t idesc = (2u << 4) | ((uint32_t)(n_mma >> 3) << 17) |
                               ((uint32_t)((2 * kTcCodes) >> 4) << 24);
        const int64_t ntiles = it.chunk_end - it.chunk_begin;
        for (int64_t t = 0; t < ntiles; t++, gt++) {
          const uint32_t b = gt & 1;
          tc_wait(ready_a + 8 * b, (gt >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (lane == 0) {
#pragma unroll
            for (int ks = 0; ks < K / 32; ks++) {
              const uint64_t da = tc_smem_desc(sA_a + b * kATile + ks * 256, SBO);
              const uint64_t db = tc_smem_desc(sB_a + ks * 256, SBO);
              const uint32_t acc = ks > 0 ? 1u : 0u;
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(
                      tmem + b * (uint32_t)kTcNQ),
                  "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                " [%0], %1;" ::"r"(done_a + 8 * b),
                "h"((uint16_t)3)
                : "memory");
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ---- compute warps ----
    const uint32_t t_row = tmem + ((uint32_t)((w & 3) * 32) << 16);
    // zero this thread's accumulator columns (both D buffers) once: see k_scan_tc
    {
      const uint32_t z[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int b = 0; b < 2; b++)
#pragma unroll
        for (int c = 0; c < kCPT; c += 16)
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
              "%12,%13,%14,%15,%16};" ::"r"(t_row + b * kTcNQ + col0 + c),
              "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]),
              "r"(z[7]), "r"(z[8]), "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]),
              "r"(z[14]), "r"(z[15])
              : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // remote (cluster) address of CTA 0's ready barriers
    uint32_t ready0;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ready0) : "r"(ready_a));
    // this thread's A row (code 128 rank + row of the chunk) in buffer 0
    const uint32_t a_row0 = sA_a + (uint32_t)((row >> 3) * SBO + 16 * (row & 7) + 128 * j0);
    const int crow = (int)rank * kTcCodes + row;  // code within the chunk
    uint32_t gt = 0;
    unsigned my_head = 0;  // warp-uniform: slots this warp has published
    auto arrive_ready = [&](uint32_t b) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(ready0 + 8 * b) : "memory");
    };
    for (int item = pair; item < n_items; item += npair) {
      const WorkItem it = a.items[item];
      const int nq = it.pair_count;
      const int n_mma = max(16, (nq + 15) & ~15);
      const int half = n_mma >> 1;
      const int64_t c0g = it.chunk_begin;
      const int64_t ntiles = it.chunk_end - it.chunk_begin;
      // every compute thread is past the previous item (its tiles' MMAs all
      // completed: B may be overwritten) and, once the flushers have consumed
      // every entry, so may the query state
      asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
      if (tid < 16)
        while (*(volatile unsigned *)&s.wtail[tid] != *(volatile unsigned *)&s.whead[tid]) __nanosleep(128);
      asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
      // ---- stage this CTA's half of B and the item's query state ----
      for (int e = tid; e < half * MC; e += NT) {
        const int r = e / MC, j = e - r * MC;
        const int q = (int)rank * half + r;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (q < nq) v = ((const uint4 *)a.qt)[(size_t)a.pair_t[it.pair_begin + q] * MC + j];
        *(uint4 *)(sB + (r >> 3) * SBO + j * 128 + (r & 7) * 16) = v;
      }
      if (tid < kTcNQ) {
        const int q = tid;
        int thr = -1;
        unsigned mb = 0;
        if (q < nq) {
          const int pi = it.pair_begin + q;
          const int query = a.pair_q[pi], t = a.pair_t[pi];
          s.query[q] = query;
          s.qmin[q] = a.qmin_f[t];
          s.delta[q] = a.delta_f[t];
          mb = *(volatile unsigned *)&a.M_bits[query];
          thr = q_threshold(__uint_as_float(mb), s.qmin[q], s.delta[q]);
        } else {
          s.query[q] = 0;
          s.qmin[q] = 0.f;
          s.delta[q] = 0.f;
        }
        s.thr16[q] = (uint16_t)(thr + 0x8000);
        s.mc[q] = mb;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
      // ---- prologue: expand tiles 0 and 1 (every earlier MMA completed:
      // both A buffers and both D buffers are free), load tile 2's words ----
      uint32_t cw[MH];
      tc_load<MC, MH>(a, c0g, crow, j0, cw);
      tc2_expand<MH>(a_row0 + (gt & 1) * kATile, cw, crow);
      arrive_ready(gt & 1);
      if (ntiles > 1) {
        tc_load<MC, MH>(a, c0g + 1, crow, j0, cw);
        tc2_expand<MH>(a_row0 + ((gt + 1) & 1) * kATile, cw, crow);
        arrive_ready((gt + 1) & 1);
        if (ntiles > 2) tc_load<MC, MH>(a, c0g + 2, crow, j0, cw);
      }
      // valid byte of this thread's code, one tile ahead (read by the
      // survivor path only)
      uint32_t vb_next = __ldg(a.valid + c0g * 32 + (crow >> 3));
      for (int64_t t = 0; t < ntiles; t++, gt++) {
        const uint32_t b = gt & 1;
        const int64_t g_t = c0g + t;
        unsigned mpre = 0;
        if (tid < nq) mpre = *(volatile unsigned *)&a.M_bits[s.query[tid]];
        // ---- tile t: wait for MMA(t) (handling stashed survivors while it
        // runs), copy the sums out of D[b] ----
        tc_wait(done_a + 8 * b, (gt >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint32_t v[kCPT / 2];
        tc_ld64p(t_row + b * kTcNQ + col0, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // ---- expand tile t + 2 into A[b] (its reader MMA(t) completed) and
        // release it with D[b]: MMA(t + 2) can follow MMA(t + 1) at once,
        // and the survivor test and hits of tile t below run while MMA(t + 1)
        // executes. Global loads are issued after the arrive, so its fence
        // never waits for them ----
        if (t + 2 < ntiles) {
          if (!(a.dbg & 2)) tc2_expand<MH>(a_row0 + b * kATile, cw, crow);
          arrive_ready(b);
          if (t + 3 < ntiles) tc_load<MC, MH>(a, c0g + t + 3, crow, j0, cw);
        }
        const uint32_t vb_t = vb_next;
        if (t + 1 < ntiles) vb_next = __ldg(a.valid + (g_t + 1) * 32 + (crow >> 3));
        const uint4 *T = (const uint4 *)&s.thr16[col0];
        uint32_t any = 0;
#pragma unroll
        for (int i = 0; i < kCPT / 2 && !(a.dbg & 8); i += 4) {
          const uint4 tt = T[i / 4];
          any |= (tt.x - v[i]) | (tt.y - v[i + 1]) | (tt.z - v[i + 2]) | (tt.w - v[i + 3]);
        }
        unsigned todo = __ballot_sync(kFull, (any & 0x80008000u) && !(a.dbg & 1));
        if (todo) {
          // validity (padding codes have id -1) is checked only here, off
          // the tile's critical path
          todo &= __ballot_sync(kFull, (vb_t >> (crow & 7)) & 1u);
          if (a.dbg & 256) todo = 0;  // timing experiment: test and validity, no hit handling
        }
        // hand the codes with survivors to this warp's flusher, up to a
        // ring's worth at a time
        while (todo) {
          const unsigned room = kWRing - (my_head - *(volatile unsigned *)&s.wtail[w]);
          const unsigned take = __shfl_sync(kFull, room, 0);
          if (take == 0) {
            __nanosleep(32);
            continue;
          }
          const unsigned lt = (1u << lane) - 1u;
          const unsigned rk = __popc(todo & lt);
          if (((todo >> lane) & 1u) && rk < take) {
            Tc2Ent &e = s.ent[w][(my_head + rk) % kWRing];
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *(uint4 *)&e.sums[i] = make_uint4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            e.pos = g_t * kChunkCodes + crow;
            e.col0 = col0;
            __threadfence_block();
          }
          const unsigned n = min((unsigned)__popc(todo), take);
          // drop the lanes just published from todo
          unsigned t2 = todo;
          for (unsigned k = 0; k < n; k++) t2 &= t2 - 1;
          todo = t2;
          __syncwarp();
          my_head += n;
          if (lane == 0) *(volatile unsigned *)&s.whead[w] = my_head;
        }
        if (tid < nq && mpre < s.mc[tid]) {
          s.mc[tid] = mpre;
          const int th = q_threshold(__uint_as_float(mpre), s.qmin[tid], s.delta[tid]);
          if (th + 0x8000 < (int)s.thr16[tid]) s.thr16[tid] = (uint16_t)(th + 0x8000);
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    if (tid == 0) *(volatile int *)&s.done = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();  // the pair's MMAs and tcgen05.ld are all complete
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(s.tmem), "n"(kCols));
}

// Inline-survivor variant of the CTA-pair scan (k_scan_tc2i): the compute
// warps handle their own survivors (stashed per warp, handled while waiting
// for the next MMA; one flusher warp appends). Used for shorter scans,
// whose survivors arrive mostly in the initial burst that the per-warp
// rings of k_scan_tc2 cannot absorb.
template <int MC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(576, 1)
    k_scan_tc2i(const __grid_constant__ ScanArgs a) {
  constexpr int G = 4;
  constexpr int K = 16 * MC, SBO = 8 * K, MH = MC / G;
  constexpr int NT = 128 * G;           // compute threads
  constexpr int kCPT = kTcNQ / G;       // accumulator columns per compute thread
  constexpr int kATile = kTcCodes * K;  // bytes of one A buffer
  constexpr uint32_t kCols = 512;
  static_assert(MH >= 1 && kCPT == 64, "tile split");
  extern __shared__ __align__(16) unsigned char dsm[];
  TcSmem &s = g_tc;
  uint8_t *sB = dsm;                           // [kTcNQ / 2][K]
  uint8_t *sA = dsm + (size_t)(kTcNQ / 2) * K; // [2][kTcCodes][K]
  __shared__ __align__(8) uint64_t ready[2], done[2];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const int row = tid & 127, part = tid >> 7, j0 = part * MH, col0 = part * kCPT;
  const uint32_t sB_a = (uint32_t)__cvta_generic_to_shared(sB);
  const uint32_t sA_a = (uint32_t)__cvta_generic_to_shared(sA);
  const uint32_t ready_a = (uint32_t)__cvta_generic_to_shared(&ready[0]);
  const uint32_t done_a = (uint32_t)__cvta_generic_to_shared(&done[0]);
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s.tmem)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ready_a), "n"(2 * 4 * G));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ready_a + 8), "n"(2 * 4 * G));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(done_a));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(done_a + 8));
    asm volatile("fence.mbarrier_init.release.cluster;");
    s.done = 0;
    s.head = 0;
    s.tail = 0;
  }
  for (int i = tid; i < kRing; i += blockDim.x) s.ring[i].query = -1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s.tmem;
  const int n_items = *a.n_items;
  const int pair = blockIdx.x >> 1, npair = gridDim.x >> 1;
  if (w == 4 * G) {
    tc_flusher(a);
  } else if (w == 4 * G + 1) {
    // ---- MMA issuer (CTA 0 only) ----
    if (rank == 0) {
      uint32_t gt = 0;
      for (int item = pair; item < n_items; item += npair) {
        const WorkItem it = a.items[item];
        const int nq = it.pair_count;
        const int n_mma = max(16, (nq + 15) & ~15);
        const uint32_t idesc = (2u << 4) | ((uint32_t)(n_mma >> 3) << 17) |
                               ((uint32_t)((2 * kTcCodes) >> 4) << 24);
        const int64_t ntiles = it.chunk_end - it.chunk_begin;
        for (int64_t t = 0; t < ntiles; t++, gt++) {
          const uint32_t b = gt & 1;
          tc_wait(ready_a + 8 * b, (gt >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (lane == 0) {
#pragma unroll
            for (int ks = 0; ks < K / 32; ks++) {
              const uint64_t da = tc_smem_desc(sA_a + b * kATile + ks * 256, SBO);
              const uint64_t db = tc_smem_desc(sB_a + ks * 256, SBO);
              const uint32_t acc = ks > 0 ? 1u : 0u;
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(
                      tmem + b * (uint32_t)kTcNQ),
                  "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                " [%0], %1;" ::"r"(done_a + 8 * b),
                "h"((uint16_t)3)
                : "memory");
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ---- compute warps ----
    const uint32_t t_row = tmem + ((uint32_t)((w & 3) * 32) << 16);
    // zero this thread's accumulator columns (both D buffers) once: see k_scan_tc
    {
      const uint32_t z[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int b = 0; b < 2; b++)
#pragma unroll
        for (int c = 0; c < kCPT; c += 16)
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
              "%12,%13,%14,%15,%16};" ::"r"(t_row + b * kTcNQ + col0 + c),
              "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]),
              "r"(z[7]), "r"(z[8]), "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]),
              "r"(z[14]), "r"(z[15])
              : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // remote (cluster) address of CTA 0's ready barriers
    uint32_t ready0;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ready0) : "r"(ready_a));
    // this thread's A row (code 128 rank + row of the chunk) in buffer 0
    const uint32_t a_row0 = sA_a + (uint32_t)((row >> 3) * SBO + 16 * (row & 7) + 128 * j0);
    const int crow = (int)rank * kTcCodes + row;  // code within the chunk
    uint32_t gt = 0;
    // Survivor stash: a lane with survivors parks its packed sums in shared
    // memory (up to 4 codes per warp) and the warp handles them while it
    // would otherwise wait for the next MMA, off the MMA's critical path.
    int ns = 0;  // warp-uniform
    auto process_one = [&](int k) {
      const uint32_t vv = s.xfer[w][k][lane];
      const int q = col0 + 2 * lane;
      const uint32_t x = *(const uint32_t *)&s.thr16[q] - vv;
      tc_hit_warp(a, (x & 0x8000u) != 0, (x & 0x80000000u) != 0, q, vv, s.stash_pos[w][k]);
      __syncwarp();
    };
    auto arrive_ready = [&](uint32_t b) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(ready0 + 8 * b) : "memory");
    };
    for (int item = pair; item < n_items; item += npair) {
      const WorkItem it = a.items[item];
      const int nq = it.pair_count;
      const int n_mma = max(16, (nq + 15) & ~15);
      const int half = n_mma >> 1;
      const int64_t c0g = it.chunk_begin;
      const int64_t ntiles = it.chunk_end - it.chunk_begin;
      // every compute thread is past the previous item (its tiles' MMAs all
      // completed: B and the query state may be overwritten; its stashed
      // survivors handled)
      while (ns > 0) process_one(--ns);
      asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
      // ---- stage this CTA's half of B and the item's query state ----
      for (int e = tid; e < half * MC; e += NT) {
        const int r = e / MC, j = e - r * MC;
        const int q = (int)rank * half + r;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (q < nq) v = ((const uint4 *)a.qt)[(size_t)a.pair_t[it.pair_begin + q] * MC + j];
        *(uint4 *)(sB + (r >> 3) * SBO + j * 128 + (r & 7) * 16) = v;
      }
      if (tid < kTcNQ) {
        const int q = tid;
        int thr = -1;
        unsigned mb = 0;
        if (q < nq) {
          const int pi = it.pair_begin + q;
          const int query = a.pair_q[pi], t = a.pair_t[pi];
          s.query[q] = query;
          s.qmin[q] = a.qmin_f[t];
          s.delta[q] = a.delta_f[t];
          mb = *(volatile unsigned *)&a.M_bits[query];
          thr = q_threshold(__uint_as_float(mb), s.qmin[q], s.delta[q]);
        } else {
          s.query[q] = 0;
          s.qmin[q] = 0.f;
          s.delta[q] = 0.f;
        }
        s.thr16[q] = (uint16_t)(thr + 0x8000);
        s.mc[q] = mb;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
      // ---- prologue: expand tiles 0 and 1 (every earlier MMA completed:
      // both A buffers and both D buffers are free), load tile 2's words ----
      uint32_t cw[MH];
      tc_load<MC, MH>(a, c0g, crow, j0, cw);
      tc2_expand<MH>(a_row0 + (gt & 1) * kATile, cw, crow);
      arrive_ready(gt & 1);
      if (ntiles > 1) {
        tc_load<MC, MH>(a, c0g + 1, crow, j0, cw);
        tc2_expand<MH>(a_row0 + ((gt + 1) & 1) * kATile, cw, crow);
        arrive_ready((gt + 1) & 1);
        if (ntiles > 2) tc_load<MC, MH>(a, c0g + 2, crow, j0, cw);
      }
      // valid byte of this thread's code, one tile ahead (read by the
      // survivor path only)
      uint32_t vb_next = __ldg(a.valid + c0g * 32 + (crow >> 3));
      for (int64_t t = 0; t < ntiles; t++, gt++) {
        const uint32_t b = gt & 1;
        const int64_t g_t = c0g + t;
        unsigned mpre = 0;
        if (tid < nq) mpre = *(volatile unsigned *)&a.M_bits[s.query[tid]];
        // ---- tile t: wait for MMA(t) (handling stashed survivors while it
        // runs), copy the sums out of D[b] ----
        while (ns > 0 && !tc_try_warp(done_a + 8 * b, (gt >> 1) & 1)) process_one(--ns);
        tc_wait(done_a + 8 * b, (gt >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint32_t v[kCPT / 2];
        tc_ld64p(t_row + b * kTcNQ + col0, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // ---- expand tile t + 2 into A[b] (its reader MMA(t) completed) and
        // release it with D[b]: MMA(t + 2) can follow MMA(t + 1) at once,
        // and the survivor test and hits of tile t below run while MMA(t + 1)
        // executes. Global loads are issued after the arrive, so its fence
        // never waits for them ----
        if (t + 2 < ntiles) {
          if (!(a.dbg & 2)) tc2_expand<MH>(a_row0 + b * kATile, cw, crow);
          arrive_ready(b);
          if (t + 3 < ntiles) tc_load<MC, MH>(a, c0g + t + 3, crow, j0, cw);
        }
        const uint32_t vb_t = vb_next;
        if (t + 1 < ntiles) vb_next = __ldg(a.valid + (g_t + 1) * 32 + (crow >> 3));
        const uint4 *T = (const uint4 *)&s.thr16[col0];
        uint32_t any = 0;
#pragma unroll
        for (int i = 0; i < kCPT / 2 && !(a.dbg & 8); i += 4) {
          const uint4 tt = T[i / 4];
          any |= (tt.x - v[i]) | (tt.y - v[i + 1]) | (tt.z - v[i + 2]) | (tt.w - v[i + 3]);
        }
        unsigned todo = __ballot_sync(kFull, (any & 0x80008000u) && !(a.dbg & 1));
        if (todo) {
          // validity (padding codes have id -1) is checked only here, off
          // the tile's critical path
          todo &= __ballot_sync(kFull, (vb_t >> (crow & 7)) & 1u);
          if (a.dbg & 256) todo = 0;  // timing experiment: test and validity, no hit handling
        }
        while (todo) {
          if (ns == 4) process_one(--ns);  // stash full: make room
          const int src = __ffs(todo) - 1;
          todo &= todo - 1;
          if (lane == src) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *(uint4 *)&s.xfer[w][ns][i] = make_uint4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            s.stash_pos[w][ns] = g_t * kChunkCodes + crow;
          }
          __syncwarp();
          ns++;
        }
        if (tid < nq && mpre < s.mc[tid]) {
          s.mc[tid] = mpre;
          const int th = q_threshold(__uint_as_float(mpre), s.qmin[tid], s.delta[tid]);
          if (th + 0x8000 < (int)s.thr16[tid]) s.thr16[tid] = (uint16_t)(th + 0x8000);
        }
      }
    }
    while (ns > 0) process_one(--ns);
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    if (tid == 0) *(volatile int *)&s.done = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();  // the pair's MMAs and tcgen05.ld are all complete
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(s.tmem), "n"(kCols));
}

template <int MC>
size_t tc2_smem_bytes() { return (size_t)(kTcNQ / 2) * 16 * MC + 2 * (size_t)kTcCodes * 16 * MC; }

template <int MC>
void launch_tc2(const ScanArgs &a, int nsm, cudaStream_t st) {
  const size_t smem = tc2_smem_bytes<MC>();
  if (a.pair_cta == 2) {
    cudaFuncSetAttribute(k_scan_tc2i<MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_scan_tc2i<MC>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    k_scan_tc2i<MC><<<nsm & ~1, 576, smem, st>>>(a);
    return;
  }
  cudaFuncSetAttribute(k_scan_tc2<MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_scan_tc2<MC>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  k_scan_tc2<MC><<<nsm & ~1, 128 * 4 + 32 * (kFlushers + 1), smem, st>>>(a);
}

template <int MC>
size_t tc_smem_bytes() { return (size_t)kTcNQ * 16 * MC; }

// Compute warp groups of the tensor-core scan: 4 (16 compute warps, each a
// quarter of the one-hot expansion and of the query columns: latency hidden
// by 4 warps per scheduler); QADC_B200_TC_GROUPS=2 selects 8 warps.
int tc_groups() {
  static const int g = scan_env_int("QADC_B200_TC_GROUPS", 4) == 2 ? 2 : 4;
  return g;
}

template <int MC, int G>
void launch_tc_g(const ScanArgs &a, int nsm, cudaStream_t st) {
  const size_t smem = tc_smem_bytes<MC>();
  cudaFuncSetAttribute(k_scan_tc<MC, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_scan_tc<MC, G>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  // TMEM: every resident CTA holds all 512 columns of its SM (A and D,
  // double-buffered): one CTA per SM
  k_scan_tc<MC, G><<<nsm, 128 * G + 32 + 32 * kMmaWarps, smem, st>>>(a);
}

template <int MC>
void launch_tc(const ScanArgs &a, int nsm, cudaStream_t st) {
  if (tc_groups() == 2) launch_tc_g<MC, 2>(a, nsm, st);
  else launch_tc_g<MC, 4>(a, nsm, st);
}

template <int MC>
int tc_resident(int nsm) {
  return nsm;
}

// ---- work list construction ----

__global__ void k_count_pairs(const int64_t *__restrict__ cells, int npairs, int nslots,
                              int *list_pairs, int *slot_cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += gridDim.x * blockDim.x) {
    const int L = cells ? (int)cells[i] : 0;
    atomicAdd(&list_pairs[L], 1);
    atomicAdd(&slot_cnt[(size_t)L * nslots + i % nslots], 1);
  }
}

// Per list: exclusive scan of its pair counts over probe slots, so a
// list's pairs are laid out by probe rank (its tiles then group queries
// for which this list is near the front of the probe order).
__global__ void k_slot_offsets(int *slot_cnt, int nlists, int nslots) {
  for (int L = blockIdx.x * blockDim.x + threadIdx.x; L < nlists; L += gridDim.x * blockDim.x) {
    int o = 0;
    for (int k = 0; k < nslots; k++) {
      const int c = slot_cnt[(size_t)L * nslots + k];
      slot_cnt[(size_t)L * nslots + k] = o;
      o += c;
    }
  }
}

// Exclusive scans of pairs and items over the lists, three small launches:
// per-block sums (one list per thread, coalesced), a one-block scan of the
// block sums, and the per-list offsets (block-level scan + block offset). The
// single-CTA version took 0.27 ms at K = 65 536 (64 strided lists per thread,
// two passes of dependent L2 round trips).
constexpr int kSlBlock = 1024;

__device__ __forceinline__ void sl_values(const int *__restrict__ list_pairs,
                                          const int64_t *__restrict__ chunk_off, int nlists,
                                          int qt_tile, int64_t range_chunks, int L, int64_t &it,
                                          int &pr) {
  it = 0;
  pr = 0;
  if (L < nlists) {
    const int p = list_pairs[L];
    const int64_t nch = chunk_off[L + 1] - chunk_off[L];
    it = (int64_t)((p + qt_tile - 1) / qt_tile) * ((nch + range_chunks - 1) / range_chunks);
    pr = p;
  }
}

// Block-wide inclusive scan of (it, pr); returns the block totals.
__device__ __forceinline__ void sl_block_scan(int64_t &it, int &pr, int64_t &tot_it, int &tot_pr) {
  __shared__ int64_t w_it[32];
  __shared__ int w_pr[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t a = __shfl_up_sync(0xffffffffu, it, o);
    const int c = __shfl_up_sync(0xffffffffu, pr, o);
    if (lane >= o) {
      it += a;
      pr += c;
    }
  }
  if (lane == 31) {
    w_it[w] = it;
    w_pr[w] = pr;
  }
  __syncthreads();
  if (w == 0) {
    int64_t a = w_it[lane];
    int c = w_pr[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t x = __shfl_up_sync(0xffffffffu, a, o);
      const int y = __shfl_up_sync(0xffffffffu, c, o);
      if (lane >= o) {
        a += x;
        c += y;
      }
    }
    w_it[lane] = a;
    w_pr[lane] = c;
  }
  __syncthreads();
  if (w > 0) {
    it += w_it[w - 1];
    pr += w_pr[w - 1];
  }
  tot_it = w_it[31];
  tot_pr = w_pr[31];
  __syncthreads();
}

__global__ void __launch_bounds__(kSlBlock) k_sl_partial(const int *__restrict__ list_pairs,
                                                        const int64_t *__restrict__ chunk_off,
                                                        int nlists, int qt_tile, int64_t range_chunks,
                                                        int64_t *blk_it, int *blk_pr) {
  int64_t it, tot_it;
  int pr, tot_pr;
  sl_values(list_pairs, chunk_off, nlists, qt_tile, range_chunks, blockIdx.x * kSlBlock + threadIdx.x,
            it, pr);
  sl_block_scan(it, pr, tot_it, tot_pr);
  if (threadIdx.x == 0) {
    blk_it[blockIdx.x] = tot_it;
    blk_pr[blockIdx.x] = tot_pr;
  }
}

// One block: exclusive scan of the block sums (any number of blocks, in
// rounds of kSlBlock) and the total item count.
__global__ void __launch_bounds__(kSlBlock) k_sl_blocks(int64_t *blk_it, int *blk_pr, int nblk,
                                                       int *n_items) {
  int64_t carry_it = 0;
  int carry_pr = 0;
  for (int base = 0; base < nblk; base += kSlBlock) {
    const int i = base + threadIdx.x;
    int64_t it = i < nblk ? blk_it[i] : 0, tot_it;
    int pr = i < nblk ? blk_pr[i] : 0, tot_pr;
    const int64_t own_it = it;
    const int own_pr = pr;
    sl_block_scan(it, pr, tot_it, tot_pr);
    if (i < nblk) {
      blk_it[i] = carry_it + it - own_it;
      blk_pr[i] = carry_pr + pr - own_pr;
    }
    carry_it += tot_it;
    carry_pr += tot_pr;
  }
  if (threadIdx.x == 0) *n_items = (int)carry_it;
}

__global__ void __launch_bounds__(kSlBlock) k_sl_final(const int *__restrict__ list_pairs,
                                                      const int64_t *__restrict__ chunk_off,
                                                      int nlists, int qt_tile, int64_t range_chunks,
                                                      const int64_t *__restrict__ blk_it,
                                                      const int *__restrict__ blk_pr, int *pair_off,
                                                      int64_t *item_off) {
  const int L = blockIdx.x * kSlBlock + threadIdx.x;
  int64_t it, tot_it;
  int pr, tot_pr;
  sl_values(list_pairs, chunk_off, nlists, qt_tile, range_chunks, L, it, pr);
  const int64_t own_it = it;
  const int own_pr = pr;
  sl_block_scan(it, pr, tot_it, tot_pr);
  if (L < nlists) {
    item_off[L] = blk_it[blockIdx.x] + it - own_it;
    pair_off[L] = blk_pr[blockIdx.x] + pr - own_pr;
  }
}

__global__ void k_scatter_pairs(const int64_t *__restrict__ cells, int npairs, int nslots,
                                const int *__restrict__ pair_off, const int *__restrict__ slot_off,
                                int *slot_fill, int32_t *pair_q, int32_t *pair_t) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += gridDim.x * blockDim.x) {
    const int L = cells ? (int)cells[i] : 0;
    const size_t ls = (size_t)L * nslots + i % nslots;
    const int pos = pair_off[L] + slot_off[ls] + atomicAdd(&slot_fill[ls], 1);
    pair_q[pos] = i / nslots;
    pair_t[pos] = i;
  }
}

// One CTA per list, threads over the list's (range, tile) items.
__global__ void k_emit_items(const int *__restrict__ list_pairs, const int *__restrict__ pair_off,
                             const int64_t *__restrict__ item_off, const int64_t *__restrict__ chunk_off,
                             int nlists, int qt_tile, int64_t range_chunks, WorkItem *items) {
  for (int L = blockIdx.x; L < nlists; L += gridDim.x) {
    const int p = list_pairs[L];
    if (p == 0) continue;
    const int64_t c0 = chunk_off[L], nch = chunk_off[L + 1] - c0;
    if (nch == 0) continue;
    const int tiles = (p + qt_tile - 1) / qt_tile;
    const int64_t ranges = (nch + range_chunks - 1) / range_chunks;
    for (int64_t k = threadIdx.x; k < ranges * tiles; k += blockDim.x) {
      const int64_t r = k / tiles;
      const int t = (int)(k - r * tiles);
      WorkItem wi;
      wi.list = L;
      wi.pair_begin = pair_off[L] + t * qt_tile;
      wi.pair_count = min(qt_tile, p - t * qt_tile);
      wi.variant = 0;
      wi.chunk_begin = c0 + r * range_chunks;
      wi.chunk_end = min(c0 + nch, wi.chunk_begin + range_chunks);
      items[item_off[L] + k] = wi;
    }
  }
}

// Stable partition of the items into buckets (probe rank, loop variant),
// 256 items per block: bucket + per-block bucket counts, a scan over
// blocks, then a scatter that keeps the original order inside each bucket
// (list / tile / range order keeps concurrently running CTAs on shared L2
// lines). Rank-major order scans every query's nearest cells first, so its
// bound has converged before the far cells; variant contiguity keeps one
// loop body hot in the instruction cache.
constexpr int kRankBuckets = 16;
constexpr int kBuckets = kRankBuckets * 8;

__global__ void k_item_class(WorkItem *__restrict__ items, const int *__restrict__ n_items,
                             const int32_t *__restrict__ pair_t,
                             const uint8_t *__restrict__ pair_depth, int qh, int nslots,
                             int rank_buckets, unsigned *__restrict__ blk_cnt) {
  __shared__ unsigned cnt[kBuckets];
  for (int k = threadIdx.x; k < kBuckets; k += blockDim.x) cnt[k] = 0;
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < *n_items) {
    const WorkItem it = items[i];
    int d = 16, rank = nslots;
    for (int q = 0; q < it.pair_count; q++) {
      const int t = pair_t[it.pair_begin + q];
      d = min(d, (int)pair_depth[t]);
      rank = min(rank, t % nslots);
    }
    const int half = it.pair_count <= qh ? 1 : 0;
    const int cls = half * 4 + (d >= 16 ? 0 : d >= 8 ? 1 : d >= 4 ? 2 : 3);
    const int bucket = min(rank, rank_buckets - 1) * 8 + cls;
    items[i].variant = d | (half << 8) | (bucket << 16);
    atomicAdd(&cnt[bucket], 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kBuckets; k += blockDim.x)
    blk_cnt[(size_t)blockIdx.x * kBuckets + k] = cnt[k];
}

__global__ void k_item_offsets(unsigned *__restrict__ blk_cnt, int nblk, unsigned *__restrict__ cls_n) {
  __shared__ unsigned tot[kBuckets];
  const int c = threadIdx.x;  // one thread per bucket
  unsigned t = 0;
  for (int b = 0; b < nblk; b++) t += blk_cnt[(size_t)b * kBuckets + c];
  tot[c] = t;
  __syncthreads();
  if (c < 8) {
    unsigned v = 0;
    for (int r = 0; r < kRankBuckets; r++) v += tot[r * 8 + c];
    cls_n[c] = v;  // items per loop variant
  }
  unsigned o = 0;
  for (int k = 0; k < c; k++) o += tot[k];
  for (int b = 0; b < nblk; b++) {
    const unsigned v = blk_cnt[(size_t)b * kBuckets + c];
    blk_cnt[(size_t)b * kBuckets + c] = o;
    o += v;
  }
}

__global__ void k_item_scatter(const WorkItem *__restrict__ in, const int *__restrict__ n_items,
                               const unsigned *__restrict__ blk_off, WorkItem *__restrict__ out) {
  __shared__ unsigned char bucket_of[256];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = i < *n_items;
  WorkItem it;
  int bk = 255;
  if (ok) {
    it = in[i];
    bk = (it.variant >> 16) & 255;
  }
  bucket_of[threadIdx.x] = (unsigned char)bk;
  __syncthreads();
  if (!ok) return;
  unsigned r = 0;
  for (int k = 0; k < (int)threadIdx.x; k++) r += bucket_of[k] == bk;
  out[blk_off[(size_t)blockIdx.x * kBuckets + bk] + r] = it;
}

}  // namespace

int64_t order_items_scratch(int64_t max_items) {
  return ((max_items + 255) / 256) * kBuckets + 16;
}

void order_items(const WorkItem *items, const int *n_items, int64_t max_items,
                 const int32_t *pair_t, const uint8_t *pair_depth, int qh, int nslots,
                 unsigned *scratch, WorkItem *out, cudaStream_t st) {
  const int nblk = (int)std::max<int64_t>((max_items + 255) / 256, 1);
  unsigned *cls_n = scratch, *blk = scratch + 16;
  static const int rank_buckets =
      std::min(kRankBuckets, std::max(1, scan_env_int("QADC_B200_RANK_BUCKETS", 4)));
  k_item_class<<<nblk, 256, 0, st>>>(const_cast<WorkItem *>(items), n_items, pair_t, pair_depth,
                                     qh, nslots, rank_buckets, blk);
  k_item_offsets<<<1, kBuckets, 0, st>>>(blk, nblk, cls_n);
  k_item_scatter<<<nblk, 256, 0, st>>>(items, n_items, blk, out);
}

// Queries per tile: 8 by default (selector construction amortized over 8
// queries at 96 registers, 5 CTAs/SM); QADC_B200_QT=4|16 overrides (tuning).
int scan_env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}

int scan_qt_per_cta(int m) {
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("QADC_B200_QT");
    env = e ? atoi(e) : 0;
  }
  if (env == 4 || env == 8 || env == 16) return (m > 64 && env > 4) ? 4 : env;
  return m <= 64 ? 8 : 4;
}

// Tensor-core scan for m in {16, 32}; the PRMT kernel otherwise, or when the
// call asks for it (QADC_B200_SCAN_PRMT) or QADC_B200_TC=0.
void tc_stats_dump() {
  unsigned long long h[4] = {0, 0, 0, 0};
  cudaMemcpyFromSymbol(h, g_tc_stats, sizeof(h));
  fprintf(stderr, "qadc_b200 tc stats: slow-path entries %llu, hits %llu, ring pushes %llu, direct %llu\n",
          h[0], h[1], h[2], h[3]);
  const unsigned long long z[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(g_tc_stats, z, sizeof(z));
}

bool scan_use_tc(int m, bool prmt) {
  static const int env = scan_env_int("QADC_B200_TC", 1);
  return !prmt && env != 0 && (m == 16 || m == 32);
}

int scan_tile_queries(int m, bool prmt, bool tcw) {
  return scan_use_tc(m, prmt) ? (tcw ? kTcwNQ : kTcNQ) : scan_qt_per_cta(m);
}

void launch_scan(const ScanArgs &a, int nsm, cudaStream_t st, bool prmt) {
  if (scan_use_tc(a.m, prmt)) {
    if (a.tcw) {
      if (a.m == 32) launch_tcw<32>(a, nsm, st);
      else launch_tcw<16>(a, nsm, st);
    } else if (a.pair_cta) {
      if (a.m == 32) launch_tc2<32>(a, nsm, st);
      else launch_tc2<16>(a, nsm, st);
    } else if (a.m == 32) launch_tc<32>(a, nsm, st);
    else launch_tc<16>(a, nsm, st);
    return;
  }
  const int qt = scan_qt_per_cta(a.m);
  if (qt == 16) {
    if (a.m == 32) launch_t<32, 16>(a, nsm, st);
    else launch_t<0, 16>(a, nsm, st);
  } else if (qt == 8) {
    if (a.m == 16) launch_t<16, 8>(a, nsm, st);
    else if (a.m == 32) launch_t<32, 8>(a, nsm, st);
    else launch_t<0, 8>(a, nsm, st);
  } else {
    if (a.m == 16) launch_t<16, 4>(a, nsm, st);
    else if (a.m == 32) launch_t<32, 4>(a, nsm, st);
    else launch_t<0, 4>(a, nsm, st);
  }
}

int scan_resident_ctas(int m, int cap_l, int nsm, int linear, bool prmt) {
  if (scan_use_tc(m, prmt)) return m == 32 ? tc_resident<32>(nsm) : tc_resident<16>(nsm);
  const int qt = scan_qt_per_cta(m);
  const bool lin = linear != 0;
  if (qt == 16) {
    if (m == 32) return lin ? resident_t<32, 16, true>(m, cap_l, nsm) : resident_t<32, 16, false>(m, cap_l, nsm);
    return resident_t<0, 16, false>(m, cap_l, nsm);
  }
  if (qt == 8) {
    if (m == 16) return lin ? resident_t<16, 8, true>(m, cap_l, nsm) : resident_t<16, 8, false>(m, cap_l, nsm);
    if (m == 32) return lin ? resident_t<32, 8, true>(m, cap_l, nsm) : resident_t<32, 8, false>(m, cap_l, nsm);
    return resident_t<0, 8, false>(m, cap_l, nsm);
  }
  if (m == 16) return lin ? resident_t<16, 4, true>(m, cap_l, nsm) : resident_t<16, 4, false>(m, cap_l, nsm);
  if (m == 32) return lin ? resident_t<32, 4, true>(m, cap_l, nsm) : resident_t<32, 4, false>(m, cap_l, nsm);
  return resident_t<0, 4, false>(m, cap_l, nsm);
}

int64_t build_work_scratch(int nlists, int nslots) {
  const int64_t nblk = (nlists + kSlBlock - 1) / kSlBlock;
  // per-list arrays, per-(list, slot) arrays, then the block sums of the
  // list scan (int64 items + int pairs per block, 8-byte aligned)
  return 6 * (int64_t)nlists + 8 + 2 * (int64_t)nlists * nslots + 3 * nblk + 2;
}

int64_t build_work(const qadc_b200_index *idx, const int64_t *cells, int nq, int nslots,
                   int qt_tile, int64_t range_chunks, int32_t *pair_q, int32_t *pair_t,
                   WorkItem *items, int *n_items, int *scratch, int64_t max_items,
                   cudaStream_t st) {
  (void)max_items;
  const int nl = idx->nlists;
  const int npairs = nq * nslots;
  int *list_pairs = scratch, *pair_off = scratch + nl;
  int64_t *item_off = (int64_t *)(scratch + 4 * nl + 2);  // 8-byte aligned region
  int *slot_off = scratch + 6 * nl + 8, *slot_fill = slot_off + (size_t)nl * nslots;
  cudaMemsetAsync(list_pairs, 0, sizeof(int) * nl, st);
  cudaMemsetAsync(slot_off, 0, sizeof(int) * 2 * (size_t)nl * nslots, st);
  const int g = std::min(std::max((npairs + 255) / 256, 1), 4096);
  k_count_pairs<<<g, 256, 0, st>>>(cells, npairs, nslots, list_pairs, slot_off);
  k_slot_offsets<<<(nl + 255) / 256, 256, 0, st>>>(slot_off, nl, nslots);
  {
    // block sums live behind the per-list scratch (build_work_scratch)
    const int nblk = (nl + kSlBlock - 1) / kSlBlock;
    int64_t *blk_it = (int64_t *)(scratch + 6 * (int64_t)nl + 8 + 2 * (int64_t)nl * nslots);
    int *blk_pr = (int *)(blk_it + nblk);
    k_sl_partial<<<nblk, kSlBlock, 0, st>>>(list_pairs, idx->chunk_off, nl, qt_tile, range_chunks,
                                             blk_it, blk_pr);
    k_sl_blocks<<<1, kSlBlock, 0, st>>>(blk_it, blk_pr, nblk, n_items);
    k_sl_final<<<nblk, kSlBlock, 0, st>>>(list_pairs, idx->chunk_off, nl, qt_tile, range_chunks,
                                           blk_it, blk_pr, pair_off, item_off);
  }
  k_scatter_pairs<<<g, 256, 0, st>>>(cells, npairs, nslots, pair_off, slot_off, slot_fill, pair_q,
                                     pair_t);
  k_emit_items<<<std::min(nl, 65535), 128, 0, st>>>(list_pairs, pair_off, item_off, idx->chunk_off,
                                                 nl, qt_tile, range_chunks, items);
  return 0;
}

}  // namespace qadc
