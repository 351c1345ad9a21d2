// Coarse probe (ivf.py:166-182) and coarse assignment (kmeans.py:52-78) as
// ONE fused tcgen05 kernel per query batch: the Q x K dot
// products run on the 5th-generation tensor cores (bf16 operands from
// shared memory, fp32 accumulators in TMEM) and the epilogue selects the
// cells that can still reach a query's top ma on the fly — the Q x K score
// matrix never exists in HBM; a second kernel re-ranks those candidates by
// the exact NumPy-einsum-order distance (bit-identical to
// np.lexsort((cells, d2))[:ma] of ivf.py:178-180).
//
// Arithmetic (unchanged from the rigorous bound of the split-bf16 scheme):
//   * centring: q' = q - mu, c' = c - mu (mu = centroid mean) leaves every
//     squared distance unchanged and shrinks |q'| |c'|;
//   * split bf16: v = hi + lo (hi = bf16(v), lo = bf16(v - hi)); rows
//     [q_hi | q_hi | q_lo] . [c_hi | c_lo | c_hi] (K = 3d) give q'.c' up to
//     the dropped lo*lo term and the remainders (<= 3.1 * 2^-18 |q'| |c'|)
//     plus the fp32 accumulation error (<= 3d u sum|terms|), products exact;
//   * bounds: A = fl(|q'|^2 + |c'|^2 - 2 S), |A - D| <= mg = eps (|q'|^2 +
//     |c'|^2), eps = 2^-15 + 4 (3d) u + 16 u, and the einsum value E the
//     reference ranks by has |E - D| <= (d + 4) u D, so E lies in [L, U],
//     U = (A + mg)(1 + g), L = max(0, (A - mg)(1 - g)), g = (d + 4) u,
//     with directed rounding;
//   * selection: U* = the ma-th smallest U over all K cells. Each epilogue
//     thread owns one query and keeps the ma smallest U seen so far (T =
//     their max, never below U*), and emits every cell with L <= T at the
//     time it is seen: a superset of {L <= U*}. The re-rank kernel merges
//     the per-slice top-ma sets into U*, keeps the candidates with
//     L <= U*, computes their exact einsum distances and sorts (E, cell).
//     Overflowing candidate lists fall back to the exact scan of all K.
//
// Kernel structure (one CTA per SM: 128 queries x one slice of the
// centroids): warp 0 moves operand blocks with 1-D bulk async copies
// (cp.async.bulk + mbarrier transaction counts; both operands are stored in
// HBM already in the canonical no-swizzle K-major core-matrix layout, so a
// 16 / 32 KB block is one contiguous copy), warp 1 issues
// tcgen05.mma.cta_group::1.kind::f16 (M = 128, N = 256, K = 16; A resident
// in shared memory for the whole CTA, B streamed through a 2-stage ring in
// K-chunks of 64), warps 2-5 drain the double-buffered TMEM accumulator
// (2 x 256 columns) with tcgen05.ld and run the selection (a per-query
// max-heap of the kept U values in shared memory).
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.cuh"
#include "probe_util.cuh"

namespace qadc {
namespace {

constexpr int kNM = 128;          // queries per CTA (MMA M, TMEM lanes)
constexpr int kNN = 256;          // centroids per tile (MMA N)
constexpr int kNKC = 64;          // bf16 K elements per staged chunk (128-byte rows)
constexpr int kNStages = 2;       // B ring depth (shared memory also holds the kept-set heaps)
constexpr int kNMaxMa = 64;       // fused selection keeps <= 64 per query
constexpr int kNThreads = 192;    // warp 0 copies, warp 1 MMA, warps 2-5 epilogue
constexpr int kNABlock = kNM * kNKC * 2;  // 16 KB
constexpr int kNBBlock = kNN * kNKC * 2;  // 32 KB
constexpr int kNRerankWarps = 4;
constexpr int kNCand = 512;       // exact re-rank candidates per query

// Byte offset of element (r, k) inside one K-chunk block: core matrices of
// 8 rows x 16 bytes (128 contiguous bytes), K-adjacent core matrices 128 B
// apart (LBO), 8-row groups 1024 B apart (SBO).
__device__ __forceinline__ uint32_t core_off(int r, int kk) {
  return (uint32_t)((r >> 3) * 1024 + ((kk >> 3) << 7) + ((r & 7) << 4) + ((kk & 7) << 1));
}

__device__ __forceinline__ uint64_t nn_desc(uint32_t saddr) {
  // start >> 4, LBO = 128 B, SBO = 1024 B, sm100 descriptor version bit 46
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | (1ull << 46);
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tNN_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra NN_DONE;\n\tbra NN_WAIT;\n\tNN_DONE:\n\t}" ::"r"(mbar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_copy(uint32_t dst, const void *src, uint32_t bytes,
                                          uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}

// Index / query side: centroid mean (fp64 accumulation), centred split-bf16
// rows in the tiled layout (rows padded to RT with zeros), |v'|^2.
// One CTA per dimension: fp64 partial sums over strided rows, then a
// block reduction (the serial per-dimension loop took ms at K = 65536).
__global__ void __launch_bounds__(256) k_nn_mean(const float *__restrict__ C, int K, int d,
                                                 float *__restrict__ mu) {
  __shared__ double part[8];
  const int t = blockIdx.x;
  double s = 0.0;
  for (int k = threadIdx.x; k < K; k += blockDim.x) s += (double)C[(size_t)k * d + t];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < 8; w++) tot += part[w];
    mu[t] = (float)(tot / K);
  }
}

// One warp per row r < n_pad. coarse rows [hi | lo | hi], query rows
// [hi | hi | lo]; rows >= n are zero. Block (tile, chunk) of RT rows sits at
// ((tile * nch + chunk) * RT * 128) bytes.
template <int RT>
__global__ void k_nn_split(const float *__restrict__ V, int64_t n, int64_t n_pad, int d,
                           const float *__restrict__ mu, bool coarse_side,
                           uint8_t *__restrict__ out, float *__restrict__ n2) {
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (r >= n_pad) return;
  const int lane = threadIdx.x & 31;
  const int nch = 3 * d / kNKC;
  const int64_t tile = r / RT;
  const int rr = (int)(r % RT);
  uint8_t *base = out + (size_t)tile * nch * RT * 128;
  double acc = 0.0;
  for (int t = lane; t < d; t += 32) {
    float x = 0.f;
    if (r < n) x = __fsub_rn(V[(size_t)r * d + t], mu[t]);
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    const __nv_bfloat16 lo = __float2bfloat16_rn(__fsub_rn(x, __bfloat162float(hi)));
    const __nv_bfloat16 part[3] = {hi, coarse_side ? lo : hi, coarse_side ? hi : lo};
#pragma unroll
    for (int p = 0; p < 3; p++) {
      const int kk = p * d + t;
      *(__nv_bfloat16 *)(base + (size_t)(kk / kNKC) * RT * 128 + core_off(rr, kk % kNKC)) = part[p];
    }
    acc += (double)x * (double)x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && r < n) n2[r] = (float)acc;
}

// Pre-filter cell term: c2p = c2 (1 - e) rounded down (e = eps + 64u);
// padded to a multiple of 32 cells with +huge (never passes).
__global__ void k_nn_c2p(const float *__restrict__ c2, int K, int K_pad, float f,
                         float *__restrict__ out) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K_pad; k += gridDim.x * blockDim.x)
    out[k] = k < K ? __fmul_rd(c2[k], f) : 3.0e38f;
}

struct NnArgs {
  const uint8_t *qtiled;  // [q_tiles][nch][16 KB]
  const float *qn2;       // [nq]
  const uint8_t *ctiled;  // [c_tiles][nch][32 KB]
  const float *cn2;       // [K]
  int nq, K, nch, c_tiles, tiles_per_slice, ma, cap, nq_pad;
  float eps, gam;
  uint64_t *cand;         // [slices][nq_pad][cap]  (A bits << 32 | cell)
  int *cand_n;            // [slices][nq_pad]  (> cap: overflow)
  float *tops;            // [slices][nq_pad][kNMaxMa]
  float *dbg_S;           // diagnostics: raw dot products of CTA (0, 0), tile t0 ([128][256]) or null
  unsigned *bound;        // [nq_pad] per-query bound shared by the slices (float bits, atomicMin)
  const float *c2p;       // [K] c2 (1 - eps - 64u) rounded down: the pre-filter's cell term
  float pre_q;            // 1 - eps - 64u (the pre-filter's query factor, see the epilogue)
};

__global__ void __launch_bounds__(kNThreads, 1) k_nn_tc(const __grid_constant__ NnArgs a) {
  extern __shared__ __align__(1024) unsigned char nsm[];
  __shared__ __align__(8) uint64_t bars[2 * kNStages + 5];
  __shared__ uint32_t s_tmem;
  uint8_t *sA = nsm;                                      // nch x 16 KB
  uint8_t *sB = nsm + (size_t)a.nch * kNABlock;           // kNStages x 32 KB
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qtile = blockIdx.x, slice = blockIdx.y;
  const int t0 = slice * a.tiles_per_slice;
  const int t1 = min(a.c_tiles, t0 + a.tiles_per_slice);
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars);
  // bars: full[s], empty[s], tmem_full[2], tmem_empty[2], a_full
  auto full_b = [&](int s) { return bar0 + 8u * s; };
  auto empty_b = [&](int s) { return bar0 + 8u * (kNStages + s); };
  auto tfull_b = [&](int b) { return bar0 + 8u * (2 * kNStages + b); };
  auto tempty_b = [&](int b) { return bar0 + 8u * (2 * kNStages + 2 + b); };
  const uint32_t afull_b = bar0 + 8u * (2 * kNStages + 4);
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < kNStages; s++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full_b(s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty_b(s)));
    }
    for (int b = 0; b < 2; b++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tfull_b(b)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tempty_b(b)), "n"(kNM));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(afull_b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  const uint32_t sA_a = (uint32_t)__cvta_generic_to_shared(sA);
  const uint32_t sB_a = (uint32_t)__cvta_generic_to_shared(sB);

  if (w == 0) {
    // ---- operand copies ----
    if (lane == 0) {
      const uint32_t abytes = (uint32_t)a.nch * kNABlock;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(afull_b),
                   "r"(abytes)
                   : "memory");
      bulk_copy(sA_a, a.qtiled + (size_t)qtile * abytes, abytes, afull_b);
      int it = 0;
      for (int t = t0; t < t1; t++) {
        for (int c = 0; c < a.nch; c++, it++) {
          const int s = it % kNStages;
          const uint32_t round = (uint32_t)(it / kNStages);
          mbar_wait(empty_b(s), (round & 1u) ^ 1u);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full_b(s)),
                       "n"(kNBBlock)
                       : "memory");
          bulk_copy(sB_a + (uint32_t)s * kNBBlock,
                    a.ctiled + ((size_t)t * a.nch + c) * kNBBlock, kNBBlock, full_b(s));
        }
      }
    }
  } else if (w == 1) {
    // ---- MMA issue (one thread) ----
    // kind::f16: D f32 (bit 4), A bf16 (bits 7-9 = 1), B bf16 (bits 10-12
    // = 1), both K-major, N >> 3 at bit 17, M >> 4 at bit 24
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kNN >> 3) << 17) |
                           ((uint32_t)(kNM >> 4) << 24);
    mbar_wait(afull_b, 0);
    int it = 0;
    for (int t = t0, j = 0; t < t1; t++, j++) {
      const int buf = j & 1;
      mbar_wait(tempty_b(buf), ((uint32_t)(j >> 1) & 1u) ^ 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t dcol = tmem + (uint32_t)buf * kNN;
      for (int c = 0; c < a.nch; c++, it++) {
        const int s = it % kNStages;
        mbar_wait(full_b(s), (uint32_t)(it / kNStages) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (lane == 0) {
#pragma unroll
          for (int kk = 0; kk < kNKC / 16; kk++) {
            const uint64_t da = nn_desc(sA_a + (uint32_t)c * kNABlock + kk * 256);
            const uint64_t db = nn_desc(sB_a + (uint32_t)s * kNBBlock + kk * 256);
            const uint32_t acc = (c | kk) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dcol),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                  empty_b(s))
              : "memory");
          if (c == a.nch - 1)
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    tfull_b(buf))
                : "memory");
        }
        __syncwarp();
      }
    }
  } else {
    // ---- epilogue: one thread per query (TMEM lane) ----
    // Per batch of 32 cells: masks of candidates (L <= T) and of kept-set
    // insertions (U < T) from one branch-free pass, then only the set bits
    // are visited (a warp iterates as often as its busiest lane, not once
    // per cell whenever any lane inserts). The kept set is a max-heap of
    // ma values in shared memory, slot-major (bank = lane: conflict-free
    // for any slot pattern); its root is T.
    const int quarter = w & 3;  // warps 2..5 -> lanes 64, 96, 0, 32
    const int row = quarter * 32 + lane;
    const int q = qtile * kNM + row;
    const bool live = q < a.nq;
    const float a2 = live ? a.qn2[q] : 0.f;
    const float onep = __fadd_ru(1.f, a.gam), onem = __fsub_rd(1.f, a.gam);
    const int ma = a.ma;
    float *heap = (float *)(sB + (size_t)kNStages * kNBBlock) + row;     // [ma][kNM]
    float *stage = heap + (size_t)kNMaxMa * kNM;                           // [32][kNM] S
    for (int i = 0; i < ma; i++) heap[i * kNM] = __int_as_float(0x7f800000);
    float T = __int_as_float(0x7f800000);  // this slice's kept-set root
    int nc = 0;
    uint64_t *cand = a.cand + ((size_t)slice * a.nq_pad + (live ? q : 0)) * a.cap;
    // The slices of a query share a bound Tg = min over slices of their
    // kept-set roots (each >= U*, the global ma-th smallest U, so Tg >= U*):
    // a cell is kept / emitted only below min(T, Tg). Slices later in the
    // grid then start from an almost converged bound.
    unsigned *gb = a.bound + (live ? q : 0);
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    float Tg = __uint_as_float(*(volatile unsigned *)gb);
    for (int t = t0, j = 0; t < t1; t++, j++) {
      const int buf = j & 1;
      // the shared bound is read once per tile, requested before the wait
      const unsigned tg_next = *(volatile unsigned *)gb;
      mbar_wait(tfull_b(buf), (uint32_t)(j >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
      for (int b = 0; b < kNN / 32; b++) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
            "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31},"
            " [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
              "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
              "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
              "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(trow + (uint32_t)(buf * kNN + b * 32)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int kb = t * kNN + b * 32;
        if (a.dbg_S && qtile == 0 && slice == 0 && j == 0) {
#pragma unroll
          for (int i = 0; i < 32; i++) a.dbg_S[row * kNN + b * 32 + i] = __uint_as_float(v[i]);
        }
        // pass 1 (branch-free, ~4 instructions per cell): a conservative
        // pre-filter that never rejects a cell with L <= Tu. With
        // Y = fl(c2 (1 - e) - 2 S), e = eps + 64u, L <= Tu implies
        //   Y <= Tu / (1 - g) - a2 (1 - e) + 64u (a2 + Tu)
        // (A = a2 + c2 - 2 S and mg = eps (a2 + c2) up to rounding terms
        // of size u (a2 + 2 c2), which the extra 64u on both sides cover:
        // |S| <= (a2 + c2) / 2). Survivors get the exact L / U.
        const int nk = min(32, a.K - kb);
        const float Tu = fminf(T, Tg);
        const float thr = __fadd_ru(__fadd_ru(__fdiv_ru(Tu, onem), -a.pre_q * a2),
                                    __fmul_ru(3.9e-6f, __fadd_ru(a2, Tu)));
        uint32_t pmask = 0;
        const float4 *cp4 = (const float4 *)(a.c2p + kb);
#pragma unroll
        for (int i4 = 0; i4 < 8; i4++) {
          const float4 c4 = __ldg(cp4 + i4);
          const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const int i = 4 * i4 + u;
            stage[i * kNM] = __uint_as_float(v[i]);
            pmask |= (uint32_t)(__fmaf_rn(-2.f, __uint_as_float(v[i]), cc[u]) <= thr) << i;
          }
        }
        pmask &= (live && nk > 0) ? (nk >= 32 ? 0xffffffffu : ((1u << nk) - 1u)) : 0u;
        // exact bounds of the pre-filter's survivors: candidates (every
        // cell with L <= Tu; T only decreases, so the batch-start Tu is
        // conservative) and kept-set insertions (U below the current root
        // and the shared bound)
        const float T_before = T;
        while (pmask) {
          const int i = __ffs(pmask) - 1;
          pmask &= pmask - 1;
          const int k = kb + i;
          const float S = stage[i * kNM];
          const float c2 = __ldg(a.cn2 + k);
          const float n2 = __fadd_ru(a2, c2);
          const float A = __fmaf_rn(-2.f, S, __fadd_rn(a2, c2));
          const float mg = __fmul_ru(a.eps, n2);
          const float L = fmaxf(__fmul_rd(__fsub_rd(A, mg), onem), 0.f);
          if (!(L <= Tu)) continue;
          if (nc < a.cap) cand[nc] = ((uint64_t)__float_as_uint(A) << 32) | (uint32_t)k;
          nc++;
          const float U = fmaxf(__fmul_ru(__fadd_ru(A, mg), onep), 0.f);
          if (!(U < fminf(T, Tu))) continue;
          // replace the root of the kept-set max-heap, sift down
          int pos = 0;
          for (;;) {
            const int l = 2 * pos + 1;
            if (l >= ma) break;
            int c = l;
            float cv = heap[l * kNM];
            if (l + 1 < ma) {
              const float rv = heap[(l + 1) * kNM];
              if (rv > cv) {
                c = l + 1;
                cv = rv;
              }
            }
            if (!(cv > U)) break;
            heap[pos * kNM] = cv;
            pos = c;
          }
          heap[pos * kNM] = U;
          T = heap[0];
        }
        if (T < T_before && T < __uint_as_float(0x7f800000) && live)
          atomicMin(gb, __float_as_uint(T));
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty_b(buf)) : "memory");
      Tg = fminf(Tg, __uint_as_float(tg_next));
    }
    if (live) {
      a.cand_n[(size_t)slice * a.nq_pad + q] = nc;
      float *tp = a.tops + ((size_t)slice * a.nq_pad + q) * kNMaxMa;
      for (int i = 0; i < ma; i++) tp[i] = heap[i * kNM];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// One warp per query: U* from the slices' kept sets, the candidates with
// L <= U*, their exact einsum distances, top ma by (E, cell); overflow ->
// exact einsum of every cell.
__global__ void __launch_bounds__(kNRerankWarps * 32) k_nn_rerank(
    const NnArgs a, int slices, const float *__restrict__ coarse,
    const float *__restrict__ queries, int d, int64_t *__restrict__ cells, int tops_cap) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int vcap = tops_cap;  // power of two >= max(slices * ma, ma + kSelBuf)
  uint64_t *v = (uint64_t *)smem + (size_t)w * vcap;
  uint64_t *cq = (uint64_t *)smem + (size_t)kNRerankWarps * vcap + (size_t)w * kNCand;
  float *sq = (float *)((uint64_t *)smem + (size_t)kNRerankWarps * (vcap + kNCand)) + (size_t)w * d;
  const int q = blockIdx.x * kNRerankWarps + w;
  if (q >= a.nq) return;
  for (int t = lane; t < d; t += 32) sq[t] = queries[(size_t)q * d + t];
  const int ma = a.ma;
  bool overflow = false;
  for (int s = 0; s < slices; s++) overflow |= a.cand_n[(size_t)s * a.nq_pad + q] > a.cap;
  float Ustar = 0.f;
  if (!overflow) {
    // U* = the ma-th smallest of the slices' kept sets; only their finite
    // entries can matter (slices after the first mostly kept nothing below
    // the shared bound), so those are compacted before the sort
    const int n = slices * ma;
    int nf = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      float u = __int_as_float(0x7f800000);
      if (i < n) {
        const int s = i / ma, j = i - s * ma;
        u = a.tops[((size_t)s * a.nq_pad + q) * kNMaxMa + j];
      }
      const bool fin = u < 3.0e38f;
      const unsigned bal = __ballot_sync(0xffffffffu, fin);
      if (fin) v[nf + __popc(bal & ((1u << lane) - 1))] = (uint64_t)__float_as_uint(u);
      nf += __popc(bal);
    }
    int p2 = 1;
    while (p2 < max(nf, ma)) p2 <<= 1;
    for (int i = nf + lane; i < p2; i += 32) v[i] = ~0ull;
    __syncwarp();
    warp_sort_u64(v, p2);
    Ustar = nf >= min(ma, a.K) ? __uint_as_float((uint32_t)v[min(ma, a.K) - 1])
                               : __int_as_float(0x7f800000);
  }
  __syncwarp();
  const float a2 = a.qn2[q];
  const float onem = __fsub_rd(1.f, a.gam);
  int nc = 0;
  for (int s = 0; s < slices && !overflow; s++) {
    const int n = a.cand_n[(size_t)s * a.nq_pad + q];
    const uint64_t *cs = a.cand + ((size_t)s * a.nq_pad + q) * a.cap;
    for (int i0 = 0; i0 < n && !overflow; i0 += 32) {
      const int i = i0 + lane;
      bool take = false;
      uint32_t k = 0;
      if (i < n) {
        const uint64_t e = cs[i];
        k = (uint32_t)e;
        const float A = __uint_as_float((uint32_t)(e >> 32));
        const float c2 = a.cn2[k];
        const float mg = __fmul_ru(a.eps, __fadd_ru(a2, c2));
        const float L = fmaxf(__fmul_rd(__fsub_rd(A, mg), onem), 0.f);
        take = L <= Ustar;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, take);
      if (nc + __popc(bal) > kNCand) {
        overflow = true;
        break;
      }
      if (take) cq[nc + __popc(bal & ((1u << lane) - 1))] = (uint64_t)k;
      nc += __popc(bal);
    }
  }
  __syncwarp();
  if (!overflow) {
    for (int i = lane; i < nc; i += 32) {
      const int k = (int)cq[i];
      const float *crow = coarse + (size_t)k * d;
      const float E = einsum_sq([&](int t) { return crow[t]; }, sq, d);
      cq[i] = ((uint64_t)__float_as_uint(E) << 32) | (uint32_t)k;
    }
    __syncwarp();
    int p2 = 1;
    while (p2 < nc) p2 <<= 1;
    for (int i = nc + lane; i < p2; i += 32) cq[i] = ~0ull;
    __syncwarp();
    warp_sort_u64(cq, p2);
    for (int i = lane; i < ma; i += 32)
      cells[(size_t)q * ma + i] = i < nc ? (int64_t)(cq[i] & 0xffffffffu) : -1;
    return;
  }
  // overflow (massive near-ties): exact einsum of every cell
  int nb = 0, bn = 0;
  uint64_t T = ~0ull;
  for (int i0 = 0; i0 < a.K; i0 += 32) {
    const int k = i0 + lane;
    uint64_t key = ~0ull;
    if (k < a.K) {
      const float *crow = coarse + (size_t)k * d;
      const float E = einsum_sq([&](int t) { return crow[t]; }, sq, d);
      key = ((uint64_t)__float_as_uint(E) << 32) | (uint32_t)k;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, key < T);
    if (bal) {
      if (bn + __popc(bal) > kSelBuf) warp_merge(v, nb, bn, ma, T);
      const bool take = key < T;
      const unsigned bal2 = __ballot_sync(0xffffffffu, take);
      if (take) v[nb + bn + __popc(bal2 & ((1u << lane) - 1))] = key;
      bn += __popc(bal2);
      __syncwarp();
    }
  }
  warp_merge(v, nb, bn, ma, T);
  for (int i = lane; i < ma; i += 32) cells[(size_t)q * ma + i] = (int64_t)(v[i] & 0xffffffffu);
}

}  // namespace

bool probe_tc_supported(int K, int d, int ma) {
  return K >= kNN && d % kNKC == 0 && d <= 128 && ma >= 1 && ma <= kNMaxMa;
}

int probe_tc_prepare(const float *coarse, int K, int d, float **mu, void **ctiled, float **cn2,
                     cudaStream_t st) {
  const int c_tiles = (K + kNN - 1) / kNN;
  const int64_t k_pad = (int64_t)c_tiles * kNN;
  QADC_CUDA(cudaMalloc(mu, (size_t)d * 4));
  QADC_CUDA(cudaMalloc(ctiled, (size_t)k_pad * 3 * d * 2));
  QADC_CUDA(cudaMalloc(cn2, (size_t)K * 4));
  k_nn_mean<<<d, 256, 0, st>>>(coarse, K, d, *mu);
  k_nn_split<kNN><<<(unsigned)((k_pad * 32 + 255) / 256), 256, 0, st>>>(
      coarse, K, k_pad, d, *mu, true, (uint8_t *)*ctiled, *cn2);
  QADC_CUDA(cudaGetLastError());
  return kOk;
}

bool launch_probe_tc(const float *coarse, const float *mu, const void *ctiled, const float *cn2,
                     int K, int d, const float *queries, int nq, int ma, int64_t *cells,
                     cudaStream_t st, float *dbg_S, int *dbg_counts) {
  if (nq <= 0) return true;
  if (!probe_tc_supported(K, d, ma)) return false;
  (void)cudaGetLastError();  // a stale error of an earlier call must not read as ours
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int nch = 3 * d / kNKC;
  const int c_tiles = (K + kNN - 1) / kNN;
  // candidate capacity per (slice, query): the kept set's warm-up (ma) plus
  // its ~ma ln(cells / ma) later insertions and the bound's slack (an
  // overflowing query falls back to the exact scan, still exact)
  const int cap = ma == 1 ? 64 : (ma >= 16 ? 1024 : 512);
  // slices of the centroid range: whole waves of one-CTA-per-SM work
  static const int max_sl = std::max(1, std::min(16, scan_env_int("QADC_B200_PROBE_SLICES", 5)));
  auto pick_slices = [&](int qtiles) {
    int best = 1;
    double best_t = 1e30;
    for (int s = 1; s <= max_sl && s <= c_tiles; s++) {
      const int per = (c_tiles + s - 1) / s;
      const double waves = std::ceil((double)qtiles * s / nsm);
      const double t = waves * per + 0.02 * s * per;  // small cost per extra slice (merges)
      if (t < best_t * 0.999) {
        best_t = t;
        best = s;
      }
    }
    return best;
  };
  // query chunks: candidate buffers (slices x queries x cap) <= ~1 GB
  int64_t chunk_q = std::min<int64_t>(nq, 16384);
  while (chunk_q > kNM &&
         (int64_t)pick_slices((int)((chunk_q + kNM - 1) / kNM)) * chunk_q * cap * 8 > (1LL << 30))
    chunk_q = std::max<int64_t>(kNM, chunk_q / 2);
  const int64_t qpad_max = (chunk_q + kNM - 1) / kNM * kNM;
  const int max_slices = pick_slices((int)(qpad_max / kNM));
  uint8_t *qt = nullptr;
  float *qn2 = nullptr, *tops = nullptr;
  uint64_t *cand = nullptr;
  int *cand_n = nullptr;
  unsigned *bound = nullptr;
  float *c2p = nullptr;
  const double u = 1.0 / 16777216.0;
  const float eps = (float)(1.0 / 32768.0 + (4.0 * 3 * d + 16.0) * u);
  const float pre_f = (float)(1.0 - (double)eps - 64.0 * u);
  if (cudaMallocAsync(&c2p, (size_t)c_tiles * kNN * 4, st) != cudaSuccess ||
      cudaMallocAsync(&bound, (size_t)qpad_max * 4, st) != cudaSuccess ||
      cudaMallocAsync(&qt, (size_t)qpad_max * 3 * d * 2, st) != cudaSuccess ||
      cudaMallocAsync(&qn2, (size_t)qpad_max * 4, st) != cudaSuccess ||
      cudaMallocAsync(&cand, (size_t)max_slices * qpad_max * cap * 8, st) != cudaSuccess ||
      cudaMallocAsync(&cand_n, (size_t)max_slices * qpad_max * 4, st) != cudaSuccess ||
      cudaMallocAsync(&tops, (size_t)max_slices * qpad_max * kNMaxMa * 4, st) != cudaSuccess)
    return false;
  k_nn_c2p<<<(c_tiles * kNN + 255) / 256, 256, 0, st>>>(cn2, K, c_tiles * kNN, pre_f, c2p);
  const size_t smem = (size_t)nch * kNABlock + (size_t)kNStages * kNBBlock +
                      (size_t)(kNMaxMa + 32) * kNM * 4;  // + kept-set heaps and the S stage
  cudaFuncSetAttribute(k_nn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bool ok = true;
  for (int64_t q0 = 0; q0 < nq && ok; q0 += chunk_q) {
    const int n = (int)std::min<int64_t>(chunk_q, nq - q0);
    const int qtiles = (n + kNM - 1) / kNM;
    const int slices = std::min(max_slices, pick_slices(qtiles));
    NnArgs a;
    a.qtiled = qt;
    a.qn2 = qn2;
    a.ctiled = (const uint8_t *)ctiled;
    a.cn2 = cn2;
    a.nq = n;
    a.K = K;
    a.nch = nch;
    a.c_tiles = c_tiles;
    a.tiles_per_slice = (c_tiles + slices - 1) / slices;
    a.ma = ma;
    a.cap = cap;
    a.nq_pad = qtiles * kNM;
    a.eps = eps;
    a.gam = (float)((d + 4) * u);
    a.cand = cand;
    a.cand_n = cand_n;
    a.tops = tops;
    a.dbg_S = q0 == 0 ? dbg_S : nullptr;
    a.bound = bound;
    a.c2p = c2p;
    a.pre_q = pre_f;
    // 0x7f7f7f7f = 3.4e38: above every real U
    cudaMemsetAsync(bound, 0x7f, (size_t)a.nq_pad * 4, st);
    k_nn_split<kNM><<<(unsigned)(((int64_t)a.nq_pad * 32 + 255) / 256), 256, 0, st>>>(
        queries + (size_t)q0 * d, n, a.nq_pad, d, mu, false, qt, qn2);
    k_nn_tc<<<dim3(qtiles, slices), kNThreads, smem, st>>>(a);
    int vcap = 1;
    while (vcap < std::max(slices * ma, ma + kSelBuf)) vcap <<= 1;
    const size_t rsmem = (size_t)kNRerankWarps * (vcap + kNCand) * 8 + (size_t)kNRerankWarps * d * 4;
    cudaFuncSetAttribute(k_nn_rerank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
    k_nn_rerank<<<(n + kNRerankWarps - 1) / kNRerankWarps, kNRerankWarps * 32, rsmem, st>>>(
        a, slices, coarse, queries + (size_t)q0 * d, d, cells + (size_t)q0 * ma, vcap);
    ok = cudaGetLastError() == cudaSuccess;
    if (dbg_counts && q0 == 0) {  // diagnostics: slices, then per-(slice, query) candidate counts
      const int nc = std::min(slices * a.nq_pad, 1 << 20);
      cudaMemcpyAsync(dbg_counts, &slices, 4, cudaMemcpyHostToDevice, st);
      cudaMemcpyAsync(dbg_counts + 1, cand_n, (size_t)nc * 4, cudaMemcpyDeviceToDevice, st);
      cudaStreamSynchronize(st);
    }
  }
  cudaFreeAsync(bound, st);
  cudaFreeAsync(c2p, st);
  cudaFreeAsync(qt, st);
  cudaFreeAsync(qn2, st);
  cudaFreeAsync(cand, st);
  cudaFreeAsync(cand_n, st);
  cudaFreeAsync(tops, st);
  if (!ok) set_error("tensor-core probe launch failed");
  return ok;
}

}  // namespace qadc

// Diagnostics (C ABI, device pointers): the fused probe on nq queries with
// the raw dot products of the first CTA's first tile (S, 128 x 256 fp32)
// and the candidate counts ([0] = slices, then slices x nq_pad ints).
extern "C" __attribute__((visibility("default"))) int qadc_b200_debug_probe_tc(const float *coarse, int K, int d, const float *queries,
                                        int nq, int ma, int64_t *cells, float *S, int *counts,
                                        float *mu_out, void *stream) {
  using namespace qadc;
  cudaStream_t st = (cudaStream_t)stream;
  if (!probe_tc_supported(K, d, ma)) return kErrArgs;
  float *mu = nullptr, *cn2 = nullptr;
  void *cs = nullptr;
  if (int rc = probe_tc_prepare(coarse, K, d, &mu, &cs, &cn2, st)) return rc;
  const bool ok = launch_probe_tc(coarse, mu, cs, cn2, K, d, queries, nq, ma, cells, st, S, counts);
  cudaStreamSynchronize(st);
  if (mu_out) cudaMemcpy(mu_out, mu, (size_t)d * 4, cudaMemcpyDeviceToDevice);
  cudaFree(mu);
  cudaFree(cs);
  cudaFree(cn2);
  return ok ? kOk : kErrCuda;
}
