// Prototype (developer tool): Quick ADC lane sums as an int8 tcgen05 GEMM.
//
// lane_sum(code, query) = sum_j T_q[j][c_j] = onehot(code) . T_q  with the
// one-hot expansion (16 m bytes per code, one 1 per sub-quantizer) as the A
// operand (M = 128 codes, K-major, SMEM) and the uint8 tables of NQ queries
// as the B operand (N = NQ, K-major, SMEM, resident); D (int32) in TMEM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tc_proto tools/tc_proto.cu
//   tools/tc_proto check      # exact vs CPU
//   tools/tc_proto bench N    # throughput
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);    \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

constexpr int kM = 128;  // codes per tile (MMA M)

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <int M_SUB, int NQ, bool CHECK>
__global__ void __launch_bounds__(128) k_tc(const uint4 *__restrict__ rows, int64_t n,
                                            const uint4 *__restrict__ tables, int thr,
                                            int32_t *__restrict__ out, unsigned long long *sum) {
  constexpr int K = 16 * M_SUB;          // bytes per one-hot row
  constexpr int SBO = 8 * K;             // bytes between 8-row core-matrix groups
  constexpr int TCOLS = NQ < 32 ? 32 : NQ;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *sB = smem;                    // [NQ rows][K]
  uint8_t *sA = smem + NQ * K;           // [128 rows][K]
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, w = tid >> 5;
  const uint32_t sB_a = (uint32_t)__cvta_generic_to_shared(sB);
  const uint32_t sA_a = (uint32_t)__cvta_generic_to_shared(sA);
  const uint32_t mbar_a = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_slot)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_a));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // tables -> B (canonical K-major, no swizzle): row n, 16-byte column j
  for (int e = tid; e < NQ * M_SUB; e += 128) {
    const int q = e / M_SUB, j = e % M_SUB;
    *(uint4 *)(sB + (q >> 3) * SBO + j * 128 + (q & 7) * 16) = tables[e];
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  // instruction descriptor: D s32, A/B u8, K-major, N = NQ, M = 128
  const uint32_t idesc = (2u << 4) | ((uint32_t)(NQ >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);
  uint32_t phase = 0;
  unsigned long long acc = 0;
  const int64_t ntiles = (n + kM - 1) / kM;
  uint4 nxt = make_uint4(0, 0, 0, 0);
  if (blockIdx.x * kM + tid < n) nxt = rows[blockIdx.x * kM + tid];
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t code = t * kM + tid;
    // one-hot expansion of this thread's code into A row `tid`
    const uint4 rw = nxt;
    const int64_t cn = (t + gridDim.x) * kM + tid;
    if (cn < n) nxt = rows[cn];
    const uint32_t wd[4] = {rw.x, rw.y, rw.z, rw.w};
    uint8_t *arow = sA + (tid >> 3) * SBO + (tid & 7) * 16;
#pragma unroll
    for (int j = 0; j < M_SUB; j++) {
      const uint32_t c = (wd[j >> 3] >> (4 * (j & 7))) & 15u;
      const uint64_t v = 1ull << ((c & 7u) << 3);
      const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
      uint4 oh = c < 8 ? make_uint4(lo, hi, 0, 0) : make_uint4(0, 0, lo, hi);
      if (code >= n) oh = make_uint4(0, 0, 0, 0);
      *(uint4 *)(arow + j * 128) = oh;
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int ks = 0; ks < K / 32; ks++) {
        const uint64_t da = smem_desc(sA_a + ks * 256, 128, SBO);
        const uint64_t db = smem_desc(sB_a + ks * 256, 128, SBO);
        const uint32_t accum = ks > 0 ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(accum));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          mbar_a)
                   : "memory");
    }
    // wait for the MMA
    asm volatile(
        "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(mbar_a),
        "r"(phase));
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
    for (int c0 = 0; c0 < NQ; c0 += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(w * 32) << 16) + c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
            "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
            "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      if (CHECK) {
        if (code < n)
          for (int i = 0; i < 32 && c0 + i < NQ; i++) out[code * NQ + c0 + i] = (int32_t)v[i];
      } else {
        uint32_t hits = 0;
#pragma unroll
        for (int i = 0; i < 32; i++) hits += (int)v[i] <= thr;
        acc += hits;
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
  }
  if (!CHECK) atomicAdd(sum, acc);
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS));
}

template <int M_SUB, int NQ>
int run(bool check, int64_t n);

int main(int argc, char **argv) {
  const bool check = argc > 1 && argv[1][0] == 'c';
  const int64_t n = check ? 5000 : (argc > 2 ? atoll(argv[2]) : 10000000);
  constexpr int M_SUB = 32;
  const int nqa = argc > 3 ? atoi(argv[3]) : 64;
  if (nqa == 128) return run<M_SUB, 128>(check, n);
  if (nqa == 256) return run<M_SUB, 256>(check, n);
  if (nqa == 32) return run<M_SUB, 32>(check, n);
  return run<M_SUB, 64>(check, n);
}

template <int M_SUB, int NQ>
int run(bool check, int64_t n) {
  const int K = 16 * M_SUB;
  std::vector<uint8_t> rows(n * (M_SUB / 2)), tab(NQ * K);
  srand(1);
  for (auto &x : rows) x = rand() & 255;
  for (auto &x : tab) x = rand() % 128;
  uint8_t *d_rows, *d_tab;
  int32_t *d_out = nullptr;
  unsigned long long *d_sum;
  CK(cudaMalloc(&d_rows, rows.size()));
  CK(cudaMalloc(&d_tab, tab.size()));
  CK(cudaMalloc(&d_sum, 8));
  CK(cudaMemset(d_sum, 0, 8));
  CK(cudaMemcpy(d_rows, rows.data(), rows.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_tab, tab.data(), tab.size(), cudaMemcpyHostToDevice));
  const size_t smem = (size_t)NQ * K + (size_t)kM * K;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  if (check) {
    CK(cudaMalloc(&d_out, (size_t)n * NQ * 4));
    auto kern = k_tc<M_SUB, NQ, true>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<nsm, 128, smem>>>((const uint4 *)d_rows, n, (const uint4 *)d_tab, 0, d_out, d_sum);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> out((size_t)n * NQ);
    CK(cudaMemcpy(out.data(), d_out, out.size() * 4, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t i = 0; i < n; i++)
      for (int q = 0; q < NQ; q++) {
        int s = 0;
        for (int j = 0; j < M_SUB; j++) {
          const int c = (rows[i * (M_SUB / 2) + j / 2] >> (4 * (j & 1))) & 15;
          s += tab[q * K + j * 16 + c];
        }
        if (s != out[i * NQ + q]) {
          if (bad < 5) printf("mismatch code %ld q %d: gpu %d cpu %d\n", (long)i, q, out[i * NQ + q], s);
          bad++;
        }
      }
    printf("check: %ld mismatches of %ld\n", (long)bad, (long)(n * NQ));
    return bad != 0;
  }
  auto kern = k_tc<M_SUB, NQ, false>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem));
  printf("smem %zu B, %d CTAs/SM\n", smem, per_sm);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 2; it++)
    kern<<<nsm * per_sm, 128, smem>>>((const uint4 *)d_rows, n, (const uint4 *)d_tab, 600, d_out, d_sum);
  CK(cudaDeviceSynchronize());
  const int reps = 5;
  cudaEventRecord(e0);
  for (int it = 0; it < reps; it++)
    kern<<<nsm * per_sm, 128, smem>>>((const uint4 *)d_rows, n, (const uint4 *)d_tab, 600, d_out, d_sum);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double pairs = (double)n * NQ;
  printf("n=%ld NQ=%d: %.3f ms, %.3g pairs/s, %.3g lookup-adds/s\n", (long)n, NQ, ms,
         pairs / (ms * 1e-3), pairs * M_SUB / (ms * 1e-3));
  return 0;
}
