// Developer microbenchmark: int8 tcgen05.mma pacing for the tensor-core
// scan's shape (M = 128 codes, N = queries, K = 16 m bytes per tile as
// m/2 MMAs of K = 32). One CTA per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tc_mma_bench tools/tc_mma_bench.cu
//   tools/tc_mma_bench
//
// modes: 0 = A and B in SMEM, back to back; 1 = A in TMEM, back to back;
//        2 = A in TMEM, per tile commit, tile t+2 issued after tile t's
//            commit is observed (the scan's double-buffered chain without
//            any epilogue work);
//        6 / 7 = four independent accumulator chains (N <= 64), A in TMEM / SMEM;
//        4 = as 1, but the tile's K steps alternate between two
//            accumulators (two independent chains of ksteps / 2);
//        5 = single accumulator: tile t+1 issued after all 4 warps read
//            tile t's N columns (N = 256: the scan's single-D plan);
//        3 = as 2, plus all 4 warps wait for the commit and tcgen05.ld the
//            tile's N columns (x32 per warp per 32 columns) before the next
//            issue (issue gated by a named barrier, like the scan).
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

constexpr int kTiles = 2048;

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__device__ __forceinline__ void wait_mb(uint32_t mb, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(mb),
      "r"(ph)
      : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) k_bench(int N, int ksteps, long long *cyc) {
  extern __shared__ __align__(16) unsigned char sm[];  // A [128][K], B [N][K]
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, K = 32 * ksteps;
  for (int i = tid; i < (128 + N) * K / 16; i += 128) ((uint4 *)sm)[i] = make_uint4(0, 0, 0, 0);
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar[0]);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb + 8));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t sb = sa + 128 * K;
  const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t a_t = tmem + 256;  // A in TMEM columns 256.. (K/4 per buffer)
  long long t0 = clock64();
  uint32_t ph[2] = {0, 0};
  for (int t = 0; t < kTiles; t++) {
    const int buf = t & 1;
    if (MODE == 5 && t >= 1) {
      wait_mb(mb, ph[0]);
      ph[0] ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int c = 0; c < N; c += 32) {
        uint32_t v[4];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                     : "r"(tmem + ((uint32_t)(tid & 96) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (v[0] == 12345u) cyc[1] = v[1];
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;");
    }
    if (MODE >= 2 && MODE <= 3 && t >= 2) {
      if (MODE == 2) {
        if (tid == 0) wait_mb(mb + 8 * buf, ph[buf]);
        if (tid == 0 && blockIdx.x == 0 && t < 66) cyc[2 + 2 * t] = clock64() - t0;
      } else {
        wait_mb(mb + 8 * buf, ph[buf]);
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int c = 0; c < N; c += 32) {
          uint32_t v[4];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                       : "r"(tmem + ((uint32_t)(tid & 96) << 16) + buf * 128 + c));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (v[0] == 12345u) cyc[1] = v[1];
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
      ph[buf] ^= 1;
    }
    if (tid == 0) {
      for (int ks = 0; ks < ksteps; ks++) {
        const uint64_t db = desc(sb + ks * 256, 8 * K);
        const uint32_t acc = ks > 0;
        if (MODE == 6 || MODE == 7) {
          // four independent accumulator chains (N <= 64), A in TMEM (6) or SMEM (7)
          const uint32_t d = tmem + (ks & 3) * 64;
          const uint32_t acc4 = ks > 3;
          if (MODE == 6) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                "r"(a_t + buf * (K / 4) + ks * 8), "l"(db), "r"(idesc), "r"(acc4));
          } else {
            const uint64_t da = desc(sa + ks * 256, 8 * K);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                "l"(da), "l"(db), "r"(idesc), "r"(acc4));
          }
        } else if (MODE == 4) {
          const uint32_t d = tmem + (ks & 1) * 128;
          const uint32_t acc4 = ks > 1;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
              "r"(a_t + ks * 8), "l"(db), "r"(idesc), "r"(acc4));
        } else if (MODE == 5) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
              "r"(a_t + buf * (K / 4) + ks * 8), "l"(db), "r"(idesc), "r"(acc));
        } else if (MODE == 0) {
          const uint64_t da = desc(sa + ks * 256, 8 * K);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + buf * 128),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        } else {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + buf * 128),
              "r"(a_t + buf * (K / 4) + ks * 8), "l"(db), "r"(idesc), "r"(acc));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       MODE == 5 ? mb : mb + 8 * buf)
                   : "memory");
      if (MODE == 2 && blockIdx.x == 0 && t < 66) cyc[3 + 2 * t] = clock64() - t0;
    }
    __syncwarp();
  }
  // drain
  if (tid == 0) {
    if (MODE == 5) wait_mb(mb, ph[0]);
    for (int b = 0; b < 2; b++) {
      if (MODE >= 2 && MODE <= 3) wait_mb(mb + 8 * ((kTiles - 2 + b) & 1), ph[(kTiles - 2 + b) & 1]);
    }
    if (MODE < 2 || MODE == 4 || MODE == 6 || MODE == 7) {
      // every commit arrived once per tile: wait for the last phase of each buffer
      wait_mb(mb, (kTiles / 2 - 1) & 1);
      wait_mb(mb + 8, (kTiles / 2 - 1) & 1);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int MODE>
void run(int N, int ksteps, int sms) {
  long long *d;
  cudaMalloc(&d, 16 * 1024);
  const size_t smem = (size_t)(128 + N) * 32 * ksteps;
  cudaFuncSetAttribute(k_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_bench<MODE><<<sms, 128, smem>>>(N, ksteps, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_bench<MODE><<<sms, 128, smem>>>(N, ksteps, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double ops = (double)sms * kTiles * 128.0 * N * 32.0 * ksteps * 2.0;
  printf("mode %d N %3d ksteps %2d: %7.1f cycles/tile (ideal %5d), %7.1f TOP/s  %s\n", MODE, N,
         ksteps, (double)c / kTiles, 128 * N / 256 * ksteps, ops / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  if (MODE == 2) {
    long long h[140];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int t = 0; t < 24; t++)
      printf("  tile %2d: wait done %8lld  issued+committed %8lld\n", t, t >= 2 ? h[2 + 2 * t] : -1, h[3 + 2 * t]);
  }
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int ns[5] = {16, 32, 64, 128, 256};
  for (int i = 0; i < 5; i++) run<0>(ns[i], 16, sms);   // A, B in SMEM, one chain
  for (int i = 0; i < 5; i++) run<1>(ns[i], 16, sms);   // A in TMEM, one chain
  for (int i = 0; i < 4; i++) run<4>(ns[i], 16, sms);   // A in TMEM, two chains
  for (int i = 0; i < 3; i++) run<6>(ns[i], 16, sms);   // A in TMEM, four chains
  for (int i = 0; i < 3; i++) run<7>(ns[i], 16, sms);   // A in SMEM, four chains
  return 0;
}
