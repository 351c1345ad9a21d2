// Developer microbenchmark: cycles per tcgen05.mma instruction (32 bytes of K
// per row) by kind, M and N, A in TMEM or SMEM, back to back on one
// accumulator. Operand contents are zero (timing only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tc_kind_bench tools/tc_kind_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kTiles = 1024;

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__device__ __forceinline__ void wait_mb(uint32_t mb, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(mb), "r"(ph) : "memory");
}

// KIND: 0 = i8, 1 = f8f6f4 (e4m3 x e4m3 -> f32), 2 = f16 (bf16 -> f32), 3 = tf32
template <int KIND, bool ATMEM>
__global__ void __launch_bounds__(128, 1) k_bench(int M, int N, int ksteps, long long *cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, K = 32 * ksteps;
  for (int i = tid; i < (128 + N) * K / 16; i += 128) ((uint4 *)sm)[i] = make_uint4(0, 0, 0, 0);
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t sb = sa + 128 * K;
  uint32_t idesc = ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (KIND == 0) idesc |= (2u << 4);
  if (KIND == 1) idesc |= (1u << 4);
  if (KIND == 2) idesc |= (1u << 4) | (1u << 7) | (1u << 10);
  if (KIND == 3) idesc |= (1u << 4) | (2u << 7) | (2u << 10);
  const uint32_t a_t = tmem + 256;
  long long t0 = clock64();
  if (tid == 0) {
    for (int t = 0; t < kTiles; t++) {
      for (int ks = 0; ks < ksteps; ks++) {
        const uint64_t db = desc(sb + ks * 256, 8 * K);
        const uint64_t da = desc(sa + ks * 256, 8 * K);
        const uint32_t acc = ks > 0;
#define MMA_T(KS) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t" \
            "tcgen05.mma.cta_group::1.kind::" KS " [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), \
            "r"(a_t + ks * 8), "l"(db), "r"(idesc), "r"(acc))
#define MMA_S(KS) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t" \
            "tcgen05.mma.cta_group::1.kind::" KS " [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), \
            "l"(da), "l"(db), "r"(idesc), "r"(acc))
        if (ATMEM) {
          if (KIND == 0) MMA_T("i8"); else if (KIND == 1) MMA_T("f8f6f4"); else if (KIND == 2) MMA_T("f16"); else MMA_T("tf32");
        } else {
          if (KIND == 0) MMA_S("i8"); else if (KIND == 1) MMA_S("f8f6f4"); else if (KIND == 2) MMA_S("f16"); else MMA_S("tf32");
        }
      }
    }
    // one commit tracks every MMA issued before it
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb) : "memory");
    wait_mb(mb, 0);
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// NW warps issue concurrently (i8, A in TMEM), each its own accumulator (N <= 64 columns each)
__global__ void __launch_bounds__(128, 1) k_multi(int NW, int N, int ksteps, long long *cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar[4];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, K = 32 * ksteps, w = tid >> 5;
  for (int i = tid; i < (128 + N) * K / 16; i += 128) ((uint4 *)sm)[i] = make_uint4(0, 0, 0, 0);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid < 4) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar[tid])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t sb = sa + 128 * K;
  const uint32_t idesc = ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24) | (2u << 4);
  const uint32_t a_t = tmem + 256;
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar[w]);
  long long t0 = clock64();
  if ((tid & 31) == 0 && w < NW) {
    for (int t = 0; t < kTiles; t++) {
      for (int ks = 0; ks < ksteps; ks++) {
        const uint64_t db = desc(sb + ks * 256, 8 * K);
        const uint32_t acc = ks > 0;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + w * 64),
            "r"(a_t + ks * 8), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb) : "memory");
    wait_mb(mb, 0);
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// One warp, 16 MMAs per tile with operands = loop-invariant bases + compile-time
// offsets (no per-MMA register-to-uniform moves): the issue rate of clean code.
__global__ void __launch_bounds__(128, 1) k_clean(int N, long long *cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, K = 512;
  for (int i = tid; i < (128 + N) * K / 16; i += 128) ((uint4 *)sm)[i] = make_uint4(0, 0, 0, 0);
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm) + 128 * K;
  const uint32_t idesc = ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24) | (2u << 4);
  const uint32_t a_t = tmem + 256;
  const uint64_t db0 = desc(sb, 8 * K);
  long long t0 = clock64();
  if (tid < 32) {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    if (pred) {
      for (int t = 0; t < kTiles; t++) {
#pragma unroll
        for (int ks = 0; ks < 16; ks++)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
              "r"(a_t + ks * 8), "l"(db0 + 16ull * ks), "r"(idesc), "r"(1u));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb) : "memory");
      wait_mb(mb, 0);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

void run_clean(int N, int sms) {
  long long *d;
  cudaMalloc(&d, 1024);
  const size_t smem = (size_t)(128 + N) * 512;
  cudaFuncSetAttribute(k_clean, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_clean<<<sms, 128, smem>>>(N, d);
  k_clean<<<sms, 128, smem>>>(N, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("i8 one warp, uniform operands, N %3d: %6.1f cycles per mma  %s\n", N, (double)c / kTiles / 16,
         cudaGetErrorString(e));
  cudaFree(d);
}

void run_multi(int NW, int N, int sms) {
  const int ksteps = 16;
  long long *d;
  cudaMalloc(&d, 1024);
  const size_t smem = (size_t)(128 + N) * 32 * ksteps;
  cudaFuncSetAttribute(k_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_multi<<<sms, 128, smem>>>(NW, N, ksteps, d);
  k_multi<<<sms, 128, smem>>>(NW, N, ksteps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("i8 multi-warp issue NW %d N %3d: %6.1f cycles per mma (all warps' mmas counted)  %s\n", NW, N,
         (double)c / kTiles / ksteps / NW, cudaGetErrorString(e));
  cudaFree(d);
}

template <int KIND, bool ATMEM>
void run(int M, int N, int sms) {
  const int ksteps = 16;
  long long *d;
  cudaMalloc(&d, 1024);
  const size_t smem = (size_t)(128 + N) * 32 * ksteps;
  cudaFuncSetAttribute(k_bench<KIND, ATMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_bench<KIND, ATMEM><<<sms, 128, smem>>>(M, N, ksteps, d);
  k_bench<KIND, ATMEM><<<sms, 128, smem>>>(M, N, ksteps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  static const char *kn[4] = {"i8", "f8f6f4", "f16(bf16)", "tf32"};
  printf("%-10s A=%s M %3d N %3d: %6.1f cycles/mma  %s\n", kn[KIND], ATMEM ? "tmem" : "smem", M, N,
         (double)c / kTiles / ksteps, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_clean(16, sms); run_clean(32, sms); run_clean(64, sms); run_clean(128, sms);
  for (int nw = 1; nw <= 4; nw++) { run_multi(nw, 16, sms); run_multi(nw, 64, sms); }
  const int ns[6] = {16, 32, 64, 96, 128, 256};
  if (sms > 0) return 0;
  for (int i = 0; i < 6; i++) run<0, true>(128, ns[i], sms);
  for (int i = 0; i < 6; i++) run<1, true>(128, ns[i], sms);
  for (int i = 0; i < 6; i++) run<1, false>(128, ns[i], sms);
  for (int i = 0; i < 6; i++) run<2, true>(128, ns[i], sms);
  for (int i = 0; i < 6; i++) run<3, true>(128, ns[i], sms);
  for (int i = 0; i < 6; i++) run<0, true>(64, ns[i], sms);
  for (int i = 0; i < 6; i++) run<1, true>(64, ns[i], sms);
  for (int i = 0; i < 6; i++) run<1, false>(64, ns[i], sms);
  return 0;
}
