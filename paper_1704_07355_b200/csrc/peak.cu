// Peak microbenchmarks (the measured roofline denominators). Integer issue-rate microbenchmark: the measured denominator R_int of the
// scan's roofline ("measure them with a PRMT/LOP3/IADD3
// microbenchmark. Do not assume them"). Each thread runs 8 independent
// dependency chains of PRMT (ALU pipe) and/or IMAD (FMA pipe); the grid
// fills every SM 8 CTAs deep. Timed with CUDA events, best of 5.
#include "qadc_b200.h"
#include "internal.cuh"

namespace qadc {
namespace {

constexpr int kIters = 4096;

template <bool MIX>
__global__ void __launch_bounds__(256) k_peak(uint32_t seed, uint32_t one, uint32_t *out) {
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; i++) x[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
  const uint32_t y = seed ^ 0x5bd1e995u;
  for (int it = 0; it < kIters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (MIX && (i & 1)) x[i] = imad(x[i], one, x[(i + 1) & 7]);
      else x[i] = prmt(x[i], y, x[(i + 1) & 7]);
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) r ^= x[i];
  if (r == 0x12345678u) out[0] = r;
}

template <bool MIX>
int run(int sms, double *rate) {
  uint32_t *out = nullptr;
  QADC_CUDA(cudaMalloc(&out, 4));
  const dim3 grid(sms * 8), block(256);
  k_peak<MIX><<<grid, block>>>(1u, 1u, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(a);
    k_peak<MIX><<<grid, block>>>(2u + rep, 1u, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  QADC_CUDA(cudaGetLastError());
  *rate = (double)grid.x * block.x * kIters * 8 / (best * 1e-3);
  return kOk;
}

// int8 tensor-core rate: one CTA per SM issues back-to-back
// tcgen05.mma.cta_group::1.kind::i8 (M = 128, N = 256, K = 32; operands in
// SMEM, accumulator in TMEM), the shape family of the tensor-core scan.
constexpr int kMmaIters = 4096;

__global__ void __launch_bounds__(128, 1) k_mma_peak(int iters, uint32_t *out) {
  extern __shared__ __align__(16) unsigned char sm[];  // A [128][32] u8, B [256][32] u8
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 + 256) * 32 / 16; i += 128) ((uint4 *)sm)[i] = make_uint4(0, 0, 0, 0);
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
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
  if (tid == 0) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm);
    const uint64_t da = (uint64_t)((sa >> 4) & 0x3FFF) | (8ull << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
    const uint64_t db = (uint64_t)(((sa + 128 * 32) >> 4) & 0x3FFF) | (8ull << 16) |
                        ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
    const uint32_t idesc = (2u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int i = 0; i < iters; i++) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(1u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb)
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\n\tPK_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@P1 bra PK_DONE;\n\tbra PK_WAIT;\n\tPK_DONE:\n\t}" ::"r"(mb)
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  if (tid == 0 && iters < 0) out[0] = tmem;
}

int run_mma(int sms, double *rate) {
  uint32_t *out = nullptr;
  QADC_CUDA(cudaMalloc(&out, 4));
  const size_t smem = (128 + 256) * 32;
  k_mma_peak<<<sms, 128, smem>>>(64, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(a);
    k_mma_peak<<<sms, 128, smem>>>(kMmaIters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  QADC_CUDA(cudaGetLastError());
  *rate = (double)sms * kMmaIters * 128.0 * 256.0 * 32.0 * 2.0 / (best * 1e-3);
  return kOk;
}

}  // namespace
}  // namespace qadc

extern "C" int qadc_b200_mma_peak(double *out) {
  using namespace qadc;
  set_error("");
  if (!out) {
    set_error("null argument");
    return kErrArgs;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return run_mma(sms, out);
}

extern "C" int qadc_b200_int_peak(double *out) {
  using namespace qadc;
  set_error("");
  if (!out) {
    set_error("null argument");
    return kErrArgs;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int rc = run<true>(sms, &out[0]);
  if (!rc) rc = run<false>(sms, &out[1]);
  return rc;
}
