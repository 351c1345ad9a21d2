// Integer issue-rate microbenchmark: the measured denominator R_int of the
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

}  // namespace
}  // namespace qadc

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
