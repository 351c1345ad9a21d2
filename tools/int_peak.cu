// Integer issue-rate microbenchmark for the Quick ADC roofline (R_int).
//
// Measures, on the B200 it runs on, the sustained lane-instruction rate of
// the ops the LUT-lookup scan is built from: PRMT / IADD3 / LOP3 (ALU pipe)
// and IMAD (FMA pipe), alone and mixed 1:1. Each thread runs 8 independent
// dependency chains so latency is hidden; grid = 148 SMs x 8 CTAs x 256
// threads. Timed with CUDA events after a warm-up launch. Prints one JSON
// line. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 int_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t iadd3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("add.u32 %0, %1, %2; add.u32 %0, %0, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_peak(uint32_t seed, uint32_t one, uint32_t* out) {
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; i++) x[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
  uint32_t y = seed ^ 0x5bd1e995u;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (MODE == 0) x[i] = prmt(x[i], y, x[(i + 1) & 7]);
      if (MODE == 1) x[i] = iadd3(x[i], y, x[(i + 1) & 7]);
      if (MODE == 2) x[i] = imad(x[i], one, x[(i + 1) & 7]);
      if (MODE == 3) x[i] = lop3(x[i], y, x[(i + 1) & 7]);
      if (MODE == 4) {  // 1:1 PRMT + IMAD
        if (i & 1) x[i] = imad(x[i], one, x[(i + 1) & 7]);
        else x[i] = prmt(x[i], y, x[(i + 1) & 7]);
      }
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) r ^= x[i];
  if (r == 0x12345678u) out[0] = r;
}

template <int MODE>
double run(int sms) {
  uint32_t* out;
  cudaMalloc(&out, 4);
  dim3 grid(sms * 8), block(256);
  k_peak<MODE><<<grid, block>>>(1u, 1u, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(a);
    k_peak<MODE><<<grid, block>>>(1u + rep, 1u, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  double ops = (double)grid.x * block.x * ITERS * 8;
  cudaFree(out);
  return ops / (best * 1e-3);  // lane-instructions per second
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double prmt_r = run<0>(sms), iadd3_r = run<1>(sms), imad_r = run<2>(sms),
         lop3_r = run<3>(sms), mix_r = run<4>(sms);
  // the iadd3 mode issues two PTX adds that ptxas fuses into one IADD3
  printf("{\"sms\": %d, \"clock_khz\": %d, \"prmt_lane_ops_per_s\": %.4e, "
         "\"iadd3_lane_ops_per_s\": %.4e, \"imad_lane_ops_per_s\": %.4e, "
         "\"lop3_lane_ops_per_s\": %.4e, \"prmt_imad_mix_lane_ops_per_s\": %.4e}\n",
         sms, clk, prmt_r, iadd3_r, imad_r, lop3_r, mix_r);
  return 0;
}
