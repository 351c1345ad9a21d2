// Prototype of the Quick ADC lane-sum inner loop (throughput only, no
// candidate emission): measures (query, code) lookups/s for the PRMT
// lookup + byte-pair sum + 16-bit widening scheme on B200, with the adds
// either forced onto the FMA pipe (IMAD) or left to ptxas.
//
// Layout: chunk of 256 codes = m x 32 words; word (j, o) holds the 4-bit
// sub-code j of codes 8o..8o+7 (code k at bits 4k..4k+3).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

template <int M, int QT, bool FMA_ADDS, int CT, int JU>
__global__ void __launch_bounds__(128) k_scan(const uint32_t* __restrict__ codes, int nchunks,
                                               const uint4* __restrict__ tables, int nq,
                                               uint32_t one, uint32_t* out) {
  __shared__ uint4 st[QT * M];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint32_t best = 0xffffffffu;
  for (int qt0 = 0; qt0 < nq; qt0 += QT) {
    __syncthreads();
    for (int i = threadIdx.x; i < QT * M; i += blockDim.x) st[i] = tables[qt0 * M + i];
    __syncthreads();
    for (int c0 = (blockIdx.x * 4 + warp) * CT; c0 < nchunks; c0 += gridDim.x * 4 * CT) {
      uint32_t acc_a[CT][QT][2], acc_o[CT][QT][2];
#pragma unroll
      for (int cc = 0; cc < CT; cc++)
#pragma unroll
      for (int q = 0; q < QT; q++) acc_a[cc][q][0] = acc_a[cc][q][1] = acc_o[cc][q][0] = acc_o[cc][q][1] = 0;
#pragma unroll JU
      for (int j = 0; j < M; j += 2) {
        uint32_t A0[CT], A1[CT], A0x[CT], A1x[CT], B0[CT], B1[CT], B0x[CT], B1x[CT];
#pragma unroll
        for (int cc = 0; cc < CT; cc++) {
          const uint32_t* cw = codes + (size_t)min(c0 + cc, nchunks - 1) * M * 32 + lane;
          uint32_t w0 = __ldg(cw + j * 32), w1 = __ldg(cw + (j + 1) * 32);
          A0[cc] = w0; A1[cc] = w0 >> 16; A0x[cc] = w0 ^ 0x88888888u; A1x[cc] = A0x[cc] >> 16;
          B0[cc] = w1; B1[cc] = w1 >> 16; B0x[cc] = w1 ^ 0x88888888u; B1x[cc] = B0x[cc] >> 16;
        }
#pragma unroll
        for (int q = 0; q < QT; q++) {
          uint4 t = st[q * M + j], u = st[q * M + j + 1];
#pragma unroll
          for (int cc = 0; cc < CT; cc++) {
          uint32_t a0 = A0[cc], a1 = A1[cc], a0x = A0x[cc], a1x = A1x[cc];
          uint32_t b0 = B0[cc], b1 = B1[cc], b0x = B0x[cc], b1x = B1x[cc];
          uint32_t p0 = prmt(t.x, t.y, a0), p1 = prmt(t.z, t.w, a0x);
          uint32_t p2 = prmt(u.x, u.y, b0), p3 = prmt(u.z, u.w, b0x);
          uint32_t r0 = prmt(t.x, t.y, a1), r1 = prmt(t.z, t.w, a1x);
          uint32_t r2 = prmt(u.x, u.y, b1), r3 = prmt(u.z, u.w, b1x);
          uint32_t s0, s1;
          if (FMA_ADDS) {
            s0 = imad(p0, one, imad(p1, one, imad(p2, one, p3)));
            s1 = imad(r0, one, imad(r1, one, imad(r2, one, r3)));
            acc_a[cc][q][0] = imad(s0, one, acc_a[cc][q][0]);
            acc_a[cc][q][1] = imad(s1, one, acc_a[cc][q][1]);
            acc_o[cc][q][0] = imad(prmt(s0, 0, 0x4341), one, acc_o[cc][q][0]);
            acc_o[cc][q][1] = imad(prmt(s1, 0, 0x4341), one, acc_o[cc][q][1]);
          } else {
            s0 = p0 + p1 + p2 + p3;
            s1 = r0 + r1 + r2 + r3;
            acc_a[cc][q][0] += s0;
            acc_a[cc][q][1] += s1;
            acc_o[cc][q][0] += prmt(s0, 0, 0x4341);
            acc_o[cc][q][1] += prmt(s1, 0, 0x4341);
          }
          }
        }
      }
#pragma unroll
      for (int cc = 0; cc < CT; cc++)
#pragma unroll
      for (int q = 0; q < QT; q++) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
          uint32_t e = acc_a[cc][q][h] - (acc_o[cc][q][h] << 8);
          best = min(best, min(min(e & 0xffff, e >> 16), min(acc_o[cc][q][h] & 0xffff, acc_o[cc][q][h] >> 16)));
        }
      }
    }
  }
  atomicMin(out, best);
}

template <int M, int QT, bool F, int CT, int JU>
void bench(const char* name, int nchunks, int nq) {
  uint32_t *codes, *out;
  uint4* tables;
  size_t nw = (size_t)nchunks * M * 32;
  cudaMalloc(&codes, nw * 4);
  cudaMalloc(&tables, (size_t)nq * M * 16);
  cudaMalloc(&out, 4);
  cudaMemset(codes, 0x5a, nw * 4);
  cudaMemset(tables, 0x11, (size_t)nq * M * 16);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sms * 4;
  k_scan<M, QT, F, CT, JU><<<grid, 128>>>(codes, nchunks, tables, nq, 1u, out);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(a);
    k_scan<M, QT, F, CT, JU><<<grid, 128>>>(codes, nchunks, tables, nq, 1u, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  double lookups = (double)nchunks * 256 * nq * M;
  printf("{\"variant\": \"%s\", \"ju\": %d, \"ct\": %d, \"m\": %d, \"qt\": %d, \"ms\": %.4f, \"lookups_per_s\": %.4e, \"err\": \"%s\"}\n",
         name, JU, CT, M, QT, best, lookups / (best * 1e-3), cudaGetErrorString(cudaGetLastError()));
  cudaFree(codes);
  cudaFree(tables);
  cudaFree(out);
}

#include <cstring>
int main(int argc, char** argv) {
  const int nchunks = 16384;  // 4.2M codes
  int which = argc > 1 ? atoi(argv[1]) : -1;
  int v = 0;
#define B(...) if (which < 0 || which == v) bench<__VA_ARGS__>("v" #__VA_ARGS__, nchunks, 64); v++;
  B(32, 4, true, 1, 16)
  B(32, 4, true, 1, 2)
  B(32, 4, true, 1, 1)
  B(32, 8, true, 1, 2)
  B(32, 8, true, 1, 1)
  B(32, 4, true, 2, 2)
  B(32, 4, true, 2, 1)
  B(32, 8, true, 2, 1)
  B(32, 4, false, 1, 2)
  B(32, 8, false, 1, 1)
  B(32, 16, true, 1, 1)
  return 0;
}
