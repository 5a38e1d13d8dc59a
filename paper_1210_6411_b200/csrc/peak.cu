// Roofline denominator: the chip's sustained 32-bit LOP3 issue rate, measured.
// Every thread runs 8 independent LOP3 chains (inline PTX so nothing folds away); the
// grid fills every SM at full occupancy.  Reported as LOP3 results/s together with the
// SM clock observed during the run (clock64 ticks per %globaltimer ns).
#include <cuda_runtime.h>

#include <cstdint>

#include "lfsr_internal.h"

namespace lc {

namespace {

__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) lop3_peak_kernel(uint32_t iters, uint32_t* sink,
                                                        unsigned long long* clk) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, a4 = a0 * 11u, a5 = a0 * 13u,
           a6 = a0 * 17u, a7 = a0 * 19u;
  const uint32_t b = blockIdx.x * 0x9E3779B9u, c = ~b;
  const long long c0 = clock64();
  const uint64_t g0 = globaltimer();
#pragma unroll 1
  for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a0 = lop3(a0, b, c);
      a1 = lop3(a1, b, c);
      a2 = lop3(a2, b, c);
      a3 = lop3(a3, b, c);
      a4 = lop3(a4, b, c);
      a5 = lop3(a5, b, c);
      a6 = lop3(a6, b, c);
      a7 = lop3(a7, b, c);
    }
  }
  const long long c1 = clock64();
  const uint64_t g1 = globaltimer();
  const uint32_t r = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
  if (r == 0x12345678u) sink[0] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    clk[0] = static_cast<unsigned long long>(c1 - c0);
    clk[1] = g1 - g0;
  }
}

}  // namespace

cudaError_t measure_lop3_peak(int sms, double* ops_per_s, double* sm_mhz) {
  const int blocks = sms * 8;  // 8 x 256 threads = 2048 threads/SM (full occupancy)
  const uint32_t iters = 1u << 14;
  uint32_t* sink = nullptr;
  unsigned long long* clk = nullptr;
  cudaEvent_t e0, e1;
  cudaError_t e = cudaMalloc(&sink, 4);
  if (e == cudaSuccess) e = cudaMalloc(&clk, 16);
  if (e != cudaSuccess) return e;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  lop3_peak_kernel<<<blocks, 256>>>(iters / 8, sink, clk);  // warm-up
  cudaEventRecord(e0);
  lop3_peak_kernel<<<blocks, 256>>>(iters, sink, clk);
  cudaEventRecord(e1);
  e = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
  const double ops = static_cast<double>(blocks) * 256.0 * iters * 64.0;
  *ops_per_s = ops / (ms * 1e-3);
  *sm_mhz = h[1] ? static_cast<double>(h[0]) / static_cast<double>(h[1]) * 1e3 : 0.0;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  cudaFree(clk);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace lc
