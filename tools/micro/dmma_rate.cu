// Microbenchmark: FP64 tensor (DMMA m8n8k4) vs FP64 FMA throughput on B200,
// and whether they overlap (separate pipes).  nvcc -arch=sm_100a -O3 dmma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>  // 0: DMMA only, 1: DFMA only, 2: both interleaved
__global__ void k(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, b0 = 1.0 + threadIdx.x * 1e-4;
  double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double f[16];
  for (int i = 0; i < 16; ++i) f[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[2 * q]), "+d"(c[2 * q + 1]) : "d"(a0), "d"(b0));
    }
    if (MODE != 0) {
#pragma unroll
      for (int q = 0; q < 16; ++q) f[q] = fma(f[q], b0, a0);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  for (int i = 0; i < 16; ++i) s += f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 8);
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps = 8; warps <= 32; warps *= 2) {
    for (int mode = 0; mode < 3; ++mode) {
      auto fn = mode == 0 ? k<0> : (mode == 1 ? k<1> : k<2>);
      fn<<<sm, 32 * warps>>>(out, 16);
      cudaEventRecord(e0);
      fn<<<sm, 32 * warps>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double n_dmma = mode != 1 ? 4.0 * iters * warps * sm : 0;
      const double n_dfma = mode != 0 ? 16.0 * iters * warps * sm * 32 : 0;
      printf("warps/SM %2d mode %d: %.3f ms  DMMA %.1f TFLOP/s  DFMA %.1f TFLOP/s\n", warps, mode, ms,
             n_dmma * 512 / (ms * 1e-3) / 1e12, n_dfma * 2 / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
