// Throughput of float->double conversion on the B200: F2F.F64.F32 (cvt.f64.f32)
// vs an integer bit-construction, vs DFMA.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 4096
__device__ __forceinline__ double f2d_int(float f) {
  const uint32_t b = __float_as_uint(f);
  const uint32_t m = b & 0x7fffffffu;
  uint32_t hi = (m >> 3) + (896u << 20);
  hi = m == 0u ? 0u : hi;
  hi |= b & 0x80000000u;
  return __hiloint2double((int)hi, (int)(b << 29));
}
template <int MODE>
__global__ void k(const float* in, double* out) {
  float f[8];
  for (int i = 0; i < 8; ++i) f[i] = in[(threadIdx.x + i) & 255];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) acc[i] += (double)f[i];          // F2F + DADD
      if (MODE == 1) acc[i] += f2d_int(f[i]);         // INT + DADD
      if (MODE == 2) acc[i] = fma(acc[i], 1.0000001, 0.5);  // DFMA only
      f[i] = __uint_as_float(__float_as_uint(f[i]) ^ 1u);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* in; double* out;
  cudaMalloc(&in, 256 * 4); cudaMalloc(&out, 148 * 8 * 1024 * 8);
  float h[256]; for (int i = 0; i < 256; ++i) h[i] = 0.001f * i;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[3] = {"F2F+DADD", "INT+DADD", "DFMA"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<148 * 8, 256>>>(in, out);
      if (mode == 1) k<1><<<148 * 8, 256>>>(in, out);
      if (mode == 2) k<2><<<148 * 8, 256>>>(in, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double ops = 148.0 * 8 * 256 * ITERS * 8;
      if (rep) printf("%s: %.3f ms, %.1f G elem/s, %.2f elem/clk/SM at 1.965 GHz\n", names[mode], ms, ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
