// Latency of one grid-wide deterministic all-sum (G CTAs x 256 threads,
// co-resident) on the B200, per variant:
//  A  counter barrier: partial store, red.release.gpu, ld.acquire poll, then
//     warp 0 reads the G partials (the PCG's current scheme)
//  B  as A with relaxed polling and one acquire fence after the poll
//  C  flag-in-data: each CTA stores {value, epoch} as one 16-byte store after
//     a release fence into its own 256-byte-padded slot; warp 0 of every CTA
//     polls the G slots (relaxed) until every epoch matches, then one fence
//  D  as C, slots packed (16 B apart: hot lines)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsum_rate gridsum_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 2000
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void st128(double* p, double v, unsigned long long e) {
  asm volatile("{\n\t.reg .b128 t;\n\tmov.b128 t, {%1, %2};\n\tst.relaxed.gpu.global.b128 [%0], t;\n\t}" ::"l"(p), "l"(__double_as_longlong(v)), "l"(e) : "memory");
}
__device__ __forceinline__ void ld128(const double* p, unsigned long long& v, unsigned long long& e) {
  asm volatile("{\n\t.reg .b128 t;\n\tld.relaxed.gpu.global.b128 t, [%2];\n\tmov.b128 {%0, %1}, t;\n\t}" : "=l"(v), "=l"(e) : "l"(p) : "memory");
}
template <int V>
__global__ void __launch_bounds__(256, 1) k(unsigned* ctr, double* part, double* out, int pad) {
  const int G = gridDim.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __shared__ double sh[8];
  __shared__ double tot;
  double x = 1.0 + 1e-3 * blockIdx.x + 1e-6 * threadIdx.x;
  unsigned epoch = 0;
  for (int it = 0; it < ITERS; ++it) {
    double v = warp_sum(x);
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    ++epoch;
    if (V == 0 || V == 1) {
      if (threadIdx.x == 0) {
        double s = 0;
        for (int w = 0; w < 8; ++w) s += sh[w];
        __stcg(&part[(epoch & 1) * 256 + blockIdx.x], s);
        const unsigned target = epoch * G;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned c;
        if (V == 0) {
          do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(ctr) : "memory"); } while (c < target);
        } else {
          do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(ctr) : "memory"); } while (c < target);
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
      }
      __syncthreads();
      if (wid == 0) {
        double s = 0;
        for (int b = lane; b < G; b += 32) s += __ldcg(&part[(epoch & 1) * 256 + b]);
        s = warp_sum(s);
        if (lane == 0) tot = s;
      }
      __syncthreads();
    } else {
      const int stride = (V == 3) ? 2 : pad;  // doubles between slots
      if (threadIdx.x == 0) {
        double s = 0;
        for (int w = 0; w < 8; ++w) s += sh[w];
        double* slot = part + (size_t)(epoch & 1) * 256 * 32 + (size_t)blockIdx.x * stride;
        if (V == 2 || V == 3 || V == 5) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (V >= 4) st128(slot, s, epoch);
        else asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(slot), "l"(__double_as_longlong(s)), "l"((unsigned long long)epoch) : "memory");
      }
      if (wid == 0) {
        double s = 0;
        for (int b = lane; b < G; b += 32) {
          const double* slot = part + (size_t)(epoch & 1) * 256 * 32 + (size_t)b * stride;
          unsigned long long val, ep;
          do {
            if (V >= 4) ld128(slot, val, ep);
            else asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(val), "=l"(ep) : "l"(slot) : "memory");
          } while (ep != epoch);
          s += __longlong_as_double(val);
        }
        if (V == 2 || V == 3) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        s = warp_sum(s);
        if (lane == 0) tot = s;
      }
      __syncthreads();
    }
    x = x * 0.999 + tot * 1e-9;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = x;
}
int main() {
  unsigned* ctr; double* part; double* out;
  cudaMalloc(&ctr, 4); cudaMalloc(&part, 2 * 256 * 32 * 8); cudaMalloc(&out, 256 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* nm[6] = {"A counter+acquire poll", "B counter+relaxed poll", "C flag-in-data padded", "D flag-in-data packed", "E flag b128 no fences", "F flag b128 writer fence"};
  int Gs[3] = {16, 63, 148};
  for (int gi = 0; gi < 3; ++gi)
    for (int v = 0; v < 6; ++v) {
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(ctr, 0, 4); cudaMemset(part, 0, 2 * 256 * 32 * 8);
        cudaEventRecord(a);
        if (v == 0) k<0><<<Gs[gi], 256>>>(ctr, part, out, 32);
        if (v == 1) k<1><<<Gs[gi], 256>>>(ctr, part, out, 32);
        if (v == 2) k<2><<<Gs[gi], 256>>>(ctr, part, out, 32);
        if (v == 3) k<3><<<Gs[gi], 256>>>(ctr, part, out, 32);
        if (v == 4) k<4><<<Gs[gi], 256>>>(ctr, part, out, 32);
        if (v == 5) k<5><<<Gs[gi], 256>>>(ctr, part, out, 32);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("G=%3d %-28s %.3f us per all-sum (%s)\n", Gs[gi], nm[v], best * 1e3 / ITERS, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
