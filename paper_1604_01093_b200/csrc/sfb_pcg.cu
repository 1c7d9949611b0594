// Block-sparse normal equations: matvec and the persistent scalar-Jacobi PCG.
//
// The system is stored as 6x6 blocks: one diagonal block per variable frame
// and one off-diagonal block per frame pair that shares a correspondence set
// or a dense edge.  NormalEquations.apply (solver.py:403-410) is then a block
// row product; pcg_solve (solver.py:463-508) runs as ONE cooperative kernel
// whose blocks all compute the same scalars from the same fixed-order
// partial sums, so control flow (breaks, restarts) is grid-uniform and
// bit-reproducible.
#include <cooperative_groups.h>

#include "sfb_kernels.cuh"

namespace cg = cooperative_groups;

#define PCG_THREADS 256
#define PCG_WARPS (PCG_THREADS / 32)

// y_v = D_v x_v + sum_w B_vw x_w for one block row, computed by one warp:
// lanes are 5 groups of 6 (lane = 6*group + row); each group walks every 5th
// neighbour block, each lane one row of it; groups are summed in fixed order.
// Returns y_v[row] in lanes 0..5 (other lanes undefined).
__device__ __forceinline__ double block_row(const PcgArgs& a, int v, const double* __restrict__ xin,
                                            int lane) {
  const int grp = lane / 6, row = lane - 6 * (lane / 6);
  double acc = 0.0;
  if (grp < 5) {
    if (grp == 0) {
      const double* Dm = a.D + (int64_t)v * 36 + row * 6;
      const double* xv = xin + 6 * v;
#pragma unroll
      for (int c = 0; c < 6; ++c) acc = fma(Dm[c], xv[c], acc);
    }
    for (int e = a.row_ptr[v] + grp; e < a.row_ptr[v + 1]; e += 5) {
      const int ent = a.row_ent[e];
      const double* Bm = a.B + (int64_t)(ent >> 1) * 36;
      const double* xw = xin + 6 * a.row_col[e];
      if (ent & 1) {
#pragma unroll
        for (int c = 0; c < 6; ++c) acc = fma(Bm[c * 6 + row], xw[c], acc);
      } else {
#pragma unroll
        for (int c = 0; c < 6; ++c) acc = fma(Bm[row * 6 + c], xw[c], acc);
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int g = 0; g < 5; ++g) s += __shfl_sync(0xffffffffu, acc, 6 * g + (lane % 6));
  return s;
}

__global__ void k_matvec(PcgArgs a, const double* xin, double* yout) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= a.n_blk) return;
  const double y = block_row(a, warp, xin, lane);
  if (lane < 6) yout[6 * warp + lane] = y;
}

void launch_matvec(const PcgArgs& a, const double* xin, double* yout, cudaStream_t s) {
  if (a.n_blk <= 0) return;
  sfb_count_launch();
  k_matvec<<<(a.n_blk * 32 + 255) / 256, 256, 0, s>>>(a, xin, yout);
}

// Deterministic block sum of NV values; every thread of the block gets them.
template <int NV>
__device__ __forceinline__ void block_allsum(double (&v)[NV], double (*sh)[PCG_WARPS]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double s = warp_sum(v[k]);
    if (lane == 0) sh[k][warp] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < PCG_WARPS; ++w) s += sh[k][w];
    v[k] = s;
  }
  __syncthreads();
}

// Every block sums the per-block partials part[k*G + b] in the same fixed order.
template <int NV>
__device__ __forceinline__ void grid_allsum(const double* part, double (&out)[NV], int G) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
    for (int b = lane; b < G; b += 32) s += __ldcg(&part[k * G + b]);
    out[k] = warp_sum(s);
  }
}

// Matvec policies: the block-sparse normal equations, or a dense padded
// matrix (pcg_solve on a duck-typed system, solver.py:463-508).
struct BsrMv {
  __device__ __forceinline__ double row(const PcgArgs& a, int v, const double* x, int lane) const {
    return block_row(a, v, x, lane);
  }
};

struct DenseMv {
  const double* A;  // (6 n_blk)^2 row-major, zero padded
  __device__ __forceinline__ double row(const PcgArgs& a, int v, const double* x, int lane) const {
    const int n6 = 6 * a.n_blk;
    double out = 0.0;
    for (int r = 0; r < 6; ++r) {
      const double* Ar = A + (int64_t)(6 * v + r) * n6;
      double s = 0.0;
      for (int c = lane; c < n6; c += 32) s = fma(Ar[c], x[c], s);
      s = warp_sum(s);
      if (lane == r) out = s;
    }
    return out;
  }
};

template <class Mv>
__global__ void __launch_bounds__(PCG_THREADS) k_pcg(PcgArgs a, Mv mv) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[4][PCG_WARPS];
  const int G = gridDim.x;
  const int n = 6 * a.n_blk;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nthreads = G * blockDim.x;
  const int lane = threadIdx.x & 31, warp_in_blk = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * PCG_WARPS + warp_in_blk, nwarps = G * PCG_WARPS;
  if (a.skip && *a.skip != 0.0) return;  // grid-uniform

  // ---- setup: b = -g, x = 0, inv_diag, r = b, z = M^-1 r, p = z (solver.py:472-481)
  {
    double v[2] = {0.0, 0.0};
    for (int i = tid; i < n; i += nthreads) {
      const double bi = -a.g[i];
      const double di = a.jdiag[i];
      const double inv = 1.0 / fmax(di, 1e-12);
      const double zi = inv * bi;
      a.b[i] = bi;
      a.x[i] = 0.0;
      a.inv_diag[i] = inv;
      a.r[i] = bi;
      a.z[i] = zi;
      a.p[i] = zi;
      v[0] += bi * bi;
      v[1] += bi * zi;
    }
    block_allsum<2>(v, sh);
    if (threadIdx.x == 0) { a.part[0 * G + blockIdx.x] = v[0]; a.part[1 * G + blockIdx.x] = v[1]; }
  }
  grid.sync();
  double tot[2];
  grid_allsum<2>(a.part, tot, G);
  const double norm_b = sqrt(tot[0]);
  double rz = tot[1];
  int iterations = 0;
  double relative = 1.0;
  int status = 0;
  if (norm_b == 0.0) {
    relative = 0.0;
  } else {
    for (int k = 1; k <= a.max_it; ++k) {
      iterations = k;
      grid.sync();  // p complete; everyone is done reading last iteration's partials
      // ---- Ap = A p, partial p.Ap (block rows -> warps)
      {
        double v[1] = {0.0};
        for (int row = gwarp; row < a.n_blk; row += nwarps) {
          const double y = mv.row(a, row, a.p, lane);
          double pa = 0.0;
          if (lane < 6) {
            a.Ap[6 * row + lane] = y;
            pa = a.p[6 * row + lane] * y;
          }
          // fixed-order sum over the 6 rows of the block
          double t = 0.0;
#pragma unroll
          for (int c = 0; c < 6; ++c) t += __shfl_sync(0xffffffffu, pa, c);
          if (lane == 0) v[0] += t;
        }
        block_allsum<1>(v, sh);
        if (threadIdx.x == 0) a.part[blockIdx.x] = v[0];
      }
      grid.sync();
      double pAp_a[1];
      grid_allsum<1>(a.part, pAp_a, G);
      const double pAp = pAp_a[0];
      if (!isfinite(pAp)) { status = 1; break; }  // PcgDivergenceError
      if (pAp <= 0.0) break;                       // singular direction
      const double alpha = rz / pAp;
      const bool restart = (k % a.restart) == 0;
      double* pr = a.part + G;  // r-phase partials live apart from the p.Ap ones
      // ---- x += alpha p ; r -= alpha Ap (or r = b - A x after a sync)
      if (!restart) {
        double v[3] = {0.0, 0.0, 0.0};
        for (int i = tid; i < n; i += nthreads) {
          const double xi = a.x[i] + alpha * a.p[i];
          const double ri = a.r[i] - alpha * a.Ap[i];
          const double zi = a.inv_diag[i] * ri;
          a.x[i] = xi;
          a.r[i] = ri;
          a.z[i] = zi;
          v[0] += ri * ri;
          v[1] += ri * zi;
          v[2] += isfinite(xi) ? 0.0 : 1.0;
        }
        block_allsum<3>(v, sh);
        if (threadIdx.x == 0)
          for (int q = 0; q < 3; ++q) pr[q * G + blockIdx.x] = v[q];
      } else {
        double v[1] = {0.0};
        for (int i = tid; i < n; i += nthreads) {
          const double xi = a.x[i] + alpha * a.p[i];
          a.x[i] = xi;
          v[0] += isfinite(xi) ? 0.0 : 1.0;
        }
        block_allsum<1>(v, sh);
        if (threadIdx.x == 0) pr[2 * G + blockIdx.x] = v[0];
        grid.sync();
        for (int row = gwarp; row < a.n_blk; row += nwarps) {
          const double y = mv.row(a, row, a.x, lane);
          if (lane < 6) a.r[6 * row + lane] = a.b[6 * row + lane] - y;
        }
        grid.sync();
        double w[2] = {0.0, 0.0};
        for (int i = tid; i < n; i += nthreads) {
          const double ri = a.r[i];
          const double zi = a.inv_diag[i] * ri;
          a.z[i] = zi;
          w[0] += ri * ri;
          w[1] += ri * zi;
        }
        block_allsum<2>(w, sh);
        if (threadIdx.x == 0) { pr[0 * G + blockIdx.x] = w[0]; pr[1 * G + blockIdx.x] = w[1]; }
      }
      grid.sync();
      double s3[3];
      grid_allsum<3>(pr, s3, G);
      if (s3[2] != 0.0) { status = 1; break; }  // non-finite iterate
      relative = sqrt(s3[0]) / norm_b;
      if (relative < a.tol) break;
      const double rz_new = s3[1];
      const double beta = rz_new / rz;
      rz = rz_new;
      for (int i = tid; i < n; i += nthreads) a.p[i] = a.z[i] + beta * a.p[i];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out_scalars[0] = (double)iterations;
    a.out_scalars[1] = relative;
    a.out_scalars[2] = (double)status;
  }
}

template <class Mv>
static cudaError_t launch_pcg_t(const PcgArgs& a, Mv mv, int n_sm, cudaStream_t s) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg<Mv>, PCG_THREADS, 0);
  if (e != cudaSuccess) return e;
  int want = (a.n_blk + PCG_WARPS - 1) / PCG_WARPS;
  const int cap = n_sm * (per_sm < 1 ? 1 : per_sm);
  if (want > n_sm) want = n_sm;  // one CTA per SM at most: cheapest grid barrier
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  PcgArgs args = a;
  Mv m = mv;
  void* params[] = {&args, &m};
  sfb_count_launch();
  return cudaLaunchCooperativeKernel((void*)k_pcg<Mv>, dim3(want), dim3(PCG_THREADS), params, 0, s);
}

cudaError_t launch_pcg(const PcgArgs& a, int n_sm, cudaStream_t s) {
  return launch_pcg_t(a, BsrMv{}, n_sm, s);
}

cudaError_t launch_pcg_dense(const PcgArgs& a, const double* A, int n_sm, cudaStream_t s) {
  return launch_pcg_t(a, DenseMv{A}, n_sm, s);
}
