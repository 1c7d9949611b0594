// Sharded PCG: every rank holds only the part of A its own
// frame-pair edges (and, on rank 0, the correspondence sets) contribute; per
// PCG iteration each rank forms its partial A.p (k_matvec over its slots),
// ONE all-reduce of that n_vars vector gives every rank the bit-identical
// A.p, and the scalar recurrence of pcg_solve (solver.py:463-508) then runs
// redundantly on every rank in one thread block (n_vars <= ~12k): fixed-order
// block reductions for the dots, so all ranks take the same decisions without
// a scalar collective.  The restart iteration adds an A.x all-reduce.
//
// Device state (st[]): 0 rz, 1 norm_b, 2 alpha, 3 relative, 4 iterations,
// 5 status (1: non-finite), 6 done, 7 pending restart residual.
#include "sfb_kernels.cuh"

#define PCGS_THREADS 1024

// fixed-order block sum of NV values (every thread gets the totals)
template <int NV>
__device__ __forceinline__ void pcgs_sum(double (&v)[NV]) {
  __shared__ double sh[NV][PCGS_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double t = warp_sum(v[k]);
    if (lane == 0) sh[k][warp] = t;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double t = 0.0;
    for (int w = 0; w < PCGS_THREADS / 32; ++w) t += sh[k][w];
    v[k] = t;
  }
  __syncthreads();
}

// z_i = M^-1 r_i for all i of block row v (scalar or block Jacobi)
__device__ __forceinline__ void pcgs_precond(const PcgArgs& a, int n6) {
  for (int i = threadIdx.x; i < n6; i += blockDim.x) {
    if (a.bj_inv == nullptr) {
      a.z[i] = a.inv_diag[i] * a.r[i];
    } else {
      const int v = i / 6, row = i - 6 * v;
      const double* M = a.bj_inv + (int64_t)v * 36 + 6 * row;
      double z = 0.0;
#pragma unroll
      for (int c = 0; c < 6; ++c) z = fma(M[c], a.r[6 * v + c], z);
      a.z[i] = z;
    }
  }
}

// setup (solver.py:472-481): b = -g, x = 0, r = b, z = M^-1 r, p = z
__global__ void __launch_bounds__(PCGS_THREADS) k_pcgs_init(PcgArgs a, double* st) {
  const int n6 = 6 * a.n_blk;
  for (int i = threadIdx.x; i < n6; i += blockDim.x) {
    const double bi = -a.g[i];
    a.b[i] = bi;
    a.x[i] = 0.0;
    a.r[i] = bi;
    a.inv_diag[i] = 1.0 / fmax(a.jdiag[i], 1e-12);
  }
  __syncthreads();
  pcgs_precond(a, n6);
  __syncthreads();
  double v[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < n6; i += blockDim.x) {
    a.p[i] = a.z[i];
    v[0] += a.b[i] * a.b[i];
    v[1] += a.b[i] * a.z[i];
  }
  pcgs_sum<2>(v);
  if (threadIdx.x == 0) {
    const double norm_b = sqrt(v[0]);
    st[0] = v[1];
    st[1] = norm_b;
    st[2] = 0.0;
    st[3] = norm_b == 0.0 ? 0.0 : 1.0;
    st[4] = 0.0;
    st[5] = 0.0;
    st[6] = norm_b == 0.0 ? 1.0 : 0.0;
    st[7] = 0.0;
  }
}

// the rest of iteration k after r is known: z, r.r, r.z, convergence, beta, p
__device__ __forceinline__ void pcgs_finish(const PcgArgs& a, double* st, int n6, bool bad_x) {
  pcgs_precond(a, n6);
  __syncthreads();
  double v[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < n6; i += blockDim.x) {
    v[0] += a.r[i] * a.r[i];
    v[1] += a.r[i] * a.z[i];
  }
  pcgs_sum<2>(v);
  if (bad_x) {  // non-finite iterate -> PcgDivergenceError
    if (threadIdx.x == 0) { st[5] = 1.0; st[6] = 1.0; }
    return;
  }
  const double relative = sqrt(v[0]) / st[1];
  if (relative < a.tol) {
    if (threadIdx.x == 0) { st[3] = relative; st[6] = 1.0; }
    return;
  }
  const double beta = v[1] / st[0];
  for (int i = threadIdx.x; i < n6; i += blockDim.x) a.p[i] = fma(beta, a.p[i], a.z[i]);
  __syncthreads();
  if (threadIdx.x == 0) {
    st[0] = v[1];
    st[3] = relative;
  }
}

// iteration k after the all-reduce of q = A p (a.Ap): pAp, alpha, x, and on
// non-restart iterations r -= alpha q and the rest of the iteration
__global__ void __launch_bounds__(PCGS_THREADS) k_pcgs_step(PcgArgs a, double* st, int k, int restart) {
  if (st[6] != 0.0) return;  // done (grid-uniform: one block)
  const int n6 = 6 * a.n_blk;
  double v[1] = {0.0};
  for (int i = threadIdx.x; i < n6; i += blockDim.x) v[0] += a.p[i] * a.Ap[i];
  pcgs_sum<1>(v);
  const double pAp = v[0];
  if (threadIdx.x == 0) st[4] = (double)k;
  if (!isfinite(pAp)) {
    if (threadIdx.x == 0) { st[5] = 1.0; st[6] = 1.0; }
    return;
  }
  if (pAp <= 0.0) {  // singular direction: stop with the current iterate
    if (threadIdx.x == 0) st[6] = 1.0;
    return;
  }
  const double alpha = st[0] / pAp;
  double bad[1] = {0.0};
  for (int i = threadIdx.x; i < n6; i += blockDim.x) {
    const double xi = fma(alpha, a.p[i], a.x[i]);
    a.x[i] = xi;
    bad[0] += isfinite(xi) ? 0.0 : 1.0;
    if (!restart) a.r[i] = fma(-alpha, a.Ap[i], a.r[i]);
  }
  pcgs_sum<1>(bad);
  if (restart) {  // r = b - A x after the A.x all-reduce (k_pcgs_restart)
    if (threadIdx.x == 0) { st[2] = alpha; st[7] = bad[0]; }
    return;
  }
  pcgs_finish(a, st, n6, bad[0] != 0.0);
}

// restart iteration, after the all-reduce of q = A x: r = b - A x, then the
// rest of the iteration
__global__ void __launch_bounds__(PCGS_THREADS) k_pcgs_restart(PcgArgs a, double* st) {
  if (st[6] != 0.0) return;
  const int n6 = 6 * a.n_blk;
  for (int i = threadIdx.x; i < n6; i += blockDim.x) a.r[i] = a.b[i] - a.Ap[i];
  __syncthreads();
  pcgs_finish(a, st, n6, st[7] != 0.0);
}

void launch_pcgs_init(const PcgArgs& a, double* st, cudaStream_t s) {
  sfb_count_launch();
  k_pcgs_init<<<1, PCGS_THREADS, 0, s>>>(a, st);
}
void launch_pcgs_step(const PcgArgs& a, double* st, int k, int restart, cudaStream_t s) {
  sfb_count_launch();
  k_pcgs_step<<<1, PCGS_THREADS, 0, s>>>(a, st, k, restart);
}
void launch_pcgs_restart(const PcgArgs& a, double* st, cudaStream_t s) {
  sfb_count_launch();
  k_pcgs_restart<<<1, PCGS_THREADS, 0, s>>>(a, st);
}

// ---------------------------------------------------------------------------
// Partial-system exchange of the sharded mode: [g | jdiag | e_photo e_geo |
// (D when block-Jacobi)] packed into one vector before the all-reduce and
// unpacked after it.
__global__ void k_sys_pack(const double* g, const double* jdiag, const double* dscal,
                           const double* D, int n6, int with_d, double* out, int unpack,
                           double* g_o, double* jdiag_o, double* dscal_o, double* D_o) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int nD = with_d ? 6 * n6 : 0;
  const int n = 2 * n6 + 2 + nD;
  if (i >= n) return;
  if (!unpack) {
    double v;
    if (i < n6) v = g[i];
    else if (i < 2 * n6) v = jdiag[i - n6];
    else if (i < 2 * n6 + 2) v = dscal[1 + i - 2 * n6];
    else v = D[i - 2 * n6 - 2];
    out[i] = v;
  } else {
    const double v = out[i];
    if (i < n6) g_o[i] = v;
    else if (i < 2 * n6) jdiag_o[i - n6] = v;
    else if (i < 2 * n6 + 2) dscal_o[1 + i - 2 * n6] = v;
    else D_o[i - 2 * n6 - 2] = v;
  }
}

int sys_pack_len(int n6, int with_d) { return 2 * n6 + 2 + (with_d ? 6 * n6 : 0); }

void launch_sys_pack(double* g, double* jdiag, double* dscal, double* D, int n6, int with_d,
                     double* buf, int unpack, cudaStream_t s) {
  const int n = sys_pack_len(n6, with_d);
  sfb_count_launch();
  k_sys_pack<<<(n + 255) / 256, 256, 0, s>>>(g, jdiag, dscal, D, n6, with_d, buf, unpack, g, jdiag,
                                            dscal, D);
}
