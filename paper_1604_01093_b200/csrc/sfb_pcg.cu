// Block-sparse normal equations: matvec and the persistent scalar-Jacobi PCG.
//
// The system is stored per block row as contiguous, pre-oriented 6x6 slot
// blocks (diagonal first, then one per coupled frame).  NormalEquations.apply
// (solver.py:403-410) is one pass over the slots; pcg_solve (solver.py:463-508)
// is ONE cooperative kernel:
//  * each CTA owns a contiguous range of block rows (one warp per row) and
//    stages that range's slot blocks in shared memory once per solve - the
//    matrix is constant across PCG iterations;
//  * per iteration a warp gathers the (6-vector) neighbour inputs of its row
//    into shared memory with all loads in flight at once, then multiplies
//    from shared memory;
//  * p = z + beta p is folded into the next matvec (neighbours form it on the
//    fly, the owner stores it in a ping-pong buffer): two grid barriers per
//    iteration, three on restart iterations;
//  * every CTA sums the per-CTA partials in the same order, so all scalars,
//    breaks and restarts are grid-uniform and bit-reproducible.
#include "sfb_kernels.cuh"
#include <type_traits>

#define PCG_THREADS 256
#define PCG_WARPS (PCG_THREADS / 32)
#define PCG_GATHER_CAP 80                    // neighbour slots gathered per pass
#define PCG_SMEM_BYTES (200 * 1024)          // dynamic smem request
#define PCG_GATHER_BYTES (PCG_WARPS * PCG_GATHER_CAP * 6 * 8)

// Grid-wide barrier for a co-resident (cooperative) grid: one arrival counter
// in global memory, zeroed before launch; thread 0 of each CTA releases the
// CTA's writes, arrives, spins on a relaxed load and acquires.
struct GridBarrier {
  unsigned* ctr;
  unsigned epoch;
  __device__ __forceinline__ void sync(unsigned G) {
    __syncthreads();  // the CTA's writes happen-before thread 0's release below
    if (threadIdx.x == 0) {
      ++epoch;
      const unsigned target = epoch * G;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      } while (v < target);
    }
    __syncthreads();
  }
  // Barrier + all-sum of the G per-CTA partials in one step, for a CTA that
  // has just run block_allsum (whose barrier already ordered every thread's
  // writes before thread 0's release): warp 0 alone arrives, polls and reads
  // the partials (grid_allsum_warp's fixed order); one CTA barrier after.
  template <int NV>
  __device__ __forceinline__ void sync_allsum(const double* part, double (&out)[NV], unsigned G);
};

// Per-CTA view of the block rows it owns.
struct RowCtx {
  int r0, r1;          // owned rows [r0, r1)
  int s0;              // first slot of r0
  const double* Bs;    // staged slot blocks (shared) or null: slots [s0, s_end)
  const int* cols;     // column block per global slot (shared for staged slots)
  int s_end;           // end of the staged slots (the rest read from global memory)
  double* gbuf;        // this warp's gather buffer (shared), PCG_GATHER_CAP x 6
};

// y = (row v of A) . xin, xin = FOLD ? z + beta*pold : pold.  Lanes 6g+r
// (g < 5) walk slots g, g+5, ... of the current gather chunk; lanes 0..5
// return y[r].
template <bool FOLD>
__device__ __forceinline__ double row_product(const PcgArgs& a, const RowCtx& rc, int v,
                                              const double* __restrict__ z,
                                              const double* __restrict__ pold, double beta,
                                              int lane, int part = 0, int nparts = 1,
                                              int pe0 = -1, int pe1 = -1) {
  const int grp = lane / 6, r = lane - 6 * grp;
  int e0 = pe0, e1 = pe1;  // the warp's slot range when the caller holds it
  if (pe0 < 0) {
    e0 = a.row_ptr[v];
    e1 = a.row_ptr[v + 1];
    if (nparts > 1) {  // this warp's share of the row's slots (split rows)
      const int n = e1 - e0;
      e1 = e0 + (n * (part + 1)) / nparts;
      e0 = e0 + (n * part) / nparts;
    }
  }
  double acc = 0.0;
  for (int c0 = e0; c0 < e1; c0 += PCG_GATHER_CAP) {
    const int c1 = min(e1, c0 + PCG_GATHER_CAP);
    // gather the chunk's neighbour vectors: the (up to three) slots of each
    // lane are loaded before any is stored, so the chunk costs one L2 round trip
    static_assert(PCG_GATHER_CAP <= 96, "gather unroll covers 3 slots per lane");
    double2 xa[3], xb[3], xc[3];
    const int ka = c0 + lane, kb = ka + 32, kc = ka + 64;
    const bool va = ka < c1, vb = kb < c1, vc = kc < c1;
    auto col = [&](int k) { return k < rc.s_end ? rc.cols[k] : a.row_col[k]; };
    const int wa = va ? col(ka) : 0, wb = vb ? col(kb) : 0, wc = vc ? col(kc) : 0;
#pragma unroll
    for (int h = 0; h < 3; ++h) {
      xa[h] = va ? __ldcg(reinterpret_cast<const double2*>(pold + 6 * wa) + h) : make_double2(0, 0);
      xb[h] = vb ? __ldcg(reinterpret_cast<const double2*>(pold + 6 * wb) + h) : make_double2(0, 0);
      xc[h] = vc ? __ldcg(reinterpret_cast<const double2*>(pold + 6 * wc) + h) : make_double2(0, 0);
    }
    if (FOLD) {
#pragma unroll
      for (int h = 0; h < 3; ++h) {
        const double2 za = va ? __ldcg(reinterpret_cast<const double2*>(z + 6 * wa) + h) : make_double2(0, 0);
        const double2 zb = vb ? __ldcg(reinterpret_cast<const double2*>(z + 6 * wb) + h) : make_double2(0, 0);
        const double2 zc = vc ? __ldcg(reinterpret_cast<const double2*>(z + 6 * wc) + h) : make_double2(0, 0);
        xa[h].x = fma(beta, xa[h].x, za.x); xa[h].y = fma(beta, xa[h].y, za.y);
        xb[h].x = fma(beta, xb[h].x, zb.x); xb[h].y = fma(beta, xb[h].y, zb.y);
        xc[h].x = fma(beta, xc[h].x, zc.x); xc[h].y = fma(beta, xc[h].y, zc.y);
      }
    }
    double2* gb = reinterpret_cast<double2*>(rc.gbuf);
#pragma unroll
    for (int h = 0; h < 3; ++h) {
      if (va) gb[3 * (ka - c0) + h] = xa[h];
      if (vb) gb[3 * (kb - c0) + h] = xb[h];
      if (vc) gb[3 * (kc - c0) + h] = xc[h];
    }
    __syncwarp();
    if (grp < 5) {
      // six independent FMA chains (one per column) instead of one 6x longer chain
      double ac[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      for (int k = c0 + grp; k < c1; k += 5) {
        const double* Bm = k < rc.s_end ? rc.Bs + (int64_t)(k - rc.s0) * 36 + r * 6
                                        : a.Brow + (int64_t)k * 36 + r * 6;
        const double* xv = rc.gbuf + 6 * (k - c0);
#pragma unroll
        for (int c = 0; c < 6; ++c) ac[c] = fma(Bm[c], xv[c], ac[c]);
      }
      acc += ((ac[0] + ac[1]) + (ac[2] + ac[3])) + (ac[4] + ac[5]);
    }
    __syncwarp();
  }
  double s = 0.0;
  const int rr = lane % 6;
#pragma unroll
  for (int g = 0; g < 5; ++g) s += __shfl_sync(0xffffffffu, acc, 6 * g + rr);
  return s;
}

// Plain matvec (NormalEquations.apply): one warp per row, no staging.
__global__ void k_matvec(PcgArgs a, const double* xin, double* yout) {
  __shared__ double gb[PCG_WARPS][PCG_GATHER_CAP * 6];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= a.n_blk) return;
  RowCtx rc{0, 0, 0, nullptr, a.row_col, 0, gb[threadIdx.x >> 5]};
  const double y = row_product<false>(a, rc, warp, nullptr, xin, 0.0, lane);
  if (lane < 6) yout[6 * warp + lane] = y;
}

void launch_matvec(const PcgArgs& a, const double* xin, double* yout, cudaStream_t s) {
  if (a.n_blk <= 0) return;
  sfb_count_launch();
  k_matvec<<<(a.n_blk * 32 + 255) / 256, 256, 0, s>>>(a, xin, yout);
}

// Deterministic block sum of NV per-warp values (lane 0 holds them); thread 0
// receives the totals (it alone publishes them).  `sh` is next rewritten only
// after the grid barrier that follows every call, which synchronises the CTA.
template <int NV>
__device__ __forceinline__ void block_allsum(double (&v)[NV], double (*sh)[PCG_WARPS]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) sh[k][warp] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < PCG_WARPS; ++w) s += sh[k][w];
      v[k] = s;
    }
  }
}

// Every CTA sums the per-CTA partials part[k*G + b] in the same order.
template <int NV>
__device__ __forceinline__ void grid_allsum_warp(const double* part, double (&out)[NV], int G);
#ifndef PCG_W0SUM
#define PCG_W0SUM 1
#endif
template <int NV>
__device__ __forceinline__ void grid_allsum(const double* part, double (&out)[NV], int G) {
#if PCG_W0SUM
  // warp 0 alone reads the G partials (L2 round trip) and shares the totals:
  // every warp reading them made 8x the requests on the same hot lines
  __shared__ double tot_sh[4];
  if (threadIdx.x < 32) {
    double t[NV];
    grid_allsum_warp<NV>(part, t, G);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) tot_sh[k] = t[k];
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = tot_sh[k];
#else
  grid_allsum_warp<NV>(part, out, G);
#endif
}

template <int NV>
__device__ __forceinline__ void grid_allsum_warp(const double* part, double (&out)[NV], int G) {
  // all NV x ceil(G/32) loads are issued before any is consumed (one L2
  // round trip); then a fixed-order per-lane sum and butterfly
  const int lane = threadIdx.x & 31;
  constexpr int MAXC = 8;  // G <= 256
  double v[NV][MAXC];
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int b = lane + 32 * c;
      v[k][c] = b < G ? __ldcg(&part[k * G + b]) : 0.0;
    }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) s += v[k][c];
    out[k] = warp_sum(s);
  }
}

template <int NV>
__device__ __forceinline__ void GridBarrier::sync_allsum(const double* part, double (&out)[NV],
                                                         unsigned G) {
  __shared__ double tot_w0[4];
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      ++epoch;
      const unsigned target = epoch * G;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      } while (v < target);
    }
    __syncwarp();  // lane 0's acquire orders the warp's partial loads below
    double t[NV];
    grid_allsum_warp<NV>(part, t, (int)G);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) tot_w0[k] = t[k];
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = tot_w0[k];
}

// z = M^-1 r for one block row: scalar Jacobi (the reference's pcg_solve,
// solver.py:477) or, opt-in, block Jacobi with the row's inverted 6x6
// diagonal block (k_block_jacobi_inv).  Called by the whole warp (r in lanes
// 0..5, grid-uniform branch); lanes 0..5 get their z.
__device__ __forceinline__ double precond(const PcgArgs& a, int row, double ri, double inv, int lane) {
  if (a.bj_inv == nullptr) return inv * ri;
  const double* M = a.bj_inv + (int64_t)row * 36 + 6 * (lane % 6);
  double z = 0.0;
#pragma unroll
  for (int c = 0; c < 6; ++c) z = fma(__ldg(M + c), __shfl_sync(0xffffffffu, ri, c), z);
  return z;
}

// fixed-order sum of lanes 0..5 (one row value each), result in all lanes
__device__ __forceinline__ double sum6(double v) {
  double t = 0.0;
#pragma unroll
  for (int c = 0; c < 6; ++c) t += __shfl_sync(0xffffffffu, v, c);
  return t;
}

// Matvec policies: block-row slots, or a dense padded matrix (pcg_solve on a
// duck-typed system, solver.py:463-508).
struct BsrMv {
  template <bool FOLD>
  __device__ __forceinline__ double row(const PcgArgs& a, const RowCtx& rc, int v, const double* z,
                                        const double* pold, double beta, int lane, int part = 0,
                                        int nparts = 1, int e0 = -1, int e1 = -1) const {
    return row_product<FOLD>(a, rc, v, z, pold, beta, lane, part, nparts, e0, e1);
  }
  __device__ __forceinline__ bool stageable() const { return true; }
  static constexpr bool kSplit = true;  // rows may be split over warps
};

struct DenseMv {
  const double* A;  // (6 n_blk)^2 row-major, zero padded
  template <bool FOLD>
  __device__ __forceinline__ double row(const PcgArgs& a, const RowCtx&, int v, const double* z,
                                        const double* pold, double beta, int lane, int = 0,
                                        int = 1, int = -1, int = -1) const {
    const int n6 = 6 * a.n_blk;
    double out = 0.0;
    for (int r = 0; r < 6; ++r) {
      const double* Ar = A + (int64_t)(6 * v + r) * n6;
      double s = 0.0;
      for (int c = lane; c < n6; c += 32) {
        const double xc = FOLD ? fma(beta, __ldcg(pold + c), __ldcg(z + c)) : __ldcg(pold + c);
        s = fma(Ar[c], xc, s);
      }
      s = warp_sum(s);
      if (lane == r) out = s;
    }
    return out;
  }
  __device__ __forceinline__ bool stageable() const { return false; }
  static constexpr bool kSplit = false;
};

#ifdef PCG_TRACE
// tuning builds only (-DPCG_TRACE): CTA 0 stamps %globaltimer at the phase
// boundaries of the first 64 iterations; read with sfb_debug_pcg_trace.
__device__ unsigned long long g_pcg_trace[64 * 8];
__device__ __forceinline__ void trace_mark(int k, int ph) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && k < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_pcg_trace[k * 8 + ph] = t;
  }
}
extern "C" int sfb_debug_pcg_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_pcg_trace, sizeof(g_pcg_trace));
}
#define TRACE(k, ph) trace_mark(k, ph)
#else
#define TRACE(k, ph)
#endif

template <class Mv>
__global__ void __launch_bounds__(PCG_THREADS, 1) k_pcg(PcgArgs a, Mv mv, int rows_per_cta) {
  extern __shared__ __align__(16) double smem[];
  GridBarrier grid{reinterpret_cast<unsigned*>(a.flags), 0u};
  __shared__ double sh[4][PCG_WARPS];
  const int G = gridDim.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool own = lane < 6;
  if (a.skip && *a.skip != 0.0) return;  // grid-uniform
  RowCtx rc;
  rc.r0 = min(a.n_blk, blockIdx.x * rows_per_cta);
  rc.r1 = min(a.n_blk, rc.r0 + rows_per_cta);
  rc.s0 = 0;
  rc.Bs = nullptr;
  rc.cols = a.row_col;
  rc.gbuf = smem + wid * PCG_GATHER_CAP * 6;
  rc.s_end = 0;
  if (mv.stageable() && rc.r1 > rc.r0) {
    // the matrix (and its column indices) is constant during the solve: stage
    // this CTA's slot blocks in shared memory once - as many as fit (cfg5's
    // 37 MB exceed the SMs' shared memory; the remaining slots are read from L2)
    rc.s0 = a.row_ptr[rc.r0];
    const int64_t cap = ((int64_t)PCG_SMEM_BYTES - (int64_t)PCG_GATHER_BYTES) / (36 * 8 + 4);
    const int64_t ns = min((int64_t)(a.row_ptr[rc.r1] - rc.s0), cap);
    const int64_t n = ns * 36;
    double* dst = smem + PCG_WARPS * PCG_GATHER_CAP * 6;
    const double* src = a.Brow + (int64_t)rc.s0 * 36;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    int* cdst = reinterpret_cast<int*>(dst + n);
    for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) cdst[i] = a.row_col[rc.s0 + i];
    rc.Bs = dst;
    rc.cols = cdst - rc.s0;  // indexed by global slot
    rc.s_end = rc.s0 + (int)ns;
  }
  __syncthreads();
  double* pa = a.p;   // p of the previous iteration (read by neighbours)
  double* pb = a.p2;  // p of this iteration (written by owners)
  double* partA = a.part;          // G   : p.Ap
  double* partB = a.part + G;      // 3G  : r.r, r.z, non-finite(x)

  // ---- setup (solver.py:472-481), owner rows
  {
    double v[2] = {0.0, 0.0};
    for (int row = rc.r0 + wid; row < rc.r1; row += PCG_WARPS) {
      double bb = 0.0, bz = 0.0;
      const int i = 6 * row + (own ? lane : 0);
      const double bi = own ? -a.g[i] : 0.0;
      const double inv = own ? 1.0 / fmax(a.jdiag[i], 1e-12) : 0.0;
      const double zi = precond(a, row, bi, inv, lane);
      if (own) {
        a.b[i] = bi;
        a.x[i] = 0.0;
        a.inv_diag[i] = inv;
        a.r[i] = bi;
        a.z[i] = zi;
        pa[i] = zi;
        bb = bi * bi;
        bz = bi * zi;
      }
      v[0] += sum6(bb);
      v[1] += sum6(bz);
    }
    block_allsum<2>(v, sh);
    if (threadIdx.x == 0) { partB[blockIdx.x] = v[0]; partB[G + blockIdx.x] = v[1]; }
  }
  grid.sync(G);
  double tot[2];
  grid_allsum<2>(partB, tot, G);
  const double norm_b = sqrt(tot[0]);
  double rz = tot[1];
  int iterations = 0;
  double relative = 1.0;
  int status = 0;
  double beta = 0.0;
  bool fold = false;  // first iteration: p = z already in pa
  if (norm_b == 0.0) {
    relative = 0.0;
  } else {
    for (int k = 1; k <= a.max_it; ++k) {
      iterations = k;
      TRACE(k, 0);
      // ---- Ap = A p with p = z + beta pold formed on the fly; owners store p
      {
        double v[1] = {0.0};
        for (int row = rc.r0 + wid; row < rc.r1; row += PCG_WARPS) {
          const double y = fold ? mv.template row<true>(a, rc, row, a.z, pa, beta, lane)
                                : mv.template row<false>(a, rc, row, a.z, pa, beta, lane);
          double pAp = 0.0;
          if (own) {
            const int i = 6 * row + lane;
            const double pi = fold ? fma(beta, __ldcg(pa + i), __ldcg(a.z + i)) : __ldcg(pa + i);
            pb[i] = pi;
            a.Ap[i] = y;
            pAp = pi * y;
          }
          v[0] += sum6(pAp);
        }
        TRACE(k, 1);
        block_allsum<1>(v, sh);
        if (threadIdx.x == 0) partA[blockIdx.x] = v[0];
      }
      grid.sync(G);
      double pAp_a[1];
      grid_allsum<1>(partA, pAp_a, G);
      TRACE(k, 2);
      const double pAp = pAp_a[0];
      if (!isfinite(pAp)) { status = 1; break; }  // PcgDivergenceError
      if (pAp <= 0.0) break;                       // singular direction
      const double alpha = rz / pAp;
      const bool restart = (k % a.restart) == 0;
      // ---- x += alpha p ; r -= alpha Ap (or r = b - A x) ; z = M^-1 r
      {
        double v[3] = {0.0, 0.0, 0.0};
        for (int row = rc.r0 + wid; row < rc.r1; row += PCG_WARPS) {
          double rr = 0.0, rzv = 0.0, bad = 0.0;
          if (own) {
            const int i = 6 * row + lane;
            const double xi = fma(alpha, pb[i], a.x[i]);
            a.x[i] = xi;
            bad = isfinite(xi) ? 0.0 : 1.0;
          }
          if (!restart) {
            const int i = 6 * row + (own ? lane : 0);
            const double ri = own ? fma(-alpha, a.Ap[i], a.r[i]) : 0.0;
            const double zi = precond(a, row, ri, own ? a.inv_diag[i] : 0.0, lane);
            if (own) {
              a.r[i] = ri;
              a.z[i] = zi;
              rr = ri * ri;
              rzv = ri * zi;
            }
          }
          v[0] += sum6(rr);
          v[1] += sum6(rzv);
          v[2] += sum6(bad);
        }
        if (restart) {
          grid.sync(G);  // x complete
          for (int row = rc.r0 + wid; row < rc.r1; row += PCG_WARPS) {
            const double y = mv.template row<false>(a, rc, row, nullptr, a.x, 0.0, lane);
            double rr = 0.0, rzv = 0.0;
            const int i = 6 * row + (own ? lane : 0);
            const double ri = own ? a.b[i] - y : 0.0;
            const double zi = precond(a, row, ri, own ? a.inv_diag[i] : 0.0, lane);
            if (own) {
              a.r[i] = ri;
              a.z[i] = zi;
              rr = ri * ri;
              rzv = ri * zi;
            }
            v[0] += sum6(rr);
            v[1] += sum6(rzv);
          }
        }
        TRACE(k, 3);
        block_allsum<3>(v, sh);
        if (threadIdx.x == 0) {
#pragma unroll
          for (int q = 0; q < 3; ++q) partB[q * G + blockIdx.x] = v[q];
        }
      }
      grid.sync(G);
      double s3[3];
      grid_allsum<3>(partB, s3, G);
      TRACE(k, 4);
      if (s3[2] != 0.0) { status = 1; break; }  // non-finite iterate
      relative = sqrt(s3[0]) / norm_b;
      if (relative < a.tol) break;
      const double rz_new = s3[1];
      beta = rz_new / rz;
      rz = rz_new;
      double* t = pa;  // this iteration's p becomes "previous"
      pa = pb;
      pb = t;
      fold = true;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out_scalars[0] = (double)iterations;
    a.out_scalars[1] = relative;
    a.out_scalars[2] = (double)status;
  }
}

// Owner-register variant of k_pcg (same recurrence, same arithmetic): when a
// warp owns at most PCG_RMAX block rows, lanes 0..5 keep x, r, z, b, M^-1, p
// and Ap of those rows in registers for the whole solve.  Only what the
// neighbours read goes to memory (p every iteration, z every iteration for
// the folded p = z + beta p, x on restart iterations) and x once at the end;
// the update phase issues no loads at all.
#ifndef PCG_RMAX
#define PCG_RMAX 2
#endif
#ifndef PCG_W0SYNC
#define PCG_W0SYNC 1  // barrier + all-sum by warp 0 with one CTA barrier (0: GridBarrier::sync + grid_allsum)
#endif
#ifndef PCG_ROWREG
#define PCG_ROWREG 1  // slot ranges in registers (0: re-read row_ptr per matvec)
#endif
#ifndef PCG_SPLIT_MAX
#define PCG_SPLIT_MAX 8     // warps per block row at most (k_pcg_reg<.., SPLIT>)
#endif
#define PCG_CLUSTER_SMALL 2  // unsplit grids of <= this many CTAs stay one cluster

__device__ __forceinline__ double rsel(const double (&a)[PCG_RMAX], int j) {
  double v = a[0];
#pragma unroll
  for (int k = 1; k < PCG_RMAX; ++k) v = (k == j) ? a[k] : v;
  return v;
}
__device__ __forceinline__ void rset(double (&a)[PCG_RMAX], int j, double v) {
#pragma unroll
  for (int k = 0; k < PCG_RMAX; ++k) a[k] = (k == j) ? v : a[k];
}

// Single-cluster synchronisation for small systems (the whole grid is one
// thread-block cluster of <= 16 CTAs, cfg1-3): a reduction is each CTA's
// block totals stored into EVERY CTA's shared memory (DSMEM, slot = rank)
// followed by one hardware cluster barrier (release/acquire at cluster scope,
// which also publishes the p / z / x writes the neighbours gather from
// global memory); each CTA then sums the G slots in rank order - identical
// bits everywhere.  Slots alternate between two buffers: a CTA writes
// reduction e + 1 only after the barrier of e, and e + 2 only after every CTA
// passed the barrier of e + 1, i.e. finished reading e.
#define PCG_CLUSTER_MAX 16
struct ClusterSync {
  double (*slot)[PCG_CLUSTER_MAX][4];  // [2][rank][value], shared memory
  unsigned epoch;
  __device__ __forceinline__ void barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  template <int NV>
  __device__ __forceinline__ void allsum(double (&v)[NV], double (*sh)[PCG_WARPS], int G) {
    block_allsum<NV>(v, sh);  // thread 0: this CTA's totals
    const int buf = epoch & 1u;
    ++epoch;
    if (threadIdx.x < G) {  // thread t stores this CTA's totals into CTA t
      uint32_t rank;
      asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
      const uint32_t local = (uint32_t)__cvta_generic_to_shared(&slot[buf][rank][0]);
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"((uint32_t)threadIdx.x));
      __shared__ double tot[4];
      if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) tot[k] = v[k];
      }
      __syncwarp((1u << G) - 1u);  // lanes 0 .. G-1 of warp 0
#pragma unroll
      for (int k = 0; k < NV; ++k)
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote + 8 * k), "d"(tot[k]) : "memory");
    }
    barrier();
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double t = 0.0;
      for (int b = 0; b < G; ++b) t += slot[buf][b][k];
      v[k] = t;
    }
  }
};

template <class Mv, bool CL, int SPLIT>
__global__ void __launch_bounds__(PCG_THREADS, 1) k_pcg_reg(PcgArgs a, Mv mv, int rows_per_cta) {
  extern __shared__ __align__(16) double smem[];
  GridBarrier grid{reinterpret_cast<unsigned*>(a.flags), 0u};
  __shared__ double cl_slot[2][PCG_CLUSTER_MAX][4];
  ClusterSync csync{cl_slot, 0u};
  __shared__ double sh[4][PCG_WARPS];
  const int G = gridDim.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // SPLIT warps per block row (each sums its share of the row's slots; the
  // first holds the row's vectors): PCG_WARPS / SPLIT row groups per CTA
  constexpr int RW = PCG_WARPS / SPLIT;
  const int rgw = wid / SPLIT, part = wid % SPLIT;
  const bool own = lane < 6 && part == 0;
  if (a.skip && *a.skip != 0.0) return;  // grid-uniform
  RowCtx rc;
  rc.r0 = min(a.n_blk, blockIdx.x * rows_per_cta);
  rc.r1 = min(a.n_blk, rc.r0 + rows_per_cta);
  rc.s0 = 0;
  rc.Bs = nullptr;
  rc.cols = a.row_col;
  rc.gbuf = smem + wid * PCG_GATHER_CAP * 6;
  rc.s_end = 0;
  if (mv.stageable() && rc.r1 > rc.r0) {
    // the matrix (and its column indices) is constant during the solve: stage
    // this CTA's slot blocks in shared memory once - as many as fit (cfg5's
    // 37 MB exceed the SMs' shared memory; the remaining slots are read from L2)
    rc.s0 = a.row_ptr[rc.r0];
    const int64_t cap = ((int64_t)PCG_SMEM_BYTES - (int64_t)PCG_GATHER_BYTES) / (36 * 8 + 4);
    const int64_t ns = min((int64_t)(a.row_ptr[rc.r1] - rc.s0), cap);
    const int64_t n = ns * 36;
    double* dst = smem + PCG_WARPS * PCG_GATHER_CAP * 6;
    const double* src = a.Brow + (int64_t)rc.s0 * 36;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    int* cdst = reinterpret_cast<int*>(dst + n);
    for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) cdst[i] = a.row_col[rc.s0 + i];
    rc.Bs = dst;
    rc.cols = cdst - rc.s0;  // indexed by global slot
    rc.s_end = rc.s0 + (int)ns;
  }
  __syncthreads();
  // rows of this warp: rc.r0 + rgw + RW * j, j < nrow (<= PCG_RMAX)
  const int nrow = rc.r1 > rc.r0 + rgw ? (rc.r1 - rc.r0 - rgw + RW - 1) / RW : 0;
  // y = A xin over this CTA's rows, the row parts added in part order
  __shared__ double ysh[PCG_WARPS][PCG_RMAX][6];
  // this warp's slot range of each of its rows, held in registers for the
  // solve (row_ptr would otherwise be re-read from L2 after every grid
  // barrier: the barrier's acquire invalidates L1)
  int re0[PCG_RMAX], re1[PCG_RMAX];
#pragma unroll
  for (int j = 0; j < PCG_RMAX; ++j) {
    re0[j] = re1[j] = -1;
    if (PCG_ROWREG && Mv::kSplit && j < nrow) {  // (DenseMv has no row_ptr)
      const int v = rc.r0 + rgw + RW * j;
      const int b0 = a.row_ptr[v], n = a.row_ptr[v + 1] - b0;
      re0[j] = b0 + (n * part) / SPLIT;
      re1[j] = b0 + (n * (part + 1)) / SPLIT;
    }
  }
  auto rows_product = [&](auto fold_tag, const double* zin, const double* xin, double bt,
                          double (&yv)[PCG_RMAX]) {
    constexpr bool FOLD = decltype(fold_tag)::value;
#pragma unroll
    for (int j = 0; j < PCG_RMAX; ++j) {
      yv[j] = 0.0;
      if (j < nrow)
        yv[j] = mv.template row<FOLD>(a, rc, rc.r0 + rgw + RW * j, zin, xin, bt, lane, part, SPLIT, re0[j], re1[j]);
    }
    if constexpr (SPLIT > 1) {
      if (part > 0 && lane < 6) {
#pragma unroll
        for (int j = 0; j < PCG_RMAX; ++j) ysh[wid][j][lane] = yv[j];
      }
      __syncthreads();
      if (part == 0) {
#pragma unroll
        for (int j = 0; j < PCG_RMAX; ++j)
#pragma unroll
          for (int h = 1; h < SPLIT; ++h) yv[j] += ysh[wid + h][j][lane < 6 ? lane : 0];
      }
    }
  };
  double xr[PCG_RMAX], rr_[PCG_RMAX], zr[PCG_RMAX], br[PCG_RMAX], idr[PCG_RMAX], pr[PCG_RMAX],
      apr[PCG_RMAX];
#pragma unroll
  for (int j = 0; j < PCG_RMAX; ++j) xr[j] = rr_[j] = zr[j] = br[j] = idr[j] = pr[j] = apr[j] = 0.0;
  double* pa = a.p;   // p of the previous iteration (read by neighbours)
  double* pb = a.p2;  // p of this iteration (written by owners)
  double* partA = a.part;
  double* partB = a.part + G;

  // ---- setup (solver.py:472-481)
  double tot[2];
  {
    double v[2] = {0.0, 0.0};
    for (int j = 0; j < nrow; ++j) {
      const int row = rc.r0 + rgw + RW * j;
      double bb = 0.0, bz = 0.0;
      const int i = 6 * row + (own ? lane : 0);
      const double bi = own ? -a.g[i] : 0.0;
      const double inv = own ? 1.0 / fmax(a.jdiag[i], 1e-12) : 0.0;
      const double zi = precond(a, row, bi, inv, lane);
      if (own) {
        rset(br, j, bi);
        rset(idr, j, inv);
        rset(rr_, j, bi);
        rset(zr, j, zi);
        rset(pr, j, zi);
        a.z[i] = zi;
        pa[i] = zi;
        bb = bi * bi;
        bz = bi * zi;
      }
      v[0] += sum6(bb);
      v[1] += sum6(bz);
    }
    if constexpr (CL) {
      csync.allsum<2>(v, sh, G);
      tot[0] = v[0];
      tot[1] = v[1];
    } else {
      block_allsum<2>(v, sh);
      if (threadIdx.x == 0) { partB[blockIdx.x] = v[0]; partB[G + blockIdx.x] = v[1]; }
    }
  }
  if constexpr (!CL) {
#if PCG_W0SYNC
    grid.sync_allsum<2>(partB, tot, G);
#else
    grid.sync(G);
    grid_allsum<2>(partB, tot, G);
#endif
  }
  const double norm_b = sqrt(tot[0]);
  double rz = tot[1];
  int iterations = 0;
  double relative = 1.0;
  int status = 0;
  double beta = 0.0;
  bool fold = false;
  if (norm_b == 0.0) {
    relative = 0.0;
  } else {
    for (int k = 1; k <= a.max_it; ++k) {
      iterations = k;
      TRACE(k, 0);
      double pAp_a[1];
      {
        double v[1] = {0.0};
        double yv[PCG_RMAX];
        if (fold) rows_product(std::true_type{}, a.z, pa, beta, yv);
        else rows_product(std::false_type{}, a.z, pa, beta, yv);
        for (int j = 0; j < nrow; ++j) {
          const int row = rc.r0 + rgw + RW * j;
          const double y = rsel(yv, j);
          double pAp = 0.0;
          if (own) {
            const double pold = rsel(pr, j);
            const double pi = fold ? fma(beta, pold, rsel(zr, j)) : pold;
            pb[6 * row + lane] = pi;
            rset(pr, j, pi);
            rset(apr, j, y);
            pAp = pi * y;
          }
          v[0] += sum6(pAp);
        }
        TRACE(k, 1);
        if constexpr (CL) {
          csync.allsum<1>(v, sh, G);
          pAp_a[0] = v[0];
        } else {
          block_allsum<1>(v, sh);
          if (threadIdx.x == 0) partA[blockIdx.x] = v[0];
        }
      }
      if constexpr (!CL) {
#if PCG_W0SYNC
        grid.sync_allsum<1>(partA, pAp_a, G);
#else
        grid.sync(G);
        grid_allsum<1>(partA, pAp_a, G);
#endif
      }
      TRACE(k, 2);
      const double pAp = pAp_a[0];
      if (!isfinite(pAp)) { status = 1; break; }
      if (pAp <= 0.0) break;
      const double alpha = rz / pAp;
      const bool restart = (k % a.restart) == 0;
      double s3[3];
      {
        double v[3] = {0.0, 0.0, 0.0};
        for (int j = 0; j < nrow; ++j) {
          const int row = rc.r0 + rgw + RW * j;
          double rrv = 0.0, rzv = 0.0, bad = 0.0;
          if (own) {
            const int i = 6 * row + lane;
            const double xi = fma(alpha, rsel(pr, j), rsel(xr, j));
            rset(xr, j, xi);
            bad = isfinite(xi) ? 0.0 : 1.0;
            if (restart) a.x[i] = xi;  // read by the neighbours' r = b - A x
          }
          if (!restart) {
            const double ri = own ? fma(-alpha, rsel(apr, j), rsel(rr_, j)) : 0.0;
            const double zi = precond(a, row, ri, rsel(idr, j), lane);
            if (own) {
              rset(rr_, j, ri);
              rset(zr, j, zi);
              a.z[6 * row + lane] = zi;
              rrv = ri * ri;
              rzv = ri * zi;
            }
          }
          v[0] += sum6(rrv);
          v[1] += sum6(rzv);
          v[2] += sum6(bad);
        }
        if (restart) {
          if constexpr (CL) csync.barrier();  // x complete
          else grid.sync(G);
          double yv[PCG_RMAX];
          rows_product(std::false_type{}, nullptr, a.x, 0.0, yv);
          for (int j = 0; j < nrow; ++j) {
            const int row = rc.r0 + rgw + RW * j;
            const double y = rsel(yv, j);
            double rrv = 0.0, rzv = 0.0;
            const double ri = own ? rsel(br, j) - y : 0.0;
            const double zi = precond(a, row, ri, rsel(idr, j), lane);
            if (own) {
              rset(rr_, j, ri);
              rset(zr, j, zi);
              a.z[6 * row + lane] = zi;
              rrv = ri * ri;
              rzv = ri * zi;
            }
            v[0] += sum6(rrv);
            v[1] += sum6(rzv);
          }
        }
        TRACE(k, 3);
        if constexpr (CL) {
          csync.allsum<3>(v, sh, G);
          s3[0] = v[0];
          s3[1] = v[1];
          s3[2] = v[2];
        } else {
          block_allsum<3>(v, sh);
          if (threadIdx.x == 0) {
#pragma unroll
            for (int q = 0; q < 3; ++q) partB[q * G + blockIdx.x] = v[q];
          }
        }
      }
      if constexpr (!CL) {
#if PCG_W0SYNC
        grid.sync_allsum<3>(partB, s3, G);
#else
        grid.sync(G);
        grid_allsum<3>(partB, s3, G);
#endif
      }
      TRACE(k, 4);
      if (s3[2] != 0.0) { status = 1; break; }
      relative = sqrt(s3[0]) / norm_b;
      if (relative < a.tol) break;
      const double rz_new = s3[1];
      beta = rz_new / rz;
      rz = rz_new;
      double* t = pa;
      pa = pb;
      pb = t;
      fold = true;
    }
  }
  for (int j = 0; j < nrow; ++j)
    if (own) a.x[6 * (rc.r0 + rgw + RW * j) + lane] = rsel(xr, j);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out_scalars[0] = (double)iterations;
    a.out_scalars[1] = relative;
    a.out_scalars[2] = (double)status;
  }
}

// Block-Jacobi preconditioner (opt-in, not the reference's scalar Jacobi):
// the inverse of each variable's 6x6 diagonal block of A (D, sparse + dense),
// by Cholesky; a block that is not numerically positive definite falls back
// to the scalar Jacobi inverse of the reference (1 / max(diag, 1e-12)).
__global__ void k_block_jacobi_inv(const double* D, const double* jdiag, int n_blk, double* out) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n_blk) return;
  double A[36];
#pragma unroll
  for (int k = 0; k < 36; ++k) A[k] = D[(int64_t)v * 36 + k];
  double L[36];
#pragma unroll
  for (int k = 0; k < 36; ++k) L[k] = 0.0;
  double dmax = 0.0;
#pragma unroll
  for (int r = 0; r < 6; ++r) dmax = fmax(dmax, fabs(A[r * 7]));
  bool ok = dmax > 0.0 && isfinite(dmax);
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double d = A[c * 7];
#pragma unroll
    for (int k = 0; k < c; ++k) d -= L[c * 6 + k] * L[c * 6 + k];
    ok = ok && d > 1e-12 * dmax;
    const double lc = sqrt(fmax(d, 1e-300));
    L[c * 7] = lc;
#pragma unroll
    for (int r = c + 1; r < 6; ++r) {
      double x = A[r * 6 + c];
#pragma unroll
      for (int k = 0; k < c; ++k) x -= L[r * 6 + k] * L[c * 6 + k];
      L[r * 6 + c] = x / lc;
    }
  }
  double* o = out + (int64_t)v * 36;
  if (!ok) {
#pragma unroll
    for (int k = 0; k < 36; ++k) o[k] = 0.0;
#pragma unroll
    for (int r = 0; r < 6; ++r) o[r * 7] = 1.0 / fmax(jdiag[6 * v + r], 1e-12);
    return;
  }
  // W = L^-1 (lower triangular), A^-1 = W^T W
  double W[36];
#pragma unroll
  for (int k = 0; k < 36; ++k) W[k] = 0.0;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    W[c * 7] = 1.0 / L[c * 7];
#pragma unroll
    for (int r = c + 1; r < 6; ++r) {
      double x = 0.0;
#pragma unroll
      for (int k = c; k < r; ++k) x -= L[r * 6 + k] * W[k * 6 + c];
      W[r * 6 + c] = x / L[r * 7];
    }
  }
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      double x = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) x += W[k * 6 + r] * W[k * 6 + c];
      o[r * 6 + c] = x;
    }
}

void launch_block_jacobi_inv(const double* D, const double* jdiag, int n_blk, double* out,
                             cudaStream_t s) {
  if (n_blk <= 0) return;
  sfb_count_launch();
  k_block_jacobi_inv<<<(n_blk + 127) / 128, 128, 0, s>>>(D, jdiag, n_blk, out);
}

template <class Mv>
static cudaError_t launch_pcg_t(const PcgArgs& a, Mv mv, int n_sm, cudaStream_t s) {
  static bool attr_set = false;
  cudaError_t e;
  if (!attr_set) {
    e = cudaFuncSetAttribute(k_pcg<BsrMv>, cudaFuncAttributeMaxDynamicSharedMemorySize, PCG_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_pcg<DenseMv>, cudaFuncAttributeMaxDynamicSharedMemorySize, PCG_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_pcg_reg<BsrMv, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, PCG_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_pcg_reg<BsrMv, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, PCG_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_pcg_reg<BsrMv, false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, PCG_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_pcg_reg<BsrMv, false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, PCG_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_pcg_reg<DenseMv, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, PCG_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  // one CTA per SM at most (co-residency, cheapest barrier); rows split
  // evenly.  A block row is summed by `split` warps when the grid still fits
  // the SMs that way (more SMs gathering the neighbour vectors).
  const char* split_s = getenv("SFB_PCG_SPLIT");  // tuning / tests: force 1, 2, 4 or 8
  const int split_env = split_s ? atoi(split_s) : 0;
  // Default: the widest split whose grid (one row group per warp group) still
  // fits the SMs, except for tiny systems (<= 2 CTAs unsplit), which run as
  // one cluster.  Measured per 50-iteration solve: cfg4 split 2 388 us vs
  // 457 unsplit; cfg3 split 8 318 vs 398 (cluster of 13); cfg2 cluster 216
  // vs 278-292 split.
  int split = PCG_SPLIT_MAX;
  if ((a.n_blk + PCG_WARPS - 1) / PCG_WARPS <= PCG_CLUSTER_SMALL) split = 1;
  if (split_env == 1 || split_env == 2 || split_env == 4 || split_env == 8) split = split_env;
  if (!Mv::kSplit) split = 1;
  while (split > 1 && (a.n_blk + PCG_WARPS / split - 1) / (PCG_WARPS / split) > n_sm) split /= 2;
  int G = (a.n_blk + PCG_WARPS / split - 1) / (PCG_WARPS / split);
  if (G > n_sm) G = n_sm;
  static const int forced = [] {
    const char* v = getenv("SFB_PCG_BLOCKS");
    return v ? atoi(v) : 0;
  }();
  if (forced > 0 && forced <= n_sm) G = forced;
  if (G < 1) G = 1;
  int rows_per_cta = (a.n_blk + G - 1) / G;
  if (rows_per_cta < 1) rows_per_cta = 1;
  G = (a.n_blk + rows_per_cta - 1) / rows_per_cta;
  if (G < 1) G = 1;
  PcgArgs args = a;
  Mv m = mv;
  void* params[] = {&args, &m, &rows_per_cta};
  e = cudaMemsetAsync(a.flags, 0, sizeof(unsigned), s);  // grid barrier counter
  if (e != cudaSuccess) return e;
  sfb_count_launch();
#ifndef PCG_REG
#define PCG_REG 1
#endif
  if (rows_per_cta > (PCG_WARPS / split) * PCG_RMAX) split = 1;
  const bool reg = PCG_REG && rows_per_cta <= (PCG_WARPS / split) * PCG_RMAX;
#ifndef PCG_CLUSTER
#define PCG_CLUSTER 1
#endif
  if (PCG_CLUSTER && reg && split == 1 && G > 1 && G <= PCG_CLUSTER_MAX) {
    // small system: the whole grid as ONE thread-block cluster (hardware
    // cluster barrier + DSMEM reductions instead of the global grid barrier)
    static int cl_ok = -1;  // cluster launch of this size available (once)
    if (cl_ok < 0) {
      cl_ok = cudaFuncSetAttribute(k_pcg_reg<Mv, true, 1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                      cudaSuccess &&
                  cudaFuncSetAttribute(k_pcg_reg<Mv, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       PCG_SMEM_BYTES) == cudaSuccess
              ? 1
              : 0;
      (void)cudaGetLastError();
    }
    if (cl_ok) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(PCG_THREADS);
      cfg.dynamicSmemBytes = PCG_SMEM_BYTES;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)k_pcg_reg<Mv, true, 1>, &cfg) == cudaSuccess &&
          ncl >= 1)
        return cudaLaunchKernelExC(&cfg, (const void*)k_pcg_reg<Mv, true, 1>, params);
      (void)cudaGetLastError();  // this cluster size does not fit: grid barrier instead
    }
  }
  void* kfn = (void*)k_pcg<Mv>;
  if (reg) {
    if constexpr (Mv::kSplit) {
      kfn = split == 8   ? (void*)k_pcg_reg<Mv, false, 8>
            : split == 4 ? (void*)k_pcg_reg<Mv, false, 4>
            : split == 2 ? (void*)k_pcg_reg<Mv, false, 2>
                         : (void*)k_pcg_reg<Mv, false, 1>;
    } else {
      kfn = (void*)k_pcg_reg<Mv, false, 1>;
    }
  }
  return cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(PCG_THREADS), params, PCG_SMEM_BYTES, s);
}

cudaError_t launch_pcg(const PcgArgs& a, int n_sm, cudaStream_t s) {
  return launch_pcg_t(a, BsrMv{}, n_sm, s);
}

cudaError_t launch_pcg_dense(const PcgArgs& a, const double* A, int n_sm, cudaStream_t s) {
  return launch_pcg_t(a, DenseMv{A}, n_sm, s);
}
