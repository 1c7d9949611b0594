// Dense photometric + point-to-plane terms.
//
//  k_dense_linearize  associate_photo/associate_geo (solver.py:216-260) +
//                     photo_linearize/geo_linearize (:286-328) + _accumulate
//                     (:615-628) fused: one CTA per (directed edge, pixel tile),
//                     one thread per source pixel, 6x6 H_e / g_e / energies
//                     reduced in registers -> warp shuffles -> smem, frozen
//                     associations written as a photo bitmask and a u16 geo
//                     target index per source pixel.
//  k_dense_energy     _energy_with_frozen_associations dense part (:662-672)
//                     through photo_residuals/geo_residuals (:263-283).
//  k_associate / k_point_eval   the per-edge API evaluators.
//
// Since J_j = -J_i for both dense terms (solver.py:310,328), one symmetric
// H_e (21) and one g_e (6) per directed edge carry the whole contribution:
// A_ii += H_e, A_jj += H_e, A_ij = A_ji -= H_e, g_i += g_e, g_j -= g_e.
#include "sfb_kernels.cuh"

#define DENSE_THREADS 256

struct EdgeCtx {
  Xf rel;      // exact pose_j^-1 o pose_i (association gates)
  double Ri[9], ti[3];    // pose_i
  double Rj[9], tj[3];    // pose_j
  double iRj[9], itj[3];  // pose_j^-1 (plain)
  double iRi[9], iti[3];  // pose_i^-1 (plain)
};

__device__ __forceinline__ void load_edge_ctx(EdgeCtx* e, const PoseDev& Pi, const PoseDev& Pj,
                                              const Rounding& rd) {
  e->rel = xf_relative_exact(Pi, Pj, rd);
  for (int k = 0; k < 9; ++k) { e->Ri[k] = Pi.R[k]; e->Rj[k] = Pj.R[k]; }
  for (int k = 0; k < 3; ++k) { e->ti[k] = Pi.t[k]; e->tj[k] = Pj.t[k]; }
  xf_inverse_plain(Pj.R, Pj.t, e->iRj, e->itj);
  xf_inverse_plain(Pi.R, Pi.t, e->iRi, e->iti);
}

// Block-wide deterministic reduction of NV doubles per thread; result in
// out[0..NV) written by thread 0.  Fixed butterfly + fixed warp order.
template <int NV>
__device__ __forceinline__ void block_reduce_store(double (&acc)[NV], double* out) {
  __shared__ double sh[DENSE_THREADS / 32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double v = warp_sum(acc[k]);
    if (lane == 0) sh[warp][k] = v;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < NV; k += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < DENSE_THREADS / 32; ++w) s += sh[w][k];
    out[k] = s;
  }
}

// Association of one source pixel of edge i->j (solver.py:216-260).  Returns
// the photo "inside" bit and the geo target pixel (-1 if not associated).
struct AssocOut {
  bool photo;
  int tgt;
};

__device__ __forceinline__ AssocOut associate_pixel(const EdgeCtx& e, const FrameDev& Fj,
                                                    const float4 P, const float4 N, bool ph,
                                                    bool ge, int ord_ph, int ord_ge,
                                                    const Rounding& rd, double dmax,
                                                    double nmin) {
  AssocOut o{false, -1};
  if (!(ph || ge)) return o;
  const double d0 = P.x, d1 = P.y, d2 = P.z;
  // warped = relative.apply(points); photo and geo index arrays can differ in
  // length, which only matters for NumPy's m == 1 (gemv) rounding order.
  double q[3];
  double u, v;
  bool front;
  if (ph) {
    xf_apply_exact(e.rel, d0, d1, d2, ord_ph, q);
    project_exact(Fj.fx, Fj.fy, Fj.cx, Fj.cy, q, &u, &v, &front);
    o.photo = front && u >= 0.0 && u <= (double)(Fj.w - 1) && v >= 0.0 && v <= (double)(Fj.h - 1);
  }
  if (ge) {
    if (!ph || ord_ge != ord_ph) {
      xf_apply_exact(e.rel, d0, d1, d2, ord_ge, q);
      project_exact(Fj.fx, Fj.fy, Fj.cx, Fj.cy, q, &u, &v, &front);
    }
    const double xr = rint(u), yr = rint(v);  // np.round: half to even
    const bool inside = front && xr >= 0.0 && xr < (double)Fj.w && yr >= 0.0 && yr < (double)Fj.h;
    if (inside) {
      const int ti = (int)yr * Fj.w + (int)xr;
      const float4 PT = __ldg(&Fj.P[ti]);
      const unsigned fl = __float_as_uint(PT.w);
      if ((fl & (SFB_FLAG_VD | SFB_FLAG_VN)) == (SFB_FLAG_VD | SFB_FLAG_VN)) {
        const float4 NT = __ldg(&Fj.N[ti]);
        // distance = np.linalg.norm(warped - targets, axis=1): sequential sum
        const double x0 = __dsub_rn(q[0], (double)PT.x);
        const double x1 = __dsub_rn(q[1], (double)PT.y);
        const double x2 = __dsub_rn(q[2], (double)PT.z);
        const double dist = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x0, x0), __dmul_rn(x1, x1)),
                                                 __dmul_rn(x2, x2)));
        // normal_dot = np.sum(relative.rotate(normals) * target_normals, axis=1)
        double nr[3];
        xf_rotate_exact(e.rel, (double)N.x, (double)N.y, (double)N.z, ord_ge, nr);
        const double nd = __dadd_rn(__dadd_rn(__dmul_rn(nr[0], (double)NT.x),
                                              __dmul_rn(nr[1], (double)NT.y)),
                                    __dmul_rn(nr[2], (double)NT.z));
        if (dist < dmax && nd > nmin) o.tgt = ti;
      }
    }
  }
  return o;
}

// photo_linearize for one pixel (solver.py:286-310): residual (2) and J_i rows
// (2x6) with J_i[r] = [(g_r x world), -g_r], g_r = dval_dq[r] R_j^T.
__device__ __forceinline__ void photo_lin_pixel(const EdgeCtx& e, const FrameDev& Fj, double d0,
                                                double d1, double d2, double ref0, double ref1,
                                                double res[2], double J[2][6]) {
  double wld[3], q[3];
  xf_apply(e.Ri, e.ti, d0, d1, d2, wld);
  xf_apply(e.iRj, e.itj, wld[0], wld[1], wld[2], q);
  const double z = q[2];
  const double zs = z > 0.0 ? z : 1.0;
  const double u = Fj.fx * q[0] / zs + Fj.cx;
  const double v = Fj.fy * q[1] / zs + Fj.cy;
  double val[2], ddx[2], ddy[2];
  bilinear_grad2(Fj, u, v, val, ddx, ddy);
  res[0] = ref0 - val[0];
  res[1] = ref1 - val[1];
  const double iz = 1.0 / z;
  const double a = Fj.fx * iz, b = Fj.fy * iz;
  const double au = -Fj.fx * q[0] * iz * iz, bv = -Fj.fy * q[1] * iz * iz;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const double dq0 = ddx[c] * a, dq1 = ddy[c] * b, dq2 = ddx[c] * au + ddy[c] * bv;
    double g[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) g[k] = dq0 * e.Rj[k * 3 + 0] + dq1 * e.Rj[k * 3 + 1] + dq2 * e.Rj[k * 3 + 2];
    J[c][0] = g[1] * wld[2] - g[2] * wld[1];
    J[c][1] = g[2] * wld[0] - g[0] * wld[2];
    J[c][2] = g[0] * wld[1] - g[1] * wld[0];
    J[c][3] = -g[0];
    J[c][4] = -g[1];
    J[c][5] = -g[2];
  }
}

// geo_linearize for one pixel (solver.py:313-328): J_i = [(world_t x m), m],
// m = R_i n.
__device__ __forceinline__ void geo_lin_pixel(const EdgeCtx& e, double d0, double d1, double d2,
                                              double n0, double n1, double n2, double t0,
                                              double t1, double t2, double* res, double J[6]) {
  double wt[3], mp[3];
  xf_apply(e.Rj, e.tj, t0, t1, t2, wt);
  xf_apply(e.iRi, e.iti, wt[0], wt[1], wt[2], mp);
  *res = n0 * (d0 - mp[0]) + n1 * (d1 - mp[1]) + n2 * (d2 - mp[2]);
  double m[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) m[k] = e.Ri[k * 3 + 0] * n0 + e.Ri[k * 3 + 1] * n1 + e.Ri[k * 3 + 2] * n2;
  J[0] = wt[1] * m[2] - wt[2] * m[1];
  J[1] = wt[2] * m[0] - wt[0] * m[2];
  J[2] = wt[0] * m[1] - wt[1] * m[0];
  J[3] = m[0];
  J[4] = m[1];
  J[5] = m[2];
}

__device__ __forceinline__ bool stride_ok(int p, int w, int stride) {
  if (stride <= 1) return true;
  const int y = p / w, x = p - y * w;
  return (y % stride) == 0 && (x % stride) == 0;
}

// Source-pixel counts of _source_pixel_data (solver.py:158-167) for frame f:
// (valid_depth, valid_depth & valid_normal) on the stride grid.  NumPy's
// rounding of relative.apply differs when exactly one pixel is selected.
__device__ __forceinline__ int2 src_counts(const DenseArgs& a, const FrameDev& F, int f) {
  if (a.stride > 1 && a.stride_counts) return a.stride_counts[f];
  return make_int2(F.n_valid_depth, F.n_valid_geo);
}

__global__ void k_stride_counts(const FrameDev* frames, int stride, int2* out) {
  const FrameDev F = frames[blockIdx.x];
  int cd = 0, cg = 0;
  for (int p = threadIdx.x; p < F.w * F.h; p += blockDim.x) {
    if (!stride_ok(p, F.w, stride)) continue;
    const unsigned fl = __float_as_uint(__ldg(&F.P[p]).w);
    cd += (fl & SFB_FLAG_VD) ? 1 : 0;
    cg += ((fl & SFB_FLAG_VD) && (fl & SFB_FLAG_VN)) ? 1 : 0;
  }
  cd = __reduce_add_sync(0xffffffffu, cd);
  cg = __reduce_add_sync(0xffffffffu, cg);
  __shared__ int sh[2][8];
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = cd;
    sh[1][threadIdx.x >> 5] = cg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a0 = 0, a1 = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a0 += sh[0][w];
      a1 += sh[1][w];
    }
    out[blockIdx.x] = make_int2(a0, a1);
  }
}

void launch_stride_counts(const FrameDev* frames, int n, int stride, int2* out, cudaStream_t s) {
  if (n <= 0) return;
  sfb_count_launch();
  k_stride_counts<<<n, 256, 0, s>>>(frames, stride, out);
}

// ---------------------------------------------------------------------------
// Fused dense pass.  For each (directed edge, pixel tile) item, at the current
// poses, one thread per source pixel:
//   LIN : associate_photo / associate_geo (solver.py:216-260), bit-exact, and
//         photo_linearize / geo_linearize + _accumulate (:286-328, :615-628)
//         into 21 packed H + 6 g + 2 energies;
//   PREV: the frozen-association energy of the PREVIOUS linearisation
//         (_energy_with_frozen_associations, :662-672) at these same poses -
//         the GN loop evaluates E_after(k) and linearises iteration k+1 at the
//         identical poses, so both share the warp, the bilinear sample and
//         the loads.
// Association decisions need NumPy's exact rounding; the division in the
// projection is replaced by a Newton-refined reciprocal and the exact IEEE
// quotient is recomputed only when the approximate pixel lies within 1e-6 px
// of a decision boundary (bounds, or a .5 for np.round), where the two could
// disagree (|u_approx - u| is ~1e-13 px).
//
// Everything after the decisions is evaluated in the target camera j, where
// both dense Jacobians take the form J_i = M_j v (M_j = [[R_j, -[t_j]x R_j],
// [0, -R_j]] per edge, applied once in k_edge_reduce):
//   photo  v = [dq x q ; dq],  dq = d value / d q at q = rel d;
//   geo    v = [t x n' ; -n'], n' = R_rel n, t = the frozen target point,
//          residual n . (d - T_i^-1 T_j t) = n' . (q - t)  (R_rel orthonormal),
// so the rotated normal and q - t of the association gate are reused.  The
// photo rows are accumulated unscaled and the geo row pre-multiplied by
// kappa = sqrt(s_geo / s_photo); k_edge_reduce applies the base scale.

#define DENSE_MAX_TILES 1024

#ifdef DENSE_COUNT
// tuning builds only: pixel counters of the fused pass (sfb_debug_dense_count)
__device__ unsigned long long g_dense_count[8];
extern "C" int sfb_debug_dense_count(unsigned long long* out, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_dense_count, sizeof(g_dense_count));
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_dense_count, z, sizeof(z));
  }
  return (int)e;
}
#endif

// round-half-even for |x| < 2^51 on the FP64 pipe
__device__ __forceinline__ double rint_magic(double x) {
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  return __dsub_rn(__dadd_rn(x, M), M);
}

// 1/z for z > 0 (depths): MUFU seed (~2^-22) + one cubic Newton step, ~1 ulp
__device__ __forceinline__ double rcp_depth(double z) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(z));
  double e = fma(-z, r, 1.0);
  e = fma(e, e, e);
  return fma(r, e, r);
}

// Can any point of this tile's bounding sphere (moved by rel) project into
// the target frustum widened to [-0.5, w-0.5] x [-0.5, h-0.5], z > 0?  The
// radius carries a 1e-7 m margin (>> rounding of the exact per-pixel path).
__device__ __forceinline__ unsigned char tile_maybe_visible(const Xf& rel, const double4 s,
                                                            const FrameDev& Fb) {
  if (s.w < 0.0) return 0;  // no valid pixel in the tile
  double c[3];
  xf_apply(rel.R, rel.t, s.x, s.y, s.z, c);
  const double r = s.w * (1.0 + 1e-7) + 1e-7;
  if (c[2] + r <= 0.0) return 0;
  const double wb = (double)Fb.w - 0.5, hb = (double)Fb.h - 0.5;
  const double n[4][3] = {{Fb.fx, 0.0, Fb.cx + 0.5}, {-Fb.fx, 0.0, wb - Fb.cx},
                          {0.0, Fb.fy, Fb.cy + 0.5}, {0.0, -Fb.fy, hb - Fb.cy}};
  for (int k = 0; k < 4; ++k) {
    const double d = n[k][0] * c[0] + n[k][1] * c[1] + n[k][2] * c[2];
    const double nn = sqrt(n[k][0] * n[k][0] + n[k][1] * n[k][1] + n[k][2] * n[k][2]);
    if (d + r * nn < 0.0) return 0;
  }
  return 1;
}

// Tensor-memory accumulators: the 27 H/g sums of each thread live in TMEM (54
// 32-bit columns of its lane; warp w uses lanes 32(w%4).. and columns
// 64(w/4)..), read-modify-written once per tile by the warp (tcgen05.ld/st,
// warp-converged), so registers hold only the tile's Jacobian rows.  The
// per-entry FMA order is photo row 0, photo row 1, geo row.
#define TM_LD8(addr, u)                                                                         \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"         \
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]),      \
                 "=r"(u[6]), "=r"(u[7])                                                        \
               : "r"(addr))
#define TM_ST8(addr, u)                                                                         \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"         \
               ::"r"(addr), "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), \
                 "r"(u[6]), "r"(u[7])                                                          \
               : "memory")
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ double tm_d(const uint32_t* u, int k) {
  return __hiloint2double((int)u[2 * k + 1], (int)u[2 * k]);
}
__device__ __forceinline__ void tm_set(uint32_t* u, int k, double v) {
  u[2 * k] = (uint32_t)__double2loint(v);
  u[2 * k + 1] = (uint32_t)__double2hiint(v);
}
__host__ __device__ constexpr int sym6_row(int e) {
  int r = 0;
  while (e >= 6 - r) { e -= 6 - r; ++r; }
  return r;
}
__host__ __device__ constexpr int sym6_col(int e) {
  int r = 0;
  while (e >= 6 - r) { e -= 6 - r; ++r; }
  return e + r;
}
// entry E of the 27 (21 packed H, then 6 g)
template <int E>
__device__ __forceinline__ double tm_update(double acc, const double (&jp)[2][6],
                                            const double (&rp)[2], const double (&jg)[6],
                                            double rg) {
  if constexpr (E < 21) {
    constexpr int r = sym6_row(E), c = sym6_col(E);
    acc = fma(jp[0][r], jp[0][c], acc);
    acc = fma(jp[1][r], jp[1][c], acc);
    return fma(jg[r], jg[c], acc);
  } else {
    constexpr int r = E - 21;
    acc = fma(jp[0][r], rp[0], acc);
    acc = fma(jp[1][r], rp[1], acc);
    return fma(jg[r], rg, acc);
  }
}
// entries 4Q..4Q+3 (x8 = 4 doubles per tcgen05.ld/st: at 64 registers the
// narrower chunk spills less than x16 - 4.34 vs 4.65 ms per launch at cfg4)
template <int Q>
__device__ __forceinline__ void tm_chunk(uint32_t tm, const double (&jp)[2][6], const double (&rp)[2],
                                         const double (&jg)[6], double rg) {
  uint32_t u[8];
  TM_LD8(tm + 8 * Q, u);
  tm_wait_ld();
  tm_set(u, 0, tm_update<4 * Q + 0>(tm_d(u, 0), jp, rp, jg, rg));
  tm_set(u, 1, tm_update<4 * Q + 1>(tm_d(u, 1), jp, rp, jg, rg));
  tm_set(u, 2, tm_update<4 * Q + 2>(tm_d(u, 2), jp, rp, jg, rg));
  if constexpr (4 * Q + 3 < 27) tm_set(u, 3, tm_update<4 * Q + 3>(tm_d(u, 3), jp, rp, jg, rg));
  TM_ST8(tm + 8 * Q, u);
}
#ifndef DENSE_F32GUARD
#define DENSE_F32GUARD 1
#endif
// DENSE_NOSKIP=1: the geo and photo sections run for every warp of a live
// tile instead of being skipped when no lane needs them, so they form one
// straight-line block the compiler interleaves (4.23 -> 4.08 ms per launch
// at cfg4; nearly every live warp needs both anyway)
#ifndef DENSE_NOSKIP
#define DENSE_NOSKIP 1
#endif
// DENSE_TMA_P=1: stage each warp's source strip by cp.async.bulk (measured
// 27% slower on the B200; kept as a compile-time variant)
#ifndef DENSE_TMA_P
#define DENSE_TMA_P 0
#endif
#ifndef DENSE_TMEM_BLOCKS
#define DENSE_TMEM_BLOCKS 4
#endif

// H / g base scale and the geo row factor of a linearisation
__host__ __device__ inline void dense_scales(double s_photo, double s_geo, double* base,
                                             double* kappa) {
  if (s_photo > 0.0) {
    *base = s_photo;
    *kappa = sqrt(s_geo / s_photo);
  } else {
    *base = s_geo;
    *kappa = 1.0;
  }
}

// Loop-invariant state of one (directed edge, tile range) item.
struct TileCtx {
  const float4* Pi;
  const float4* Ni;
  const float2* Gi;
  int wi, hi, tiles_x;
  int ord_ph, ord_ge;   // NumPy apply rounding orders (generic path)
  double wm1, hm1, dwj, dhj;
  double kappa;
  uint32_t* pmask;
  uint16_t* gtgt;
  const uint32_t* pmask_prev;
  const uint16_t* gtgt_prev;
};

// exact 3-term dot in NumPy's order: FAST = the forward FMA chain
template <bool FAST>
__device__ __forceinline__ double dotx(double a0, double a1, double a2, double b0, double b1,
                                       double b2, int o) {
  if (FAST) return __fma_rn(a2, b2, __fma_rn(a1, b1, __dmul_rn(a0, b0)));
  return dot3o(a0, a1, a2, b0, b1, b2, o);
}

// One 16x16 source tile of an item: the warp's 32 pixels are evaluated
// branch-free (every lane computes with clamped indices, results are
// selected by the lane's predicates), so all gathers of a pixel issue as
// soon as their addresses are known; sections no lane of the warp needs are
// skipped warp-uniformly.  Rare exact-rounding fallbacks stay divergent.
template <bool PREV, bool FAST>
__device__ __forceinline__ void dense_tile(const DenseArgs& a, const TileCtx& c, const Xf& rel,
                                           const FrameDev& Fj, uint32_t tm, int t, int tx, int ty,
                                           unsigned st, unsigned char* tstate, double& acc27,
                                           double& acc28, double& eprev_p, double& eprev_g,
                                           const float4* Ps) {
  const int lane = threadIdx.x & 31;
  const bool vis = st & 1u;
  const bool prev_here = PREV && (st & 2u);
  const int x = tx * SFB_TILE + (threadIdx.x & (SFB_TILE - 1));
  const int y = ty * SFB_TILE + (threadIdx.x / SFB_TILE);
  const bool live = x < c.wi && y < c.hi;
  const int p = live ? y * c.wi + x : 0;  // pixel (0: safe index)
  const int m = t * 256 + threadIdx.x;    // slot
  // source point: this warp's strip staged in shared memory by TMA (Ps), or L1
  const float4 P = Ps ? Ps[threadIdx.x & 31] : __ldg(&c.Pi[p]);
  const unsigned fl = live ? __float_as_uint(P.w) : 0u;
  const bool sok = vis && stride_ok(p, c.wi, a.stride);
  const bool ph = a.do_photo && sok && (fl & SFB_FLAG_VD);
  const bool ge = a.do_geo && sok && (fl & SFB_FLAG_VD) && (fl & SFB_FLAG_VN);
  bool pph = false;
  int ptg = 0xFFFF;
  if (prev_here) {
    const uint32_t w = c.pmask_prev[m >> 5];
    const int g = c.gtgt_prev[m];
    if (live) {
      pph = a.prev_photo && ((w >> (m & 31)) & 1u);
      ptg = a.prev_geo ? g : 0xFFFF;
    }
  }
  const bool pge = PREV && ptg != 0xFFFF;
  const bool any_ph = __any_sync(0xffffffffu, ph || pph);
  const bool any_ge = __any_sync(0xffffffffu, ge || pge);
  if (!(any_ph || any_ge)) {
    if (a.do_photo && lane == 0) c.pmask[m >> 5] = 0u;
    if (a.do_geo) c.gtgt[m] = 0xFFFF;
    return;
  }
  const double d0 = P.x, d1 = P.y, d2 = P.z;
  const int ord = FAST ? 0 : (ph ? c.ord_ph : c.ord_ge);
  // warped = relative.apply(points): NumPy rounding
  double q0 = __dadd_rn(dotx<FAST>(d0, d1, d2, rel.R[0], rel.R[1], rel.R[2], ord), rel.t[0]);
  double q1 = __dadd_rn(dotx<FAST>(d0, d1, d2, rel.R[3], rel.R[4], rel.R[5], ord), rel.t[1]);
  double q2 = __dadd_rn(dotx<FAST>(d0, d1, d2, rel.R[6], rel.R[7], rel.R[8], ord), rel.t[2]);
  bool front = q2 > 0.0;
  double z = front ? q2 : 1.0;
  const double rz = rcp_depth(z);
  const double tu = __dmul_rn(Fj.fx, q0), tv = __dmul_rn(Fj.fy, q1);
  const double ua = fma(tu, rz, Fj.cx);
  const double va = fma(tv, rz, Fj.cy);
  // associate_photo: decide with a 1e-6 px guard band, exact quotient inside it
  bool ph_in = false;
#if DENSE_F32GUARD
  // classify in float32 with a 1e-3 px band (float rounding of ua is <= 2e-5
  // px at these image sizes): the FP64 pipe only sees the rare band cases
  const float uf = __double2float_rn(ua), vf = __double2float_rn(va);
#endif
  {
#if DENSE_F32GUARD
    const float EB = 1e-3f, wf = (float)c.wm1, hf = (float)c.hm1;
    const bool in_c = uf > EB && uf < wf - EB && vf > EB && vf < hf - EB;
    const bool out_c = uf < -EB || uf > wf + EB || vf < -EB || vf > hf + EB;
#else
    const double E = 1e-6;
    const bool in_c = ua > E && ua < c.wm1 - E && va > E && va < c.hm1 - E;
    const bool out_c = ua < -E || ua > c.wm1 + E || va < -E || va > c.hm1 + E;
#endif
    ph_in = ph && front && in_c;
    if (ph && !(in_c | out_c)) {
      const double u = __dadd_rn(__ddiv_rn(tu, z), Fj.cx);
      const double v = __dadd_rn(__ddiv_rn(tv, z), Fj.cy);
      ph_in = front && u >= 0.0 && u <= c.wm1 && v >= 0.0 && v <= c.hm1;
    }
  }
  // ---- associate_geo (+ the frozen geo energy of the previous pass)
  int tgt = -1;
  double nj0 = 0.0, nj1 = 0.0, nj2 = 0.0, t0 = 0.0, t1 = 0.0, t2 = 0.0, rg = 0.0;
  if (DENSE_NOSKIP || any_ge) {
    if (!FAST && ph && c.ord_ge != c.ord_ph) {  // m == 1 special case: re-derive the warp
      q0 = __dadd_rn(dot3o(d0, d1, d2, rel.R[0], rel.R[1], rel.R[2], c.ord_ge), rel.t[0]);
      q1 = __dadd_rn(dot3o(d0, d1, d2, rel.R[3], rel.R[4], rel.R[5], c.ord_ge), rel.t[1]);
      q2 = __dadd_rn(dot3o(d0, d1, d2, rel.R[6], rel.R[7], rel.R[8], c.ord_ge), rel.t[2]);
      front = q2 > 0.0;
      z = front ? q2 : 1.0;
    }
    double u = ua, v = va;
#if DENSE_F32GUARD
    const bool finite_uv = fabsf(uf) < 1e9f && fabsf(vf) < 1e9f;
#else
    const bool finite_uv = fabs(u) < 1e9 && fabs(v) < 1e9;
#endif
    double xr = finite_uv ? rint_magic(u) : 0.0, yr = finite_uv ? rint_magic(v) : 0.0;
    // np.round ties: recompute the exact quotient when within 1e-6 px of a .5
    if (ge && finite_uv &&
        (fabs(u - xr) > 0.5 - 1e-6 || fabs(v - yr) > 0.5 - 1e-6 || (!FAST && ph && c.ord_ge != c.ord_ph))) {
      u = __dadd_rn(__ddiv_rn(__dmul_rn(Fj.fx, q0), z), Fj.cx);
      v = __dadd_rn(__ddiv_rn(__dmul_rn(Fj.fy, q1), z), Fj.cy);
      xr = rint_magic(u);
      yr = rint_magic(v);
    }
#if DENSE_F32GUARD
    // |u|, |v| < 1e9: the rounded values are exact 32-bit integers in the
    // magic sum's low word; bounds as unsigned integer compares
    const int xi = __double2loint(__dadd_rn(xr, 6755399441055744.0));
    const int yi = __double2loint(__dadd_rn(yr, 6755399441055744.0));
    const bool inside = ge && front && finite_uv && (unsigned)xi < (unsigned)Fj.w &&
                        (unsigned)yi < (unsigned)Fj.h;
    const int ti = inside ? yi * Fj.w + xi : 0;
#else
    const bool inside = ge && front && finite_uv && xr >= 0.0 && xr < c.dwj && yr >= 0.0 && yr < c.dhj;
    const int ti = inside ? __double2loint(__dadd_rn(yr, 6755399441055744.0)) * Fj.w +
                                __double2loint(__dadd_rn(xr, 6755399441055744.0))
                          : 0;
#endif
    const float4 PT = __ldg(&Fj.P[ti]);
    const float4 NT = __ldg(&Fj.N[ti]);
    const float4 N = __ldg(&c.Ni[p]);
    const float4 PP = __ldg(&Fj.P[pge ? ptg : ti]);
    // normal_dot operand: relative.rotate(normals), NumPy rounding
    const int og = FAST ? 0 : c.ord_ge;
    const double n0 = N.x, n1 = N.y, n2 = N.z;
    const double nr0 = dotx<FAST>(n0, n1, n2, rel.R[0], rel.R[1], rel.R[2], og);
    const double nr1 = dotx<FAST>(n0, n1, n2, rel.R[3], rel.R[4], rel.R[5], og);
    const double nr2 = dotx<FAST>(n0, n1, n2, rel.R[6], rel.R[7], rel.R[8], og);
    const unsigned tf = __float_as_uint(PT.w);
    const bool tvalid = inside && (tf & (SFB_FLAG_VD | SFB_FLAG_VN)) == (SFB_FLAG_VD | SFB_FLAG_VN);
    const double x0 = __dsub_rn(q0, (double)PT.x);
    const double x1 = __dsub_rn(q1, (double)PT.y);
    const double x2 = __dsub_rn(q2, (double)PT.z);
    // norm < dmax: compare squares; correctly rounded sqrt only near the gate
    const double s2 = __dadd_rn(__dadd_rn(__dmul_rn(x0, x0), __dmul_rn(x1, x1)), __dmul_rn(x2, x2));
    const double dm2 = a.geo_dmax * a.geo_dmax;
    bool near = s2 < dm2 * (1.0 - 1e-12);
    if (tvalid && !near && !(s2 > dm2 * (1.0 + 1e-12))) near = __dsqrt_rn(s2) < a.geo_dmax;
    // normal_dot = np.sum(rotated * target_normals, axis=1)
    const double nd = __dadd_rn(__dadd_rn(__dmul_rn(nr0, (double)NT.x), __dmul_rn(nr1, (double)NT.y)),
                                __dmul_rn(nr2, (double)NT.z));
    const bool gok = tvalid && near && nd > a.geo_nmin;
    tgt = gok ? ti : -1;
    const double r_new = nr0 * x0 + nr1 * x1 + nr2 * x2;  // geo_linearize residual
    const double e_new = r_new * r_new;
    acc28 += gok ? e_new : 0.0;
    if (PREV) {
      const double rpv = nr0 * (q0 - (double)PP.x) + nr1 * (q1 - (double)PP.y) + nr2 * (q2 - (double)PP.z);
      eprev_g += pge ? (ptg == tgt ? e_new : rpv * rpv) : 0.0;
    }
    const double kg = gok ? c.kappa : 0.0;
    rg = kg * r_new;
    nj0 = kg * nr0;
    nj1 = kg * nr1;
    nj2 = kg * nr2;
    t0 = PT.x;
    t1 = PT.y;
    t2 = PT.z;
  }
  // frozen sets (tile-major slots)
  const unsigned pword = __ballot_sync(0xffffffffu, ph_in);
  if (a.do_photo && lane == 0) c.pmask[m >> 5] = pword;
  if (a.do_geo) c.gtgt[m] = tgt >= 0 ? (uint16_t)tgt : (uint16_t)0xFFFF;
  const bool any_new = __any_sync(0xffffffffu, ph_in || tgt >= 0);
  // every warp that freezes an association in this tile stores the same
  // byte (bits 0-1 are constant after the barrier): no read-modify-write
  if (any_new && lane == 0) tstate[0] = (unsigned char)(st | 4u);
#ifdef DENSE_COUNT
  {
    const unsigned b0 = __ballot_sync(0xffffffffu, live && vis);
    const unsigned b1 = __ballot_sync(0xffffffffu, ph);
    const unsigned b3 = __ballot_sync(0xffffffffu, ge);
    const unsigned b4 = __ballot_sync(0xffffffffu, tgt >= 0);
    const unsigned b5 = __ballot_sync(0xffffffffu, live);
    if (lane == 0) {
      atomicAdd(&g_dense_count[0], (unsigned long long)__popc(b0));
      atomicAdd(&g_dense_count[1], (unsigned long long)__popc(b1));
      atomicAdd(&g_dense_count[2], (unsigned long long)__popc(pword));
      atomicAdd(&g_dense_count[3], (unsigned long long)__popc(b3));
      atomicAdd(&g_dense_count[4], (unsigned long long)__popc(b4));
      atomicAdd(&g_dense_count[5], (unsigned long long)__popc(b5));
      atomicAdd(&g_dense_count[6], 32ull);
    }
  }
#endif
  // ---- photometric: one bilinear sample serves the frozen energy and J
  double dq0[2] = {0.0, 0.0}, dq1[2] = {0.0, 0.0}, rp[2] = {0.0, 0.0};
  if (DENSE_NOSKIP || any_ph) {
    double val[2], ddx[2], ddy[2];
    bilinear_grad2_fast(Fj, ua, va, val, ddx, ddy);
    const float2 ref = __ldg(&c.Gi[p]);
    const double r0 = (double)ref.x - val[0], r1 = (double)ref.y - val[1];
    const double e2 = r0 * r0 + r1 * r1;
    if (PREV) eprev_p += pph ? e2 : 0.0;
    acc27 += ph_in ? e2 : 0.0;
    const double a_ = ph_in ? Fj.fx * rz : 0.0, b_ = ph_in ? Fj.fy * rz : 0.0;
    dq0[0] = ddx[0] * a_;
    dq0[1] = ddx[1] * a_;
    dq1[0] = ddy[0] * b_;
    dq1[1] = ddy[1] * b_;
    rp[0] = ph_in ? r0 : 0.0;
    rp[1] = ph_in ? r1 : 0.0;
  }
  if (any_new) {
    double jp[2][6], jg[6];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double dq2 = -(dq0[k] * q0 + dq1[k] * q1) * rz;
      jp[k][0] = dq1[k] * q2 - dq2 * q1;
      jp[k][1] = dq2 * q0 - dq0[k] * q2;
      jp[k][2] = dq0[k] * q1 - dq1[k] * q0;
      jp[k][3] = dq0[k];
      jp[k][4] = dq1[k];
      jp[k][5] = dq2;
    }
    jg[0] = t1 * nj2 - t2 * nj1;
    jg[1] = t2 * nj0 - t0 * nj2;
    jg[2] = t0 * nj1 - t1 * nj0;
    jg[3] = -nj0;
    jg[4] = -nj1;
    jg[5] = -nj2;
    tm_chunk<0>(tm, jp, rp, jg, rg);
    tm_chunk<1>(tm, jp, rp, jg, rg);
    tm_chunk<2>(tm, jp, rp, jg, rg);
    tm_chunk<3>(tm, jp, rp, jg, rg);
    tm_chunk<4>(tm, jp, rp, jg, rg);
    tm_chunk<5>(tm, jp, rp, jg, rg);
    tm_chunk<6>(tm, jp, rp, jg, rg);
    tm_wait_st();
  }
}

template <bool PREV, bool FAST>
__device__ __forceinline__ void dense_tiles(const DenseArgs& a, const TileCtx& c, const Xf& rel,
                                            const FrameDev& Fj, uint32_t tm, int4 it,
                                            unsigned char* tile_state, double& acc27, double& acc28,
                                            double& eprev_p, double& eprev_g) {
#if DENSE_TMA_P
  // The source points of each warp's 16x2 strip come in by TMA bulk copies
  // (cp.async.bulk, one per row) into a per-warp double buffer in shared
  // memory, issued one live tile ahead and completed on a per-warp mbarrier,
  // so a tile's dependency chain starts from shared memory.
  __shared__ __align__(16) float4 pstrip[DENSE_THREADS / 32][2][32];
  __shared__ __align__(8) unsigned long long pbar[DENSE_THREADS / 32][2];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&pbar[w][b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned phase = 0;  // bit b: parity of buffer b's next completion
  auto issue = [&](int t, int b) {
    if (lane != 0) return;
    const int x0 = (t % c.tiles_x) * SFB_TILE, y0 = (t / c.tiles_x) * SFB_TILE + 2 * w;
    const int nx = min(SFB_TILE, c.wi - x0);
    const int nrow = y0 >= c.hi ? 0 : (y0 + 1 < c.hi ? 2 : 1);
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&pbar[w][b]);
    const uint32_t bytes = (uint32_t)(nrow * nx * 16);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    for (int r = 0; r < nrow; ++r) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&pstrip[w][b][16 * r]);
      const float4* src = c.Pi + (int64_t)(y0 + r) * c.wi + x0;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(src), "r"((uint32_t)(nx * 16)), "r"(bar) : "memory");
    }
  };
  auto next_live = [&](int t) {
    while (t < it.z && !(tile_state[t - it.y] & 3u)) ++t;
    return t;
  };
  int t = next_live(it.y);
  int b = 0;
  if (t < it.z) issue(t, 0);
  while (t < it.z) {
    const int tn = next_live(t + 1);
    __syncwarp();  // every lane is done with buffer b ^ 1 (read two tiles ago)
    if (tn < it.z) issue(tn, b ^ 1);
    {
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&pbar[w][b]);
      const uint32_t par = (phase >> b) & 1u;
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(bar), "r"(par) : "memory");
      phase ^= 1u << b;
    }
    const unsigned st = tile_state[t - it.y];
    dense_tile<PREV, FAST>(a, c, rel, Fj, tm, t, t % c.tiles_x, t / c.tiles_x, st,
                           &tile_state[t - it.y], acc27, acc28, eprev_p, eprev_g, &pstrip[w][b][0]);
    b ^= 1;
    t = tn;
  }
#else
  int tx = it.y % c.tiles_x, ty = it.y / c.tiles_x;
  for (int t = it.y; t < it.z; ++t, (++tx == c.tiles_x ? (tx = 0, ++ty) : 0)) {
    const unsigned st = tile_state[t - it.y];
    if (!(st & 3u)) continue;  // nothing to associate, nothing frozen
    dense_tile<PREV, FAST>(a, c, rel, Fj, tm, t, tx, ty, st, &tile_state[t - it.y], acc27, acc28,
                           eprev_p, eprev_g, nullptr);
  }
#endif
}

template <bool PREV>
__global__ void __launch_bounds__(DENSE_THREADS, DENSE_TMEM_BLOCKS) k_dense_fused(DenseArgs a) {
  // per-item context in shared memory (re-read per tile instead of held in
  // registers across the tile loop)
  __shared__ Xf rel;  // pose_j^-1 o pose_i, NumPy rounding
  __shared__ TileCtx c;
  __shared__ FrameDev Fj;
  __shared__ uint32_t tm_base;
  const int4 it = a.items[blockIdx.x];
  const int2 de = a.dir_edges[it.x];
  if (a.edge_rel && threadIdx.x < 12)  // precomputed by k_edge_rel (12 parallel loads)
    (&rel.R[0])[threadIdx.x] = a.edge_rel[12 * (int64_t)it.x + threadIdx.x];
  if (threadIdx.x == 0) {
    if (!a.edge_rel) rel = xf_relative_exact(a.poses[de.x], a.poses[de.y], a.rd);
    const FrameDev Fi = a.frames[de.x];
    Fj = a.frames[de.y];
    const int2 nsrc = src_counts(a, Fi, de.x);
    c.ord_ph = (nsrc.x == 1) ? a.rd.apply_1 : a.rd.apply_n;
    c.ord_ge = (nsrc.y == 1) ? a.rd.apply_1 : a.rd.apply_n;
    c.Pi = Fi.P;
    c.Ni = Fi.N;
    c.Gi = Fi.G;
    c.wi = Fi.w;
    c.hi = Fi.h;
    c.tiles_x = Fi.tiles_x;
    c.pmask = a.photo_mask + a.photo_off[it.x];
    c.gtgt = a.geo_tgt + a.geo_off[it.x];
    c.pmask_prev = PREV ? a.photo_mask_prev + a.photo_off[it.x] : nullptr;
    c.gtgt_prev = PREV ? a.geo_tgt_prev + a.geo_off[it.x] : nullptr;
    c.wm1 = (double)(Fj.w - 1);
    c.hm1 = (double)(Fj.h - 1);
    c.dwj = (double)Fj.w;
    c.dhj = (double)Fj.h;
    double base;
    dense_scales(a.s_photo, a.s_geo, &base, &c.kappa);
  }
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tm_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp w: lanes 32*(w%4).., columns 64*(w/4) .. +54
  const uint32_t tm = tm_base + ((uint32_t)(((threadIdx.x >> 5) & 3) * 32) << 16) +
                      (uint32_t)((threadIdx.x >> 7) * 64);
  {
    uint32_t z[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) z[k] = 0u;
#pragma unroll
    for (int q = 0; q < 7; ++q) TM_ST8(tm + 8 * q, z);
    tm_wait_st();
  }

  // Tile culling: a 16x16 source tile whose bounding sphere lies outside
  // the target frustum widened to the geo rounding bounds [-0.5, w-0.5]
  // cannot associate any pixel (photo bounds [0, w-1] are inside that), so
  // its pixels skip the association entirely - decisions are unchanged.
  // tile_state bit0: may be visible now; bit1: the previous pass froze an
  // association in it; bit2 (set below): this pass freezes one.  Slots of a
  // tile whose bit2 ends up clear are never read (the flag says so).
  __shared__ unsigned char tile_state[DENSE_MAX_TILES];
  const int toff = (int)(a.geo_off[it.x] >> 8);  // this edge's first tile flag
  {
    const double4* tiles = a.frames[de.x].tiles;
    for (int t = it.y + threadIdx.x; t < it.z; t += blockDim.x) {
      unsigned char s = tile_maybe_visible(rel, tiles[t], Fj);
      if (PREV && a.tile_any_prev[toff + t]) s |= 2;
      tile_state[t - it.y] = s;
    }
  }
  __syncthreads();

  double acc27 = 0.0, acc28 = 0.0;  // photo / geo energy at association
  double eprev_p = 0.0, eprev_g = 0.0;
  // pixels in tile-major order: slot m = tile * 256 + threadIdx.x (the frozen
  // association buffers use the same slots; a warp covers 16x2 pixels)
  if (a.rd.apply_n == 0 && c.ord_ph == 0 && c.ord_ge == 0)
    dense_tiles<PREV, true>(a, c, rel, Fj, tm, it, tile_state, acc27, acc28, eprev_p, eprev_g);
  else
    dense_tiles<PREV, false>(a, c, rel, Fj, tm, it, tile_state, acc27, acc28, eprev_p, eprev_g);

  double base_scale, kappa;
  dense_scales(a.s_photo, a.s_geo, &base_scale, &kappa);
  double acc[31];
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    uint32_t u[8];
    TM_LD8(tm + 8 * q, u);
    tm_wait_ld();
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (4 * q + k < 27) acc[4 * q + k] = base_scale * tm_d(u, k);
  }
  acc[27] = acc27;
  acc[28] = acc28;
  acc[29] = eprev_p;  // zero without PREV
  acc[30] = eprev_g;
  double* out = a.item_out + (int64_t)blockIdx.x * SFB_ITEM_STRIDE;
  block_reduce_store<31>(acc, out);
  // (block_reduce_store synchronised the CTA: tile_state bit2 is final)
  for (int t = it.y + threadIdx.x; t < it.z; t += blockDim.x)
    a.tile_any[toff + t] = (tile_state[t - it.y] & 4u) ? 1 : 0;
  // every warp's last TMEM read completed (wait::ld) before block_reduce_store's barrier
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm_base));
  }
}

// relative = pose_j^-1 o pose_i with NumPy's rounding (frames.py:168,
// solver.py:221) for every directed edge, once per dense pass, so the pass's
// CTAs start with 12 parallel loads instead of one thread's serial chain
__global__ void k_edge_rel(const int2* dir_edges, const PoseDev* poses, Rounding rd, int n_dir,
                           double* out) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n_dir) return;
  const int2 e = dir_edges[d];
  const Xf r = xf_relative_exact(poses[e.x], poses[e.y], rd);
#pragma unroll
  for (int k = 0; k < 9; ++k) out[12 * (int64_t)d + k] = r.R[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) out[12 * (int64_t)d + 9 + k] = r.t[k];
}

void launch_dense_linearize(const DenseArgs& a, cudaStream_t s) {
  if (a.n_items <= 0) return;
  const bool prev = a.photo_mask_prev != nullptr;
  const DenseArgs& b = a;
  if (a.edge_rel && a.n_dir > 0) {
    sfb_count_launch();
    k_edge_rel<<<(a.n_dir + 127) / 128, 128, 0, s>>>(a.dir_edges, a.poses, a.rd, a.n_dir, a.edge_rel);
  }
  sfb_count_launch();
  if (prev) k_dense_fused<true><<<a.n_items, DENSE_THREADS, 0, s>>>(b);
  else k_dense_fused<false><<<a.n_items, DENSE_THREADS, 0, s>>>(b);
}

// Frozen-association energy at the current poses (the last GN iteration's
// energy_after, _energy_with_frozen_associations :662-672; the others are
// fused into the next k_dense_fused<PREV>): the same formulation as the fused
// pass's PREV sums - q = rel d (FMA chain), reciprocal-multiply projection,
// one bilinear sample, geo residual n' . (q - t) with n' = R_rel n - over
// the frozen sets only.  Tiles without a frozen association are skipped by
// their flag, warps without one warp-uniformly; each pixel's loads issue
// together (clamped indices, predicate selects).
__device__ __forceinline__ void bilinear_val2_fast(const FrameDev& f, double x, double y, double val[2]) {
  const int xf = __double2int_rd(x), yf = __double2int_rd(y);
  const int x0 = min(max(xf, 0), f.w - 2), y0 = min(max(yf, 0), f.h - 2);
  double ax = x - (double)x0, ay = y - (double)y0;
  ax = xf < 0 ? 0.0 : (xf > f.w - 2 ? 1.0 : ax);
  ay = yf < 0 ? 0.0 : (yf > f.h - 2 ? 1.0 : ay);
  const float4 t0 = __ldg(&f.T[2 * (y0 * f.w + x0)]);
  const float4 t1 = __ldg(&f.T[2 * (y0 * f.w + x0) + 1]);
  const double v00[2] = {t0.x, t0.y}, v01[2] = {t0.z, t0.w};
  const double v10[2] = {t1.x, t1.y}, v11[2] = {t1.z, t1.w};
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const double d01 = v01[c] - v00[c], d10 = v10[c] - v00[c];
    const double dxy = (v11[c] - v10[c]) - d01;
    val[c] = fma(ay, fma(ax, dxy, d10), fma(ax, d01, v00[c]));
  }
}

#ifndef ENERGY_ILP
#define ENERGY_ILP 2  // flagged tiles evaluated together per iteration
#endif
#ifndef ENERGY_BLOCKS
#define ENERGY_BLOCKS 4
#endif
#ifndef ENERGY_NEXT
#define ENERGY_NEXT 1  // next flagged tile by table lookup (0: scan the flags)
#endif
#ifndef ENERGY_PF
#define ENERGY_PF 0  // 1: next group's frozen-set words one group ahead (measured 1.73 vs 1.63 ms: off)
#endif
__global__ void __launch_bounds__(DENSE_THREADS, ENERGY_BLOCKS) k_dense_energy(DenseArgs a, double* item_e2) {
  __shared__ Xf rel;
  __shared__ FrameDev Fj;
  __shared__ const float4* sPi;
  __shared__ const float4* sNi;
  __shared__ const float2* sGi;
  __shared__ int swi, stx;
  __shared__ unsigned char tflag[DENSE_MAX_TILES];
  const int4 it = a.items[blockIdx.x];
  const int2 de = a.dir_edges[it.x];
  const int toff = (int)(a.geo_off[it.x] >> 8);
  if (threadIdx.x < 12) (&rel.R[0])[threadIdx.x] = a.edge_rel[12 * (int64_t)it.x + threadIdx.x];
  if (threadIdx.x == 0) {
    const FrameDev& Fi = a.frames[de.x];
    Fj = a.frames[de.y];
    sPi = Fi.P;
    sNi = Fi.N;
    sGi = Fi.G;
    swi = Fi.w;
    stx = Fi.tiles_x;
  }
  for (int t = it.y + threadIdx.x; t < it.z; t += blockDim.x) tflag[t - it.y] = a.tile_any[toff + t];
  __syncthreads();
  const uint32_t* pmask = a.photo_mask + a.photo_off[it.x];
  const uint16_t* gtgt = a.geo_tgt + a.geo_off[it.x];
  const int lane = threadIdx.x & 31;
#if ENERGY_NEXT
  // nxt[i]: the first flagged tile >= i (nt: none), by warp 0 from the back
  // in 32-tile chunks, so next() is one shared-memory read, not a scan
  __shared__ uint16_t nxt[DENSE_MAX_TILES];
  const int nt = it.z - it.y;
  if (threadIdx.x < 32) {
    int carry = nt;
    for (int base = ((nt - 1) / 32) * 32; base >= 0; base -= 32) {
      const int i = base + lane;
      const unsigned m = __ballot_sync(0xffffffffu, i < nt && tflag[i] != 0);
      const unsigned hi = m >> lane;  // flagged tiles >= i in this chunk
      if (i < nt) nxt[i] = (uint16_t)(hi ? i + __ffs(hi) - 1 : carry);
      carry = m ? base + __ffs(m) - 1 : carry;
    }
  }
  __syncthreads();
  auto next = [&](int t) { return t < it.z ? it.y + (int)nxt[t - it.y] : it.z; };
#else
  auto next = [&](int t) {
    while (t < it.z && !tflag[t - it.y]) ++t;  // nothing frozen in skipped tiles
    return t;
  };
#endif
  double acc[2] = {0.0, 0.0};
  // ENERGY_ILP flagged tiles at once, each stage's loads of all of them in
  // flight together (the pass is bound by its dependent-load chain); the
  // frozen-set words of the next group are loaded one group ahead
  auto fetch = [&](int t0_, int (&tt_)[ENERGY_ILP], uint32_t (&wb_)[ENERGY_ILP],
                   int (&tg_)[ENERGY_ILP]) {
    tt_[0] = t0_;
#pragma unroll
    for (int k = 1; k < ENERGY_ILP; ++k) tt_[k] = tt_[k - 1] < it.z ? next(tt_[k - 1] + 1) : it.z;
#pragma unroll
    for (int k = 0; k < ENERGY_ILP; ++k) {
      const bool ok = tt_[k] < it.z;
      const int m = (ok ? tt_[k] : it.y) * 256 + threadIdx.x;
      wb_[k] = ok && a.do_photo ? pmask[m >> 5] : 0u;
      tg_[k] = ok && a.do_geo ? (int)gtgt[m] : 0xFFFF;
    }
    return tt_[ENERGY_ILP - 1] < it.z ? next(tt_[ENERGY_ILP - 1] + 1) : it.z;
  };
  int tt[ENERGY_ILP];
  uint32_t wb[ENERGY_ILP];
  int tg[ENERGY_ILP];
  int t0 = fetch(next(it.y), tt, wb, tg);
  for (; tt[0] < it.z;) {
#if ENERGY_PF
    int ttn[ENERGY_ILP];
    uint32_t wbn[ENERGY_ILP];
    int tgn[ENERGY_ILP];
    const int t0n = fetch(t0, ttn, wbn, tgn);
#endif
    bool ph[ENERGY_ILP], ge[ENERGY_ILP];
    bool any = false;
#pragma unroll
    for (int k = 0; k < ENERGY_ILP; ++k) {
      ph[k] = (wb[k] >> lane) & 1u;
      ge[k] = tg[k] != 0xFFFF;
      any |= ph[k] || ge[k];
    }
    if (__any_sync(0xffffffffu, any)) {  // warp-uniform
    float4 P[ENERGY_ILP], N[ENERGY_ILP], PP[ENERGY_ILP];
    float2 G[ENERGY_ILP];
#pragma unroll
    for (int k = 0; k < ENERGY_ILP; ++k) {
      const int t = tt[k] < it.z ? tt[k] : it.y;
      const int p = ((t / stx) * SFB_TILE + (threadIdx.x / SFB_TILE)) * swi + (t % stx) * SFB_TILE +
                    (threadIdx.x & (SFB_TILE - 1));
      const int pc = (ph[k] || ge[k]) ? p : 0;  // inactive lanes: a safe index
      P[k] = __ldg(&sPi[pc]);
      N[k] = __ldg(&sNi[ge[k] ? pc : 0]);
      PP[k] = __ldg(&Fj.P[ge[k] ? tg[k] : 0]);
      G[k] = __ldg(&sGi[ph[k] ? pc : 0]);
    }
    double ua[ENERGY_ILP], va[ENERGY_ILP];
#pragma unroll
    for (int k = 0; k < ENERGY_ILP; ++k) {
      const double d0 = P[k].x, d1 = P[k].y, d2 = P[k].z;
      const double q0 = __dadd_rn(__fma_rn(d2, rel.R[2], __fma_rn(d1, rel.R[1], __dmul_rn(d0, rel.R[0]))), rel.t[0]);
      const double q1 = __dadd_rn(__fma_rn(d2, rel.R[5], __fma_rn(d1, rel.R[4], __dmul_rn(d0, rel.R[3]))), rel.t[1]);
      const double q2 = __dadd_rn(__fma_rn(d2, rel.R[8], __fma_rn(d1, rel.R[7], __dmul_rn(d0, rel.R[6]))), rel.t[2]);
      const double n0 = N[k].x, n1 = N[k].y, n2 = N[k].z;
      const double nr0 = __fma_rn(n2, rel.R[2], __fma_rn(n1, rel.R[1], __dmul_rn(n0, rel.R[0])));
      const double nr1 = __fma_rn(n2, rel.R[5], __fma_rn(n1, rel.R[4], __dmul_rn(n0, rel.R[3])));
      const double nr2 = __fma_rn(n2, rel.R[8], __fma_rn(n1, rel.R[7], __dmul_rn(n0, rel.R[6])));
      const double r = nr0 * (q0 - (double)PP[k].x) + nr1 * (q1 - (double)PP[k].y) + nr2 * (q2 - (double)PP[k].z);
      acc[1] += ge[k] ? r * r : 0.0;
      const double z = q2 > 0.0 ? q2 : 1.0;
      const double rz = rcp_depth(z);
      ua[k] = ph[k] ? fma(__dmul_rn(Fj.fx, q0), rz, Fj.cx) : 0.0;
      va[k] = ph[k] ? fma(__dmul_rn(Fj.fy, q1), rz, Fj.cy) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < ENERGY_ILP; ++k) {
      double val[2];
      bilinear_val2_fast(Fj, ua[k], va[k], val);
      const double r0 = (double)G[k].x - val[0], r1 = (double)G[k].y - val[1];
      acc[0] += ph[k] ? r0 * r0 + r1 * r1 : 0.0;
    }
    }
#if ENERGY_PF
#pragma unroll
    for (int k = 0; k < ENERGY_ILP; ++k) {
      tt[k] = ttn[k];
      wb[k] = wbn[k];
      tg[k] = tgn[k];
    }
    t0 = t0n;
#else
    t0 = fetch(t0, tt, wb, tg);
#endif
  }
  block_reduce_store<2>(acc, item_e2 + 2 * (int64_t)blockIdx.x);
}

void launch_dense_energy(const DenseArgs& a, double* item_e2, cudaStream_t s) {
  if (a.n_items <= 0) return;
  sfb_count_launch();
  k_edge_rel<<<(a.n_dir + 127) / 128, 128, 0, s>>>(a.dir_edges, a.poses, a.rd, a.n_dir, a.edge_rel);
  sfb_count_launch();
  k_dense_energy<<<a.n_items, DENSE_THREADS, 0, s>>>(a, item_e2);
}

// Sum each directed edge's tiles in tile order (one warp per edge, lane =
// slot), then map the camera-j accumulators to the pose increments:
// H_e = M_j K M_j^T, g_e = M_j k with M_j = [[R_j, -[t_j]x R_j], [0, -R_j]]
// (both dense terms' J_i = M_j v, see k_dense_fused).
// Peer-memory exchange (sharded runs, sfb_set_p2p): each owned edge's sums
// are also stored straight into every peer's edge_out (P2P over NVLink) by
// the warp that computes them - the all-gather fused into the reduction.
struct EdgePeers {
  double* const* dst;  // world pointers (own rank's entry unused), or null
  int rank, world;
};

__global__ void k_edge_reduce(const int* edge_item_ptr, const double* item_out, double* edge_out,
                              int n_dir, const int2* dir_edges, const PoseDev* poses,
                              EdgePeers peers) {
  __shared__ double sK[8][36], sM[8][36], sW[8][36], sk[8][6];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int wl = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_dir) return;
  double s = 0.0;
  for (int i = edge_item_ptr[warp]; i < edge_item_ptr[warp + 1]; ++i)
    s += item_out[(int64_t)i * SFB_ITEM_STRIDE + lane];
  double* out = edge_out + (int64_t)warp * SFB_ITEM_STRIDE;
  double val = s;  // lanes >= 27: energies pass through
  // unpack K (packed upper triangle) and k into shared memory
  for (int r = 0; r < 6; ++r)
    for (int c = r; c < 6; ++c)
      if (lane == sym6(r, c)) sK[wl][r * 6 + c] = sK[wl][c * 6 + r] = s;
  if (lane >= 21 && lane < 27) sk[wl][lane - 21] = s;
  // M_j = [[R, -[t]x R], [0, -R]], one or two entries per lane
  {
    const PoseDev& Pj = poses[dir_edges[warp].y];
    const double* R = Pj.R;
    const double* t = Pj.t;
    for (int e = lane; e < 36; e += 32) {
      const int r = e / 6, c = e % 6;
      double m = 0.0;
      if (r < 3 && c < 3) {
        m = R[r * 3 + c];
      } else if (r < 3) {
        // row r of [t]x = {{0, -t2, t1}, {t2, 0, -t0}, {-t1, t0, 0}}
        const double a0 = r == 0 ? 0.0 : (r == 1 ? t[2] : -t[1]);
        const double a1 = r == 0 ? -t[2] : (r == 1 ? 0.0 : t[0]);
        const double a2 = r == 0 ? t[1] : (r == 1 ? -t[0] : 0.0);
        double tr = 0.0;
        tr += a0 * R[c - 3];
        tr += a1 * R[3 + (c - 3)];
        tr += a2 * R[6 + (c - 3)];
        m = -tr;
      } else if (c >= 3) {
        m = -R[(r - 3) * 3 + (c - 3)];
      }
      sM[wl][e] = m;
    }
  }
  __syncwarp();
  // W = K M^T (W[k][c] = sum_l K[k][l] M[c][l]), one or two entries per lane,
  // then H = M W: two 6-long chains per entry instead of one 42-long one
  for (int e = lane; e < 36; e += 32) {
    const int k = e / 6, c = e % 6;
    double mk = 0.0;
    for (int l = 0; l < 6; ++l) mk += sK[wl][k * 6 + l] * sM[wl][c * 6 + l];
    sW[wl][e] = mk;
  }
  __syncwarp();
  if (lane < 21) {
    int r = 0, c = lane;
    while (c >= 6 - r) { c -= 6 - r; ++r; }  // packed index -> (r, c >= r)
    c += r;
    double h = 0.0;
    for (int k = 0; k < 6; ++k) h += sM[wl][r * 6 + k] * sW[wl][k * 6 + c];
    val = h;
  } else if (lane < 27) {
    const int r = lane - 21;
    double g = 0.0;
    for (int k = 0; k < 6; ++k) g += sM[wl][r * 6 + k] * sk[wl][k];
    val = g;
  }
  if (peers.dst == nullptr) {
    out[lane] = val;
  } else if (warp % peers.world == peers.rank) {  // owned edge: local row + every peer's
    out[lane] = val;
    for (int r = 0; r < peers.world; ++r)
      if (r != peers.rank) peers.dst[r][(int64_t)warp * SFB_ITEM_STRIDE + lane] = val;
  }  // (other rows arrive from their owners: writing zeros here would race them)
}

// Cross-rank barrier over peer memory after the pushes: fence (system scope),
// publish this rank's epoch in every peer's flag slot, wait for every peer's.
__global__ void k_p2p_sync(unsigned* const* peer_flags, unsigned* my_flags, int rank, int world,
                           unsigned epoch) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int r = 0; r < world; ++r)
    if (r != rank)
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peer_flags[r] + rank), "r"(epoch) : "memory");
  for (int r = 0; r < world; ++r) {
    if (r == rank) continue;
    unsigned v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(my_flags + r) : "memory");
    } while (v < epoch);
  }
}

void launch_p2p_sync(unsigned* const* peer_flags, unsigned* my_flags, int rank, int world,
                     unsigned epoch, cudaStream_t s) {
  sfb_count_launch();
  k_p2p_sync<<<1, 32, 0, s>>>(peer_flags, my_flags, rank, world, epoch);
}

void launch_edge_reduce(const int* edge_item_ptr, const double* item_out, double* edge_out,
                        int n_dir, const int2* dir_edges, const PoseDev* poses, cudaStream_t s,
                        double* const* peer_dst, int rank, int world) {
  if (n_dir <= 0) return;
  sfb_count_launch();
  k_edge_reduce<<<(n_dir * 32 + 255) / 256, 256, 0, s>>>(edge_item_ptr, item_out, edge_out, n_dir,
                                                         dir_edges, poses,
                                                         EdgePeers{peer_dst, rank, world});
}

// Frozen-energy item pairs -> per-edge pairs (zero for edges without items).
__global__ void k_edge_reduce2(const int* edge_item_ptr, const double* item_e2, double* edge_e2,
                               int n_dir) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n_dir) return;
  double a = 0.0, b = 0.0;
  for (int i = edge_item_ptr[d]; i < edge_item_ptr[d + 1]; ++i) {
    a += item_e2[2 * (int64_t)i];
    b += item_e2[2 * (int64_t)i + 1];
  }
  edge_e2[2 * (int64_t)d] = a;
  edge_e2[2 * (int64_t)d + 1] = b;
}

void launch_edge_reduce2(const int* edge_item_ptr, const double* item_e2, double* edge_e2, int n_dir,
                         cudaStream_t s) {
  if (n_dir <= 0) return;
  sfb_count_launch();
  k_edge_reduce2<<<(n_dir + 255) / 256, 256, 0, s>>>(edge_item_ptr, item_e2, edge_e2, n_dir);
}

// ---------------------------------------------------------------------------
// Block-system assembly.  Contribution entries: (id << 3) | kind.
//  D/g lists (per var):   0 set H_ii / g_i   1 set H_jj / g_j
//                         2 set H_ij (+H_ij^T, self-set only)   4 dense +H / +g
//                         5 dense +H / -g
//  B lists (per pair):    0 set +H_ij   1 set +H_ij^T   4 dense -H
__device__ __forceinline__ double sym_full(const double* h, int r, int c) { return h[sym6(r, c)]; }

// Diagonal rows: one CTA of ASM_DIAG_WARPS warps per block row; warp w sums
// the contributions w, w + W, ... of the row's list in list order, 8 loads in
// flight, and the warps' partials are added in warp order (deterministic).
// Pair blocks: one warp per pair (short lists).
#define ASM_DIAG_WARPS 4
#define ASM_BATCH 8
__global__ void __launch_bounds__(ASM_DIAG_WARPS * 32) k_assemble(AssembleArgs a) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if ((int)blockIdx.x < a.n_blk) {
    __shared__ double sd[ASM_DIAG_WARPS][3][32];
    const int v = blockIdx.x;
    double d0 = 0.0, d1 = 0.0, gv = 0.0;
    const int e0 = lane, e1 = lane + 32;  // matrix entries handled by this lane
    // one contribution's (diagonal entry pair, gradient entry); loads only,
    // so a batch of them is in flight before the in-order accumulation below
    auto fetch = [&](int ent, double& x0, double& x1, double& xg) {
      const int kind = ent & 7, id = ent >> 3;
      x0 = 0.0;
      x1 = 0.0;
      xg = 0.0;
      if (kind <= 2) {
        const double* so = a.set_out + (int64_t)id * SFB_SET_STRIDE;
        if (kind == 2) {  // self-set: H_ij + H_ij^T (both cross blocks land on the diagonal)
          const double* h = so + 72;
          x0 = h[e0] + h[(e0 % 6) * 6 + e0 / 6];
          if (e1 < 36) x1 = h[e1] + h[(e1 % 6) * 6 + e1 / 6];
        } else {
          const double* h = so + (kind == 0 ? 0 : 36);
          x0 = h[e0];
          if (e1 < 36) x1 = h[e1];
          if (lane < 6) xg = so[(kind == 0 ? SFB_SET_GI : SFB_SET_GJ) + lane];
        }
      } else if (a.dense_on) {
        const double* eo = a.edge_out + (int64_t)id * SFB_ITEM_STRIDE;
        x0 = sym_full(eo, e0 / 6, e0 % 6);
        if (e1 < 36) x1 = sym_full(eo, e1 / 6, e1 % 6);
        if (lane < 6) xg = (kind == 4 ? 1.0 : -1.0) * eo[21 + lane];
      }
    };
    const int k0 = a.d_ptr[v], k1 = a.d_ptr[v + 1];
    constexpr int SPAN = 32 * ASM_DIAG_WARPS;
    for (int kb = k0; kb < k1; kb += SPAN) {
      // this warp's entries of the span: kb + wid + W * j, j < 32
      const int kl = kb + wid + ASM_DIAG_WARPS * lane;
      const int ent_l = kl < k1 ? a.d_ent[kl] : 0;
      const int nk = max(0, min(32, (k1 - kb - wid + ASM_DIAG_WARPS - 1) / ASM_DIAG_WARPS));
      int j = 0;
      for (; j + ASM_BATCH <= nk; j += ASM_BATCH) {
        double x0[ASM_BATCH], x1[ASM_BATCH], xg[ASM_BATCH];
#pragma unroll
        for (int u = 0; u < ASM_BATCH; ++u) fetch(__shfl_sync(0xffffffffu, ent_l, j + u), x0[u], x1[u], xg[u]);
#pragma unroll
        for (int u = 0; u < ASM_BATCH; ++u) {  // list order within the warp
          d0 += x0[u];
          d1 += x1[u];
          gv += xg[u];
        }
      }
      for (; j < nk; ++j) {
        double x0, x1, xg;
        fetch(__shfl_sync(0xffffffffu, ent_l, j), x0, x1, xg);
        d0 += x0;
        d1 += x1;
        gv += xg;
      }
    }
    sd[wid][0][lane] = d0;
    sd[wid][1][lane] = d1;
    sd[wid][2][lane] = gv;
    __syncthreads();
    if (wid == 0) {
      d0 = sd[0][0][lane];
      d1 = sd[0][1][lane];
      gv = sd[0][2][lane];
#pragma unroll
      for (int w = 1; w < ASM_DIAG_WARPS; ++w) {
        d0 += sd[w][0][lane];
        d1 += sd[w][1][lane];
        gv += sd[w][2][lane];
      }
      double* D = a.D + (int64_t)v * 36;
      double* S = a.Brow + (int64_t)a.row_ptr[v] * 36;
      D[e0] = d0;
      S[e0] = d0;
      if (e1 < 36) {
        D[e1] = d1;
        S[e1] = d1;
      }
      if (lane < 6) a.g[v * 6 + lane] = gv;
      if (a.jdiag) {
        // _jacobi_diagonal (solver.py:412-428): D's diagonal without the
        // H_ij + H_ij^T cross term of a set whose two frames coincide,
        // subtracted in list order (the arithmetic of the former separate pass)
        const bool dl = (lane % 7 == 0 && lane < 35) || lane == 3;  // entries 0,7,..,28 (d0) and 35 (d1)
        const int c = lane == 3 ? 5 : lane / 7;
        double jd = lane == 3 ? d1 : d0;
        for (int kb = k0; kb < k1; kb += 32) {
          const int ent = kb + lane < k1 ? a.d_ent[kb + lane] : 0;
          unsigned m = __ballot_sync(0xffffffffu, kb + lane < k1 && (ent & 7) == 2);
          while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            const int id = __shfl_sync(0xffffffffu, ent, j) >> 3;
            if (dl) jd -= 2.0 * a.set_out[(int64_t)id * SFB_SET_STRIDE + 72 + c * 7];
          }
        }
        if (dl) a.jdiag[v * 6 + c] = jd;
      }
    }
  } else {
    const int q = ((int)blockIdx.x - a.n_blk) * ASM_DIAG_WARPS + wid;
    if (q >= a.n_pairs) return;
    double b0 = 0.0, b1 = 0.0;
    const int e0 = lane, e1 = lane + 32;
    for (int k = a.b_ptr[q]; k < a.b_ptr[q + 1]; ++k) {
      const int ent = a.b_ent[k];
      const int kind = ent & 7, id = ent >> 3;
      if (kind <= 1) {
        const double* h = a.set_out + (int64_t)id * SFB_SET_STRIDE + 72;
        if (kind == 0) {
          b0 += h[e0];
          if (e1 < 36) b1 += h[e1];
        } else {
          b0 += h[(e0 % 6) * 6 + e0 / 6];
          if (e1 < 36) b1 += h[(e1 % 6) * 6 + e1 / 6];
        }
      } else if (a.dense_on) {
        const double* eo = a.edge_out + (int64_t)id * SFB_ITEM_STRIDE;
        b0 -= sym_full(eo, e0 / 6, e0 % 6);
        if (e1 < 36) b1 -= sym_full(eo, e1 / 6, e1 % 6);
      }
    }
    double* B = a.B + (int64_t)q * 36;
    double* Sa = a.Brow + (int64_t)a.pair_slot[2 * q] * 36;      // row a: as is
    double* Sb = a.Brow + (int64_t)a.pair_slot[2 * q + 1] * 36;  // row b: transposed
    B[e0] = b0;
    Sa[e0] = b0;
    Sb[(e0 % 6) * 6 + e0 / 6] = b0;
    if (e1 < 36) {
      B[e1] = b1;
      Sa[e1] = b1;
      Sb[(e1 % 6) * 6 + e1 / 6] = b1;
    }
  }
}

void launch_assemble(const AssembleArgs& a, cudaStream_t s) {
  const int blocks = a.n_blk + (a.n_pairs + ASM_DIAG_WARPS - 1) / ASM_DIAG_WARPS;
  if (blocks <= 0) return;
  sfb_count_launch();
  k_assemble<<<blocks, ASM_DIAG_WARPS * 32, 0, s>>>(a);
}

// Deterministic sums of the per-set / per-edge / per-item energies.
// mode 0: out = {sum set E, sum edge e_photo, sum edge e_geo, sum edge prev
//                e_photo, sum edge prev e_geo}
// mode 1: out = {sum set E, sum item_e2[2i], sum item_e2[2i+1]}
// SUM_CTAS CTAs each sum a fixed contiguous chunk (thread order, then a fixed
// butterfly and warp order) into scratch[cta]; the last CTA to finish (ticket
// counter in scratch, reset by it) adds the CTA partials in CTA order.
#define SUM_CTAS 32
#define SUM_THREADS 256
__global__ void __launch_bounds__(SUM_THREADS) k_sum_energies(const double* set_out, int n_sets,
                                                           const double* edge_out, int n_dir,
                                                           const double* item_e2, int n_items,
                                                           double* out3, int mode, double* scratch) {
  __shared__ double sh[5][SUM_THREADS / 32];
  __shared__ bool last;
  double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int G = gridDim.x, b = blockIdx.x, bd = blockDim.x;
  {
    const int c0 = (int)((int64_t)n_sets * b / G), c1 = (int)((int64_t)n_sets * (b + 1) / G);
    for (int i = c0 + threadIdx.x; i < c1; i += bd) s[0] += set_out[(int64_t)i * SFB_SET_STRIDE + SFB_SET_E];
  }
  if (mode == 0) {
    const int c0 = (int)((int64_t)n_dir * b / G), c1 = (int)((int64_t)n_dir * (b + 1) / G);
    for (int i = c0 + threadIdx.x; i < c1; i += bd) {
      const double* e = edge_out + (int64_t)i * SFB_ITEM_STRIDE;
      s[1] += e[SFB_ITEM_EP];
      s[2] += e[SFB_ITEM_EG];
      s[3] += e[SFB_ITEM_PP];
      s[4] += e[SFB_ITEM_PG];
    }
  } else {
    const int c0 = (int)((int64_t)n_items * b / G), c1 = (int)((int64_t)n_items * (b + 1) / G);
    for (int i = c0 + threadIdx.x; i < c1; i += bd) {
      const double2 v = reinterpret_cast<const double2*>(item_e2)[i];
      s[1] += v.x;
      s[2] += v.y;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const double v = warp_sum(s[k]);
    if (lane == 0) sh[k][warp] = v;
  }
  __syncthreads();
  unsigned* ticket = reinterpret_cast<unsigned*>(scratch + 5 * SUM_CTAS);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      double t = 0.0;
      for (int w = 0; w < SUM_THREADS / 32; ++w) t += sh[k][w];
      scratch[5 * b + k] = t;
    }
    __threadfence();
    last = atomicAdd(ticket, 1u) == (unsigned)(G - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 5) {
    const int k = threadIdx.x;
    double t = 0.0;
    for (int c = 0; c < G; ++c) t += __ldcg(&scratch[5 * c + k]);
    if (mode == 0 || k < 3) out3[k] = t;
  }
  if (threadIdx.x == 0) *ticket = 0u;  // next launch (stream-ordered)
}

void launch_sum_energies(const double* set_out, int n_sets, const double* edge_out, int n_dir,
                         const double* item_e2, int n_items, double* out3, int mode,
                         double* scratch, cudaStream_t s) {
  sfb_count_launch();
  k_sum_energies<<<SUM_CTAS, SUM_THREADS, 0, s>>>(set_out, n_sets, edge_out, n_dir, item_e2, n_items,
                                                  out3, mode, scratch);
}

// ---------------------------------------------------------------------------
// API evaluators.
__global__ void k_associate(DenseArgs a, int src, int dst, int kind, uint8_t* sel, int* tgt) {
  __shared__ EdgeCtx ec;
  if (threadIdx.x == 0) load_edge_ctx(&ec, a.poses[src], a.poses[dst], a.rd);
  const FrameDev Fi = a.frames[src];
  const FrameDev Fj = a.frames[dst];
  __syncthreads();
  const int hw = Fi.w * Fi.h;
  const int2 nsrc = src_counts(a, Fi, src);
  const int ord_ph = (nsrc.x == 1) ? a.rd.apply_1 : a.rd.apply_n;
  const int ord_ge = (nsrc.y == 1) ? a.rd.apply_1 : a.rd.apply_n;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < hw; p += gridDim.x * blockDim.x) {
    const float4 P = Fi.P[p];
    const unsigned fl = __float_as_uint(P.w);
    const bool sok = stride_ok(p, Fi.w, a.stride);
    const bool ph = kind == 0 && sok && (fl & SFB_FLAG_VD);
    const bool ge = kind == 1 && sok && (fl & SFB_FLAG_VD) && (fl & SFB_FLAG_VN);
    const float4 N = ge ? Fi.N[p] : make_float4(0.f, 0.f, 0.f, 0.f);
    const AssocOut ao = associate_pixel(ec, Fj, P, N, ph, ge, ord_ph, ord_ge, a.rd, a.geo_dmax,
                                        a.geo_nmin);
    sel[p] = kind == 0 ? (uint8_t)ao.photo : (uint8_t)(ao.tgt >= 0);
    tgt[p] = ao.tgt;
  }
}

void launch_associate(const DenseArgs& a, int src, int dst, int kind, uint8_t* sel, int* tgt,
                      cudaStream_t s) {
  sfb_count_launch();
  k_associate<<<148, 256, 0, s>>>(a, src, dst, kind, sel, tgt);
}

__global__ void k_point_eval(const FrameDev* frames, const PoseDev* poses, int src, int dst,
                             int kind, int64_t m, const double* pts, const double* aux,
                             const double* tgts, double* res, double* jac) {
  __shared__ EdgeCtx ec;
  const Rounding rd{0, 0, 0, 0, 0, 0};
  if (threadIdx.x == 0) load_edge_ctx(&ec, poses[src], poses[dst], rd);
  const FrameDev Fj = frames[dst];
  __syncthreads();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double d0 = pts[3 * k], d1 = pts[3 * k + 1], d2 = pts[3 * k + 2];
    if (kind == 0) {
      double r[2], J[2][6];
      photo_lin_pixel(ec, Fj, d0, d1, d2, aux[2 * k], aux[2 * k + 1], r, J);
      res[2 * k] = r[0];
      res[2 * k + 1] = r[1];
      if (jac)
        for (int c = 0; c < 2; ++c)
          for (int j = 0; j < 6; ++j) jac[12 * k + 6 * c + j] = J[c][j];
    } else {
      double r, J[6];
      geo_lin_pixel(ec, d0, d1, d2, aux[3 * k], aux[3 * k + 1], aux[3 * k + 2], tgts[3 * k],
                    tgts[3 * k + 1], tgts[3 * k + 2], &r, J);
      res[k] = r;
      if (jac)
        for (int j = 0; j < 6; ++j) jac[6 * k + j] = J[j];
    }
  }
}

void launch_point_eval(const FrameDev* frames, const PoseDev* poses, int src, int dst, int kind,
                       int64_t m, const double* pts, const double* aux, const double* tgts,
                       double* res, double* jac, cudaStream_t s) {
  if (m <= 0) return;
  int blocks = (int)((m + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  sfb_count_launch();
  k_point_eval<<<blocks, 256, 0, s>>>(frames, poses, src, dst, kind, m, pts, aux, tgts, res, jac);
}
