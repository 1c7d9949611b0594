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

__device__ __forceinline__ void accum_row(double (&acc)[29], const double J[6], double res,
                                          double s) {
  double sJ[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) sJ[k] = s * J[k];
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = r; c < 6; ++c) acc[sym6(r, c)] = fma(sJ[r], J[c], acc[sym6(r, c)]);
#pragma unroll
  for (int k = 0; k < 6; ++k) acc[21 + k] = fma(sJ[k], res, acc[21 + k]);
}

__device__ __forceinline__ bool stride_ok(int p, int w, int stride) {
  if (stride <= 1) return true;
  const int y = p / w, x = p - y * w;
  return (y % stride) == 0 && (x % stride) == 0;
}

__global__ void __launch_bounds__(DENSE_THREADS, 2) k_dense_linearize(DenseArgs a) {
  __shared__ EdgeCtx ec;
  const int4 it = a.items[blockIdx.x];
  const int2 de = a.dir_edges[it.x];
  if (threadIdx.x == 0) load_edge_ctx(&ec, a.poses[de.x], a.poses[de.y], a.rd);
  const FrameDev Fi = a.frames[de.x];
  const FrameDev Fj = a.frames[de.y];
  __syncthreads();
  const int ord_ph = (Fi.n_valid_depth == 1) ? a.rd.apply_1 : a.rd.apply_n;
  const int ord_ge = (Fi.n_valid_geo == 1) ? a.rd.apply_1 : a.rd.apply_n;
  const int lane = threadIdx.x & 31;
  uint32_t* pmask = a.photo_mask + a.photo_off[it.x];
  uint16_t* gtgt = a.geo_tgt + a.geo_off[it.x];

  double acc[29];
#pragma unroll
  for (int k = 0; k < 29; ++k) acc[k] = 0.0;

  for (int base = it.y; base < it.z; base += DENSE_THREADS) {
    const int p = base + threadIdx.x;
    const bool live = p < it.z;
    float4 P = make_float4(0.f, 0.f, 0.f, 0.f), N = P;
    unsigned fl = 0;
    if (live) {
      P = __ldg(&Fi.P[p]);
      fl = __float_as_uint(P.w);
    }
    const bool sok = live && stride_ok(p, Fi.w, a.stride);
    const bool ph = a.do_photo && sok && (fl & SFB_FLAG_VD);
    const bool ge = a.do_geo && sok && (fl & SFB_FLAG_VD) && (fl & SFB_FLAG_VN);
    if (ge) N = __ldg(&Fi.N[p]);
    const AssocOut ao = associate_pixel(ec, Fj, P, N, ph, ge, ord_ph, ord_ge, a.rd, a.geo_dmax,
                                        a.geo_nmin);
    if (a.do_photo) {
      const unsigned word = __ballot_sync(0xffffffffu, ao.photo);
      if (lane == 0 && base + (threadIdx.x & ~31) < it.z) pmask[(p - lane) >> 5] = word;
    }
    if (a.do_geo && live) gtgt[p] = ao.tgt >= 0 ? (uint16_t)ao.tgt : (uint16_t)0xFFFF;
    if (ao.photo) {
      const float2 ref = __ldg(&Fi.G[p]);
      double res[2], J[2][6];
      photo_lin_pixel(ec, Fj, P.x, P.y, P.z, ref.x, ref.y, res, J);
      accum_row(acc, J[0], res[0], a.s_photo);
      accum_row(acc, J[1], res[1], a.s_photo);
      acc[27] += res[0] * res[0] + res[1] * res[1];
    }
    if (ao.tgt >= 0) {
      const float4 PT = __ldg(&Fj.P[ao.tgt]);
      double res, J[6];
      geo_lin_pixel(ec, P.x, P.y, P.z, N.x, N.y, N.z, PT.x, PT.y, PT.z, &res, J);
      accum_row(acc, J, res, a.s_geo);
      acc[28] += res * res;
    }
  }
  block_reduce_store<29>(acc, a.item_out + (int64_t)blockIdx.x * SFB_ITEM_STRIDE);
}

void launch_dense_linearize(const DenseArgs& a, cudaStream_t s) {
  if (a.n_items <= 0) return;
  sfb_count_launch();
  k_dense_linearize<<<a.n_items, DENSE_THREADS, 0, s>>>(a);
}

// Frozen-association energy at the current poses.
__global__ void __launch_bounds__(DENSE_THREADS) k_dense_energy(DenseArgs a, double* item_e2) {
  __shared__ double sh[12 * 2];  // rel (photo) and back (geo), plain
  const int4 it = a.items[blockIdx.x];
  const int2 de = a.dir_edges[it.x];
  if (threadIdx.x == 0) {
    const PoseDev& Pi = a.poses[de.x];
    const PoseDev& Pj = a.poses[de.y];
    double iR[9], itt[3];
    // relative = pose_j^-1 o pose_i (solver.py:267); back = pose_i^-1 o pose_j (:281)
    xf_inverse_plain(Pj.R, Pj.t, iR, itt);
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c)
        sh[r * 3 + c] = iR[r * 3 + 0] * Pi.R[0 * 3 + c] + iR[r * 3 + 1] * Pi.R[1 * 3 + c] + iR[r * 3 + 2] * Pi.R[2 * 3 + c];
      sh[9 + r] = iR[r * 3 + 0] * Pi.t[0] + iR[r * 3 + 1] * Pi.t[1] + iR[r * 3 + 2] * Pi.t[2] + itt[r];
    }
    xf_inverse_plain(Pi.R, Pi.t, iR, itt);
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c)
        sh[12 + r * 3 + c] = iR[r * 3 + 0] * Pj.R[0 * 3 + c] + iR[r * 3 + 1] * Pj.R[1 * 3 + c] + iR[r * 3 + 2] * Pj.R[2 * 3 + c];
      sh[21 + r] = iR[r * 3 + 0] * Pj.t[0] + iR[r * 3 + 1] * Pj.t[1] + iR[r * 3 + 2] * Pj.t[2] + itt[r];
    }
  }
  const FrameDev Fi = a.frames[de.x];
  const FrameDev Fj = a.frames[de.y];
  __syncthreads();
  const uint32_t* pmask = a.photo_mask + a.photo_off[it.x];
  const uint16_t* gtgt = a.geo_tgt + a.geo_off[it.x];
  double acc[2] = {0.0, 0.0};
  for (int p = it.y + threadIdx.x; p < it.z; p += DENSE_THREADS) {
    const bool ph = a.do_photo && ((pmask[p >> 5] >> (p & 31)) & 1u);
    const int tg = a.do_geo ? (int)gtgt[p] : 0xFFFF;
    if (!ph && tg == 0xFFFF) continue;
    const float4 P = __ldg(&Fi.P[p]);
    if (ph) {
      double q[3];
      xf_apply(sh, sh + 9, P.x, P.y, P.z, q);
      const double zs = q[2] > 0.0 ? q[2] : 1.0;
      const double u = Fj.fx * q[0] / zs + Fj.cx;
      const double v = Fj.fy * q[1] / zs + Fj.cy;
      double val[2], ddx[2], ddy[2];
      bilinear_grad2(Fj, u, v, val, ddx, ddy);
      const float2 ref = __ldg(&Fi.G[p]);
      const double r0 = (double)ref.x - val[0], r1 = (double)ref.y - val[1];
      acc[0] += r0 * r0 + r1 * r1;
    }
    if (tg != 0xFFFF) {
      const float4 N = __ldg(&Fi.N[p]);
      const float4 PT = __ldg(&Fj.P[tg]);
      double mp[3];
      xf_apply(sh + 12, sh + 21, PT.x, PT.y, PT.z, mp);
      const double r = (double)N.x * ((double)P.x - mp[0]) + (double)N.y * ((double)P.y - mp[1]) +
                       (double)N.z * ((double)P.z - mp[2]);
      acc[1] += r * r;
    }
  }
  block_reduce_store<2>(acc, item_e2 + 2 * (int64_t)blockIdx.x);
}

void launch_dense_energy(const DenseArgs& a, double* item_e2, cudaStream_t s) {
  if (a.n_items <= 0) return;
  sfb_count_launch();
  k_dense_energy<<<a.n_items, DENSE_THREADS, 0, s>>>(a, item_e2);
}

// Sum each directed edge's tiles in tile order (one warp per edge, lane = slot).
__global__ void k_edge_reduce(const int* edge_item_ptr, const double* item_out, double* edge_out,
                              int n_dir) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_dir) return;
  double s = 0.0;
  for (int i = edge_item_ptr[warp]; i < edge_item_ptr[warp + 1]; ++i)
    s += item_out[(int64_t)i * SFB_ITEM_STRIDE + lane];
  edge_out[(int64_t)warp * SFB_ITEM_STRIDE + lane] = s;
}

void launch_edge_reduce(const int* edge_item_ptr, const double* item_out, double* edge_out,
                        int n_dir, cudaStream_t s) {
  if (n_dir <= 0) return;
  sfb_count_launch();
  k_edge_reduce<<<(n_dir * 32 + 255) / 256, 256, 0, s>>>(edge_item_ptr, item_out, edge_out, n_dir);
}

// ---------------------------------------------------------------------------
// Block-system assembly.  Contribution entries: (id << 3) | kind.
//  D/g lists (per var):   0 set H_ii / g_i   1 set H_jj / g_j
//                         2 set H_ij (+H_ij^T, self-set only)   4 dense +H / +g
//                         5 dense +H / -g
//  B lists (per pair):    0 set +H_ij   1 set +H_ij^T   4 dense -H
__device__ __forceinline__ double sym_full(const double* h, int r, int c) { return h[sym6(r, c)]; }

__global__ void k_assemble(AssembleArgs a) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp < a.n_blk) {
    const int v = warp;
    double d0 = 0.0, d1 = 0.0, gv = 0.0;
    const int e0 = lane, e1 = lane + 32;  // matrix entries handled by this lane
    for (int k = a.d_ptr[v]; k < a.d_ptr[v + 1]; ++k) {
      const int ent = a.d_ent[k];
      const int kind = ent & 7, id = ent >> 3;
      if (kind <= 2) {
        const double* so = a.set_out + (int64_t)id * SFB_SET_STRIDE;
        if (kind == 2) {  // self-set: H_ij + H_ij^T (both cross blocks land on the diagonal)
          const double* h = so + 72;
          d0 += h[e0] + h[(e0 % 6) * 6 + e0 / 6];
          if (e1 < 36) d1 += h[e1] + h[(e1 % 6) * 6 + e1 / 6];
        } else {
          const double* h = so + (kind == 0 ? 0 : 36);
          d0 += h[e0];
          if (e1 < 36) d1 += h[e1];
          if (lane < 6) gv += so[(kind == 0 ? SFB_SET_GI : SFB_SET_GJ) + lane];
        }
      } else if (a.dense_on) {
        const double* eo = a.edge_out + (int64_t)id * SFB_ITEM_STRIDE;
        d0 += sym_full(eo, e0 / 6, e0 % 6);
        if (e1 < 36) d1 += sym_full(eo, e1 / 6, e1 % 6);
        if (lane < 6) gv += (kind == 4 ? 1.0 : -1.0) * eo[21 + lane];
      }
    }
    double* D = a.D + (int64_t)v * 36;
    D[e0] = d0;
    if (e1 < 36) D[e1] = d1;
    if (lane < 6) a.g[v * 6 + lane] = gv;
  } else if (warp < a.n_blk + a.n_pairs) {
    const int q = warp - a.n_blk;
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
    B[e0] = b0;
    if (e1 < 36) B[e1] = b1;
  }
}

void launch_assemble(const AssembleArgs& a, cudaStream_t s) {
  const int warps = a.n_blk + a.n_pairs;
  if (warps <= 0) return;
  sfb_count_launch();
  k_assemble<<<(warps * 32 + 255) / 256, 256, 0, s>>>(a);
}

// Deterministic single-block sums of the per-set / per-edge / per-item energies.
// mode 0: out = {sum set E, sum edge e_photo, sum edge e_geo}
// mode 1: out = {sum set E, sum item_e2[2i], sum item_e2[2i+1]}
__global__ void k_sum_energies(const double* set_out, int n_sets, const double* edge_out,
                               int n_dir, const double* item_e2, int n_items, double* out3,
                               int mode) {
  __shared__ double sh[3][32];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int i = threadIdx.x; i < n_sets; i += blockDim.x) s0 += set_out[(int64_t)i * SFB_SET_STRIDE + SFB_SET_E];
  if (mode == 0) {
    for (int i = threadIdx.x; i < n_dir; i += blockDim.x) {
      s1 += edge_out[(int64_t)i * SFB_ITEM_STRIDE + SFB_ITEM_EP];
      s2 += edge_out[(int64_t)i * SFB_ITEM_STRIDE + SFB_ITEM_EG];
    }
  } else {
    for (int i = threadIdx.x; i < n_items; i += blockDim.x) {
      s1 += item_e2[2 * (int64_t)i];
      s2 += item_e2[2 * (int64_t)i + 1];
    }
  }
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sh[0][warp] = s0; sh[1][warp] = s1; sh[2][warp] = s2; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    double a0 = lane < nw ? sh[0][lane] : 0.0;
    double a1 = lane < nw ? sh[1][lane] : 0.0;
    double a2 = lane < nw ? sh[2][lane] : 0.0;
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    if (lane == 0) { out3[0] = a0; out3[1] = a1; out3[2] = a2; }
  }
}

void launch_sum_energies(const double* set_out, int n_sets, const double* edge_out, int n_dir,
                         const double* item_e2, int n_items, double* out3, int mode,
                         cudaStream_t s) {
  sfb_count_launch();
  k_sum_energies<<<1, 1024, 0, s>>>(set_out, n_sets, edge_out, n_dir, item_e2, n_items, out3, mode);
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
  const int ord_ph = (Fi.n_valid_depth == 1) ? a.rd.apply_1 : a.rd.apply_n;
  const int ord_ge = (Fi.n_valid_geo == 1) ? a.rd.apply_1 : a.rd.apply_n;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < hw; p += gridDim.x * blockDim.x) {
    const float4 P = Fi.P[p];
    const unsigned fl = __float_as_uint(P.w);
    const bool sok = stride_ok(p, Fi.w, a.stride);
    const bool ph = kind == 0 && sok && (fl & SFB_FLAG_VD);
    const bool ge = kind == 1 && sok && (fl & SFB_FLAG_VD) && (fl & SFB_FLAG_VN);
    const float4 N = ge ? Fi.N[p] : make_float4(0.f, 0.f, 0.f, 0.f);
    // a single-pixel stride selection is not tracked here (m == 1 order)
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
