// Frame packing, sparse correspondence term, pose update.
//
//  k_pack_batch     CachedFrame planes (frames.py:38-50) -> P/N/G/T device layout
//  k_sparse         _sparse_state + sparse gradient/diagonal/J^T J blocks
//                   (solver.py:568-580, 389-428, 644-646) and eval_sparse (:114-123)
//  k_pose_update    _apply_step + exp_twist_vector (solver.py:674-677,
//                   geometry.py:40-48,78-90,183-186)
#include "sfb_kernels.cuh"

// ---------------------------------------------------------------------------
// One warp per correspondence set.  Per set we accumulate the moments that
// define the three 6x6 blocks of w_s * J^T J (H_ii, H_jj, H_ij), the two
// gradient 6-vectors and the energy.  With S = -[y]x,
//   H_ii = [[|y_i|^2 I - y_i y_i^T, [y_i]x], [-[y_i]x, I]]  summed over corr,
//   H_ij = [[y_j y_i^T - (y_i.y_j) I, -[y_i]x], [[y_j]x, -I]],
//   g_i  = [y_i x r ; r],  g_j = -[y_j x r ; r]
// which is exactly the matrix-free product of solver.py:375-401 regrouped.
// SPARSE_G lanes per set (a set holds ~20 correspondences at cfg3-5, so a
// whole warp per set left most lanes idle and spent 5 shuffle levels on each
// of the 38 moments): each lane strides over the set's correspondences, the
// moments are summed by a butterfly inside the lane group (every lane holds
// the totals) and the group's lanes share the 121 output writes.
#define SPARSE_G 8
#define SPARSE_NM 38

__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = SPARSE_G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// output entry e of a set (layout: Hii[36] Hjj[36] Hij[36] gi[6] gj[6] E)
// from the summed moments m[]: Ai 0-5, Aj 6-11, M 12-20, Si 21-23, Sj 24-26,
// gi 27-29, gj 30-32, sr 33-35, E 36, cnt 37
__device__ __forceinline__ double sparse_entry(int e, const double* m, double w, double wg) {
  if (e >= SFB_SET_E) return e == SFB_SET_E ? m[36] : 0.0;
  if (e >= SFB_SET_GJ) {
    const int k = e - SFB_SET_GJ;
    return -wg * (k < 3 ? m[30 + k] : m[33 + k - 3]);
  }
  if (e >= SFB_SET_GI) {
    const int k = e - SFB_SET_GI;
    return wg * (k < 3 ? m[27 + k] : m[33 + k - 3]);
  }
  const int blk = e / 36, r = (e % 36) / 6, c = e % 6;
  const double cnt = m[37];
  if (r >= 3 && c >= 3) {  // +-cnt I
    if (r != c) return 0.0;
    return blk == 2 ? -w * cnt : w * cnt;
  }
  if (r < 3 && c < 3) {
    const int ai[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
    if (blk == 0) return w * m[ai[r][c]];
    if (blk == 1) return w * m[6 + ai[r][c]];
    return w * m[12 + r * 3 + c];
  }
  // cross blocks with [s]x = [[0,-s2,s1],[s2,0,-s0],[-s1,s0,0]]
  auto skew = [&](const double* sv, int rr, int cc) -> double {
    if (rr == cc) return 0.0;
    const int k = 3 - rr - cc;  // the remaining index
    const double sgn = ((rr + 1) % 3 == cc) ? -1.0 : 1.0;
    return sgn * sv[k];
  };
  const double* Si = m + 21;
  const double* Sj = m + 24;
  if (r < 3) {  // upper-right
    if (blk == 0) return w * skew(Si, r, c - 3);
    if (blk == 1) return w * skew(Sj, r, c - 3);
    return -w * skew(Si, r, c - 3);
  }
  // lower-left
  if (blk == 0) return -w * skew(Si, r - 3, c);
  if (blk == 1) return -w * skew(Sj, r - 3, c);
  return w * skew(Sj, r - 3, c);
}

__global__ void __launch_bounds__(256) k_sparse(SparseArgs a) {
  const int gid = (blockIdx.x * blockDim.x + threadIdx.x) / SPARSE_G;  // set
  const int gl = threadIdx.x & (SPARSE_G - 1);
  const bool live = gid < a.n_sets;
  const int set = live ? gid : a.n_sets - 1;
  const int fi = a.set_fi[set], fj = a.set_fj[set];
  const int64_t c0 = a.set_off[set], c1 = live ? a.set_end[set] : c0;
  const PoseDev& Pi = a.poses[fi];
  const PoseDev& Pj = a.poses[fj];
  double Ri[9], ti[3], Rj[9], tj[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) { Ri[k] = Pi.R[k]; Rj[k] = Pj.R[k]; }
#pragma unroll
  for (int k = 0; k < 3; ++k) { ti[k] = Pi.t[k]; tj[k] = Pj.t[k]; }

  // moments
  double m[SPARSE_NM];
#pragma unroll
  for (int k = 0; k < SPARSE_NM; ++k) m[k] = 0.0;
  double* Ai = m;       // |y_i|^2 I - y_i y_i^T, packed (00,01,02,11,12,22)
  double* Aj = m + 6;
  double* M = m + 12;   // y_j y_i^T - (y_i.y_j) I
  double* Si = m + 21;
  double* Sj = m + 24;
  double* gi = m + 27;
  double* gj = m + 30;
  double* sr = m + 33;
  for (int64_t c = c0 + gl; c < c1; c += SPARSE_G) {
    double yi[3], yj[3];
    xf_apply(Ri, ti, a.pts_i[3 * c], a.pts_i[3 * c + 1], a.pts_i[3 * c + 2], yi);
    xf_apply(Rj, tj, a.pts_j[3 * c], a.pts_j[3 * c + 1], a.pts_j[3 * c + 2], yj);
    const double r0 = yi[0] - yj[0], r1 = yi[1] - yj[1], r2 = yi[2] - yj[2];
    m[36] += r0 * r0 + r1 * r1 + r2 * r2;
    if (a.world_i) {
      a.world_i[3 * c] = yi[0]; a.world_i[3 * c + 1] = yi[1]; a.world_i[3 * c + 2] = yi[2];
      a.world_j[3 * c] = yj[0]; a.world_j[3 * c + 1] = yj[1]; a.world_j[3 * c + 2] = yj[2];
    }
    if (a.energy_only) continue;
    m[37] += 1.0;
    Ai[0] += yi[1] * yi[1] + yi[2] * yi[2];
    Ai[1] -= yi[0] * yi[1];
    Ai[2] -= yi[0] * yi[2];
    Ai[3] += yi[0] * yi[0] + yi[2] * yi[2];
    Ai[4] -= yi[1] * yi[2];
    Ai[5] += yi[0] * yi[0] + yi[1] * yi[1];
    Aj[0] += yj[1] * yj[1] + yj[2] * yj[2];
    Aj[1] -= yj[0] * yj[1];
    Aj[2] -= yj[0] * yj[2];
    Aj[3] += yj[0] * yj[0] + yj[2] * yj[2];
    Aj[4] -= yj[1] * yj[2];
    Aj[5] += yj[0] * yj[0] + yj[1] * yj[1];
    M[0] -= yj[1] * yi[1] + yj[2] * yi[2];
    M[1] += yj[0] * yi[1];
    M[2] += yj[0] * yi[2];
    M[3] += yj[1] * yi[0];
    M[4] -= yj[0] * yi[0] + yj[2] * yi[2];
    M[5] += yj[1] * yi[2];
    M[6] += yj[2] * yi[0];
    M[7] += yj[2] * yi[1];
    M[8] -= yj[0] * yi[0] + yj[1] * yi[1];
#pragma unroll
    for (int k = 0; k < 3; ++k) { Si[k] += yi[k]; Sj[k] += yj[k]; }
    gi[0] += yi[1] * r2 - yi[2] * r1;
    gi[1] += yi[2] * r0 - yi[0] * r2;
    gi[2] += yi[0] * r1 - yi[1] * r0;
    gj[0] += yj[1] * r2 - yj[2] * r1;
    gj[1] += yj[2] * r0 - yj[0] * r2;
    gj[2] += yj[0] * r1 - yj[1] * r0;
    sr[0] += r0; sr[1] += r1; sr[2] += r2;
  }
  double* out = a.set_out + (int64_t)set * SFB_SET_STRIDE;
  if (a.energy_only) {
    const double E = group_sum(m[36]);
    if (live && gl == 0) out[SFB_SET_E] = E;
    return;
  }
  __shared__ double msh[256 / SPARSE_G][SPARSE_NM];
  double* ms = msh[threadIdx.x / SPARSE_G];
#pragma unroll
  for (int k = 0; k < SPARSE_NM; ++k) {
    const double t = group_sum(m[k]);
    if ((k & (SPARSE_G - 1)) == gl) ms[k] = t;
  }
  __syncwarp();
  if (!live) return;
  // solver.py:406,414: the J^T J blocks only exist for w_sparse > 0, while the
  // gradient always carries w_sparse (solver.py:644-645).
  const double wg = a.w_sparse;
  const double w = a.w_sparse > 0.0 ? a.w_sparse : 0.0;
  for (int e = gl; e <= SFB_SET_E; e += SPARSE_G) out[e] = sparse_entry(e, ms, w, wg);
}

void launch_sparse(const SparseArgs& a, cudaStream_t s) {
  if (a.n_sets <= 0) return;
  const int blocks = (a.n_sets * SPARSE_G + 255) / 256;
  sfb_count_launch();
  k_sparse<<<blocks, 256, 0, s>>>(a);
}

// eval_sparse residuals (solver.py:114-123) and per-set max |r| for
// max_residual_set (solver.py:765-776).
__global__ void k_sparse_residuals(SparseArgs a, double* res, double* set_max) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= a.n_sets) return;
  const PoseDev& Pi = a.poses[a.set_fi[warp]];
  const PoseDev& Pj = a.poses[a.set_fj[warp]];
  double mx = 0.0;
  for (int64_t c = a.set_off[warp] + lane; c < a.set_end[warp]; c += 32) {
    double yi[3], yj[3];
    xf_apply(Pi.R, Pi.t, a.pts_i[3 * c], a.pts_i[3 * c + 1], a.pts_i[3 * c + 2], yi);
    xf_apply(Pj.R, Pj.t, a.pts_j[3 * c], a.pts_j[3 * c + 1], a.pts_j[3 * c + 2], yj);
    const double r0 = yi[0] - yj[0], r1 = yi[1] - yj[1], r2 = yi[2] - yj[2];
    if (res) { res[3 * c] = r0; res[3 * c + 1] = r1; res[3 * c + 2] = r2; }
    mx = fmax(mx, sqrt(r0 * r0 + r1 * r1 + r2 * r2));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0 && set_max) set_max[warp] = mx;
}

void launch_sparse_residuals(const SparseArgs& a, double* res, double* set_max, cudaStream_t s) {
  if (a.n_sets <= 0) return;
  sfb_count_launch();
  k_sparse_residuals<<<(a.n_sets * 32 + 255) / 256, 256, 0, s>>>(a, res, set_max);
}

// ---------------------------------------------------------------------------
// T_f <- exp(dx_f) o T_f for every non-anchor frame (thread per frame), plus a
// deterministic |dx| in block 0.
__device__ void so3_exp_dev(const double w[3], double E[9]) {
  const double a = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double K[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
  double KK[9];
  double s1, s2;
  if (a < 1e-8) {  // geometry.py:44-46
    s1 = 1.0;
    s2 = 0.5;
  } else {
    for (int k = 0; k < 9; ++k) K[k] /= a;
    s1 = sin(a);
    s2 = 1.0 - cos(a);
  }
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      KK[r * 3 + c] = K[r * 3 + 0] * K[0 * 3 + c] + K[r * 3 + 1] * K[1 * 3 + c] + K[r * 3 + 2] * K[2 * 3 + c];
  for (int k = 0; k < 9; ++k) E[k] = ((k % 4) == 0 ? 1.0 : 0.0) + s1 * K[k] + s2 * KK[k];
}

__device__ void left_jacobian_dev(const double w[3], double V[9]) {
  const double a = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  const double K[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
  double KK[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      KK[r * 3 + c] = K[r * 3 + 0] * K[0 * 3 + c] + K[r * 3 + 1] * K[1 * 3 + c] + K[r * 3 + 2] * K[2 * 3 + c];
  const double a2 = a * a;
  double c1, c2;
  if (a < 1e-4) {  // geometry.py:85-86
    c1 = 0.5 - a2 / 24.0;
    c2 = 1.0 / 6.0 - a2 / 120.0;
  } else {
    c1 = (1.0 - cos(a)) / a2;
    c2 = (a - sin(a)) / (a2 * a);
  }
  for (int k = 0; k < 9; ++k) V[k] = ((k % 4) == 0 ? 1.0 : 0.0) + c1 * K[k] + c2 * KK[k];
}

__global__ void k_pose_update(PoseDev* poses, int n_frames, const double* dx, double* step_norm,
                              const double* skip) {
  if (skip && *skip != 0.0) return;
  const int f = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (f < n_frames) {
    const double* d = dx + 6 * (f - 1);
    const double w[3] = {d[0], d[1], d[2]};
    const double v[3] = {d[3], d[4], d[5]};
    double E[9], V[9];
    so3_exp_dev(w, E);
    left_jacobian_dev(w, V);
    PoseDev& P = poses[f];
    double R[9], t[3];
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c)
        R[r * 3 + c] = E[r * 3 + 0] * P.R[0 * 3 + c] + E[r * 3 + 1] * P.R[1 * 3 + c] + E[r * 3 + 2] * P.R[2 * 3 + c];
      const double te = V[r * 3 + 0] * v[0] + V[r * 3 + 1] * v[1] + V[r * 3 + 2] * v[2];
      t[r] = E[r * 3 + 0] * P.t[0] + E[r * 3 + 1] * P.t[1] + E[r * 3 + 2] * P.t[2] + te;
    }
    for (int k = 0; k < 9; ++k) P.R[k] = R[k];
    for (int k = 0; k < 3; ++k) P.t[k] = t[k];
    P.f_layout = 0;  // matmul results are C-ordered
  }
  if (blockIdx.x == 0 && step_norm) {
    // deterministic |dx|: fixed per-thread striding + fixed tree
    __shared__ double sh[32];
    const int nv = 6 * (n_frames - 1);
    double acc = 0.0;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) acc += dx[i] * dx[i];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
      double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
      v = warp_sum(v);
      if (threadIdx.x == 0) *step_norm = sqrt(v);
    }
  }
}

void launch_pose_update(PoseDev* poses, int n_frames, const double* dx, double* step_norm,
                        const double* skip, cudaStream_t s) {
  const int nv = n_frames - 1;
  int blocks = (nv + 255) / 256;
  if (blocks < 1) blocks = 1;
  sfb_count_launch();
  k_pose_update<<<blocks, 256, 0, s>>>(poses, n_frames, dx, step_norm, skip);
}

// Per-tile bounding spheres of the valid points (k_tiles_batch, one warp per
// 16x16 tile): centre = AABB centre, radius = max distance, inflated so the
// sphere bounds every point with margin to spare for rounding.
// Batched upload: blockIdx.y selects the frame.
__global__ void k_pack_batch(const PackArgs* args) {
  const PackArgs& a0 = args[blockIdx.y];
  PackArgs a = a0;
  // reuse the single-frame body through a grid-stride loop over this frame
  const int hw = a.w * a.h;
  int cnt_vd = 0, cnt_geo = 0, bad = 0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < hw; p += gridDim.x * blockDim.x) {
    const unsigned vd = a.vd[p] ? 1u : 0u;
    const unsigned vn = a.vn[p] ? 1u : 0u;
    a.P[p] = make_float4(a.pts[3 * p], a.pts[3 * p + 1], a.pts[3 * p + 2],
                         __uint_as_float(vd * SFB_FLAG_VD | vn * SFB_FLAG_VN));
    a.N[p] = make_float4(a.nrm[3 * p], a.nrm[3 * p + 1], a.nrm[3 * p + 2], 0.f);
    const float2 g = make_float2(a.grad[2 * p], a.grad[2 * p + 1]);
    a.G[p] = g;
    const int y = p / a.w, x = p - y * a.w;
    float4 t0 = make_float4(0.f, 0.f, 0.f, 0.f), t1 = t0;
    if (x + 1 < a.w && y + 1 < a.h) {
      const int q = p + 1, r = p + a.w, s = p + a.w + 1;
      t0 = make_float4(g.x, g.y, a.grad[2 * q], a.grad[2 * q + 1]);
      t1 = make_float4(a.grad[2 * r], a.grad[2 * r + 1], a.grad[2 * s], a.grad[2 * s + 1]);
    }
    a.T[2 * p] = t0;
    a.T[2 * p + 1] = t1;
    cnt_vd += (int)vd;
    cnt_geo += (int)(vd & vn);
    const bool fin = isfinite(a.pts[3 * p]) && isfinite(a.pts[3 * p + 1]) && isfinite(a.pts[3 * p + 2]) &&
                     isfinite(a.nrm[3 * p]) && isfinite(a.nrm[3 * p + 1]) && isfinite(a.nrm[3 * p + 2]) &&
                     isfinite(g.x) && isfinite(g.y);
    bad += fin ? 0 : 1;
  }
  for (int o = 16; o > 0; o >>= 1) {
    cnt_vd += __shfl_xor_sync(0xffffffffu, cnt_vd, o);
    cnt_geo += __shfl_xor_sync(0xffffffffu, cnt_geo, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&a.counts[0], cnt_vd);
    atomicAdd(&a.counts[1], cnt_geo);
    if (bad) atomicAdd(&a.counts[2], bad);
  }
}

__global__ void k_tiles_batch(const PackArgs* args) {
  const PackArgs& a = args[blockIdx.y];
  const int nt = a.tiles_x * a.tiles_y;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int tile = w0; tile < nt; tile += nwarps) {
    const int x0 = (tile % a.tiles_x) * SFB_TILE, y0 = (tile / a.tiles_x) * SFB_TILE;
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    int c = 0;
    for (int k = lane; k < SFB_TILE * SFB_TILE; k += 32) {
      const int x = x0 + (k % SFB_TILE), y = y0 + (k / SFB_TILE);
      if (x >= a.w || y >= a.h) continue;
      const float4 p = a.P[y * a.w + x];
      if (!(__float_as_uint(p.w) & SFB_FLAG_VD)) continue;
      const double q[3] = {p.x, p.y, p.z};
      for (int d = 0; d < 3; ++d) { lo[d] = fmin(lo[d], q[d]); hi[d] = fmax(hi[d], q[d]); }
      ++c;
    }
    for (int o = 16; o > 0; o >>= 1) {
      c += __shfl_xor_sync(0xffffffffu, c, o);
      for (int d = 0; d < 3; ++d) {
        lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
        hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
      }
    }
    double ctr[3];
    for (int d = 0; d < 3; ++d) ctr[d] = 0.5 * (lo[d] + hi[d]);
    double r2 = 0.0;
    for (int k = lane; k < SFB_TILE * SFB_TILE; k += 32) {
      const int x = x0 + (k % SFB_TILE), y = y0 + (k / SFB_TILE);
      if (x >= a.w || y >= a.h) continue;
      const float4 p = a.P[y * a.w + x];
      if (!(__float_as_uint(p.w) & SFB_FLAG_VD)) continue;
      const double dx = p.x - ctr[0], dy = p.y - ctr[1], dz = p.z - ctr[2];
      r2 = fmax(r2, dx * dx + dy * dy + dz * dz);
    }
    for (int o = 16; o > 0; o >>= 1) r2 = fmax(r2, __shfl_xor_sync(0xffffffffu, r2, o));
    if (lane == 0) {
      const double r = sqrt(r2) * (1.0 + 1e-9) + 1e-9;
      a.tiles[tile] = c > 0 ? make_double4(ctr[0], ctr[1], ctr[2], r) : make_double4(0, 0, 0, -1.0);
      a.tile_count[tile] = c;
    }
  }
}

// Pinned host planes -> device staging: one job per plane (blockIdx.y), 16-byte
// loads when source and destination share their alignment, bytes otherwise.
__global__ void k_stage_copy(const CopyJob* jobs) {
  const CopyJob j = jobs[blockIdx.y];
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  const uintptr_t sa = (uintptr_t)j.src & 15, da = (uintptr_t)j.dst & 15;
  size_t head = 0, nv = 0;
  if (sa == da) {
    head = (16 - sa) & 15;
    if (head > j.n) head = j.n;
    nv = (j.n - head) / 16;
  }
  const uint4* s4 = reinterpret_cast<const uint4*>(j.src + head);
  uint4* d4 = reinterpret_cast<uint4*>(j.dst + head);
  for (size_t i = tid; i < nv; i += nth) d4[i] = s4[i];
  const size_t done = head + 16 * nv;
  // head and tail bytes (all bytes when the alignments differ)
  for (size_t i = tid; i < head; i += nth) j.dst[i] = j.src[i];
  for (size_t i = done + tid; i < j.n; i += nth) j.dst[i] = j.src[i];
}

cudaError_t launch_stage_copy(const CopyJob* jobs, int n_jobs, cudaStream_t s) {
  for (int j0 = 0; j0 < n_jobs; j0 += 65535) {  // gridDim.y limit
    const int nj = n_jobs - j0 < 65535 ? n_jobs - j0 : 65535;
    sfb_count_launch();
    k_stage_copy<<<dim3(16, nj), 256, 0, s>>>(jobs + j0);
  }
  return cudaGetLastError();
}

void launch_pack_batch(const PackArgs* args_dev, int n, int max_hw, int max_tiles, cudaStream_t s) {
  if (n <= 0) return;
  int bx = (max_hw + 255) / 256;
  if (bx > 64) bx = 64;
  sfb_count_launch(2);
  k_pack_batch<<<dim3(bx, n), 256, 0, s>>>(args_dev);
  int tx = (max_tiles * 32 + 255) / 256;
  if (tx < 1) tx = 1;
  k_tiles_batch<<<dim3(tx, n), 256, 0, s>>>(args_dev);
}
