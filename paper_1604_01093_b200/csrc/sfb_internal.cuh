// sfb_internal.cuh — device data layout and math shared by the sfb kernels.
//
// HBM layout (one allocation per frame slot, all planes pixel-major):
//   P  float4[hw]   (x, y, z, flags)  flags bit0 valid_depth, bit1 valid_normal
//   N  float4[hw]   (nx, ny, nz, 0)
//   G  float2[hw]   grad_low (d/dx, d/dy)                     (frames.py:45)
//   T  float4[2hw]  bilinear taps of grad_low at (y,x),(y,x+1) | (y+1,x),(y+1,x+1)
// so a source pixel is 2x16B + 8B of coalesced loads and a bilinear sample of
// the 2-channel gradient image is two aligned 16B loads (interp.py:36-58).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define SFB_FLAG_VD 1u
#define SFB_FLAG_VN 2u

struct FrameDev {
  const float4* P;
  const float4* N;
  const float2* G;
  const float4* T;
  double fx, fy, cx, cy;
  int w, h;
  int n_valid_depth;  // #valid_depth pixels (NumPy m == 1 rounding special case)
  int n_valid_geo;    // #(valid_depth & valid_normal) pixels
  // 16x16 pixel tiles: conservative bounding sphere of the valid points
  // (cx, cy, cz, r) and their count; used to cull the frame-pair filter.
  const double4* tiles;
  const int* tile_count;
  int tiles_x, tiles_y;
  const float* I;     // intensity_low (dense_verify only), null until uploaded
};

#define SFB_TILE 16

struct PoseDev {
  double R[9];  // row-major
  double t[3];
  int f_layout;  // host rotation array was Fortran-ordered
  int pad_;
};

struct Rounding {
  int mv_c, mv_f, gemm, apply_n, apply_1, dot3;
};

// ---------------------------------------------------------------------------
// Exact NumPy/OpenBLAS rounding replication.  A 3-term dot product is the FMA
// chain fma(a_k b_k, fma(a_j b_j, a_i*b_i)); `o` selects the permutation
// (i,j,k) = 0:(0,1,2) 1:(0,2,1) 2:(1,0,2) 3:(1,2,0) 4:(2,0,1) 5:(2,1,0).
__device__ __forceinline__ double dot3o(double a0, double a1, double a2, double b0,
                                        double b1, double b2, int o) {
  double x0, y0, x1, y1, x2, y2;
  switch (o) {
    default:
    case 0: x0 = a0; y0 = b0; x1 = a1; y1 = b1; x2 = a2; y2 = b2; break;
    case 1: x0 = a0; y0 = b0; x1 = a2; y1 = b2; x2 = a1; y2 = b1; break;
    case 2: x0 = a1; y0 = b1; x1 = a0; y1 = b0; x2 = a2; y2 = b2; break;
    case 3: x0 = a1; y0 = b1; x1 = a2; y1 = b2; x2 = a0; y2 = b0; break;
    case 4: x0 = a2; y0 = b2; x1 = a0; y1 = b0; x2 = a1; y2 = b1; break;
    case 5: x0 = a2; y0 = b2; x1 = a1; y1 = b1; x2 = a0; y2 = b0; break;
  }
  return __fma_rn(x2, y2, __fma_rn(x1, y1, __dmul_rn(x0, y0)));
}

// Rigid transform in registers / shared memory.
struct Xf {
  double R[9];
  double t[3];
};

// RigidTransform.inverse (geometry.py:144-146): R^T exactly, t = -(R^T t).
// NumPy evaluates (-R.T) @ t; R.T is F-ordered when R is C-ordered.
__device__ __forceinline__ Xf xf_inverse_exact(const PoseDev& p, const Rounding& rd) {
  Xf o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o.R[r * 3 + c] = p.R[c * 3 + r];
  const int ord = p.f_layout ? rd.mv_c : rd.mv_f;
#pragma unroll
  for (int r = 0; r < 3; ++r)
    o.t[r] = -dot3o(o.R[r * 3 + 0], o.R[r * 3 + 1], o.R[r * 3 + 2], p.t[0], p.t[1], p.t[2], ord);
  return o;
}

// RigidTransform.compose (geometry.py:127-130) with a C-ordered left operand
// (the result of inverse() is a .copy()).
__device__ __forceinline__ Xf xf_compose_exact(const Xf& a, const PoseDev& b, const Rounding& rd) {
  Xf o;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
      o.R[r * 3 + c] = dot3o(a.R[r * 3 + 0], a.R[r * 3 + 1], a.R[r * 3 + 2], b.R[0 * 3 + c],
                             b.R[1 * 3 + c], b.R[2 * 3 + c], rd.gemm);
    o.t[r] = __dadd_rn(
        dot3o(a.R[r * 3 + 0], a.R[r * 3 + 1], a.R[r * 3 + 2], b.t[0], b.t[1], b.t[2], rd.mv_c),
        a.t[r]);
  }
  return o;
}

// relative = pose_b.inverse() @ pose_a, exactly as frames.py:168 / solver.py:221.
__device__ __forceinline__ Xf xf_relative_exact(const PoseDev& pa, const PoseDev& pb,
                                                const Rounding& rd) {
  Xf ib = xf_inverse_exact(pb, rd);
  return xf_compose_exact(ib, pa, rd);
}

// RigidTransform.apply (geometry.py:148-151): points @ R.T + t.
__device__ __forceinline__ void xf_apply_exact(const Xf& x, double p0, double p1, double p2,
                                               int ord, double q[3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
    q[r] = __dadd_rn(dot3o(p0, p1, p2, x.R[r * 3 + 0], x.R[r * 3 + 1], x.R[r * 3 + 2], ord),
                     x.t[r]);
}

// RigidTransform.rotate (geometry.py:153-155).
__device__ __forceinline__ void xf_rotate_exact(const Xf& x, double p0, double p1, double p2,
                                                int ord, double q[3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
    q[r] = dot3o(p0, p1, p2, x.R[r * 3 + 0], x.R[r * 3 + 1], x.R[r * 3 + 2], ord);
}

// Intrinsics.project_many (geometry.py:219-227): separate mul, div, add.
__device__ __forceinline__ void project_exact(double fx, double fy, double cx, double cy,
                                              const double q[3], double* u, double* v,
                                              bool* in_front) {
  const bool f = q[2] > 0.0;
  const double z = f ? q[2] : 1.0;
  *u = __dadd_rn(__ddiv_rn(__dmul_rn(fx, q[0]), z), cx);
  *v = __dadd_rn(__ddiv_rn(__dmul_rn(fy, q[1]), z), cy);
  *in_front = f;
}

// Plain (contractible) transform helpers for the smooth parts of the path.
__device__ __forceinline__ void xf_apply(const double* R, const double* t, double p0, double p1,
                                         double p2, double q[3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r) q[r] = R[r * 3 + 0] * p0 + R[r * 3 + 1] * p1 + R[r * 3 + 2] * p2 + t[r];
}

__device__ __forceinline__ void xf_inverse_plain(const double* R, const double* t, double* Ri,
                                                 double* ti) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) Ri[r * 3 + c] = R[c * 3 + r];
  for (int r = 0; r < 3; ++r) ti[r] = -(Ri[r * 3 + 0] * t[0] + Ri[r * 3 + 1] * t[1] + Ri[r * 3 + 2] * t[2]);
}

// bilinear_sample_with_grad (interp.py:8-14,36-58) on the 2-channel gradient
// image via the pre-expanded taps plane.
__device__ __forceinline__ void bilinear_grad2(const FrameDev& f, double x, double y,
                                               double val[2], double ddx[2], double ddy[2]) {
  const double wm1 = (double)(f.w - 1), hm1 = (double)(f.h - 1);
  x = fmin(fmax(x, 0.0), wm1);
  y = fmin(fmax(y, 0.0), hm1);
  int x0 = min((int)floor(x), f.w - 2);
  int y0 = min((int)floor(y), f.h - 2);
  const double ax = x - (double)x0, ay = y - (double)y0;
  const float4 t0 = __ldg(&f.T[2 * (y0 * f.w + x0)]);
  const float4 t1 = __ldg(&f.T[2 * (y0 * f.w + x0) + 1]);
  const double bx = 1.0 - ax, by = 1.0 - ay;
  const double v00[2] = {t0.x, t0.y}, v01[2] = {t0.z, t0.w};
  const double v10[2] = {t1.x, t1.y}, v11[2] = {t1.z, t1.w};
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    val[c] = v00[c] * bx * by + v01[c] * ax * by + v10[c] * bx * ay + v11[c] * ax * ay;
    ddx[c] = (v01[c] - v00[c]) * by + (v11[c] - v10[c]) * ay;
    ddy[c] = (v10[c] - v00[c]) * bx + (v11[c] - v01[c]) * ax;
  }
}


// The same sample, evaluated with integer clamping and the difference form
// val = v00 + ax d01 + ay (d10 + ax dxy), ddx = d01 + ay dxy, ddy = d10 + ax dxy
// (rounding differs from interp.py's weight form at the ulp level only).
__device__ __forceinline__ void bilinear_grad2_fast(const FrameDev& f, double x, double y,
                                                    double val[2], double ddx[2], double ddy[2]) {
  const int xf = __double2int_rd(x), yf = __double2int_rd(y);  // saturating floor
  const int x0 = min(max(xf, 0), f.w - 2), y0 = min(max(yf, 0), f.h - 2);
  double ax = x - (double)x0, ay = y - (double)y0;
  // clip(x, 0, w-1): below -> weight 0, beyond w-1 -> weight 1 exactly
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
    ddx[c] = fma(ay, dxy, d01);
    ddy[c] = fma(ax, dxy, d10);
  }
}

// Warp-level deterministic butterfly sum (every lane ends with the same bits).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Symmetric 6x6 packed upper-triangle index (row-major over r <= c).
__host__ __device__ constexpr int sym6(int r, int c) {
  return r <= c ? (r * 6 - (r * (r - 1)) / 2 + (c - r)) : (c * 6 - (c * (c - 1)) / 2 + (r - c));
}

// Per-dense-item partial: 21 packed H + 6 g + e_photo + e_geo (+3 pad).
#define SFB_ITEM_STRIDE 32
#define SFB_ITEM_EP 27
#define SFB_ITEM_EG 28
#define SFB_ITEM_PP 29  // frozen energy of the previous linearisation (fused pass)
#define SFB_ITEM_PG 30
// Per-sparse-set output: Hii[36] Hjj[36] Hij[36] gi[6] gj[6] E (+3 pad).
#define SFB_SET_STRIDE 128
#define SFB_SET_GI 108
#define SFB_SET_GJ 114
#define SFB_SET_E 120
