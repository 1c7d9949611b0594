// build_cache on the device (reference frames.py:75-151): an RGB-D frame
// (H x W colour + depth) -> the downsampled CachedFrame planes, bit-identical
// to the reference's NumPy float32 pipeline, written straight into a frame
// slot of the context (so the solver needs no upload) and into a host image.
//
//  k_cache_reduce   one thread per low-res pixel (= one bh x bw block):
//                   block-mean luminance (RgbdFrame.luminance, frames.py:33-35,
//                   _block_reduce_mean :70-74), block-median depth over the
//                   valid samples (_block_reduce_median :53-67), unprojection
//                   with the scaled intrinsics (geometry.py:229-235).
//  k_cache_normals  central-difference normals facing the camera
//                   (_estimate_normals :122-151) and the intensity gradient
//                   (:101-103).
//
// NumPy semantics reproduced (measured, see tests/golden/make_cache_golden.py):
//  * luminance: float32 (H,W,3) @ (3,) is the BLAS FMA chain whose order the
//    host probes (_rounding.probe_luma), then / 255 in float32;
//  * mean over axes (1,3): each block row is NumPy's pairwise sum (n < 8
//    sequential, else 8 accumulators), the rows are added in order, and the
//    float32 sum is divided by the count in double, then rounded to float32;
//  * nanmedian: float32 (lo + hi) / 2 of the two middle valid samples;
//  * unproject: ((u - cx) / fx) * z in double, rounded to float32;
//  * cross / norm / dot: float32 products and sums, no contraction.
#include "sfb_kernels.cuh"

#define CACHE_THREADS 128

__device__ __forceinline__ float luma(const uint8_t* c, int order) {
  const float x[3] = {(float)c[0], (float)c[1], (float)c[2]};
  const float w[3] = {0.299f, 0.587f, 0.114f};
  static constexpr int P[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  const int i = P[order][0], j = P[order][1], k = P[order][2];
  const float s = __fmaf_rn(x[k], w[k], __fmaf_rn(x[j], w[j], __fmul_rn(x[i], w[i])));
  return __fdiv_rn(s, 255.0f);
}

// NumPy pairwise_sum of one block row (float32)
__device__ __forceinline__ float row_sum(const uint8_t* color, int W, int y, int x0, int bw,
                                         int order) {
  const uint8_t* row = color + ((size_t)y * W + x0) * 3;
  if (bw < 8) {
    float s = 0.0f;
    for (int l = 0; l < bw; ++l) s = __fadd_rn(s, luma(row + 3 * l, order));
    return s;
  }
  float r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = luma(row + 3 * k, order);
  int i = 8;
  for (; i < bw - (bw % 8); i += 8)
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = __fadd_rn(r[k], luma(row + 3 * (i + k), order));
  float s = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                      __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
  for (; i < bw; ++i) s = __fadd_rn(s, luma(row + 3 * i, order));
  return s;
}

// Bitonic sort of NS floats in registers (NaN-free: invalid samples are +inf).
template <int NS>
__device__ __forceinline__ void bitonic(float (&v)[NS]) {
#pragma unroll
  for (int k = 2; k <= NS; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const float a = v[i], b = v[l];
          const bool sw = up ? (a > b) : (a < b);
          v[i] = sw ? b : a;
          v[l] = sw ? a : b;
        }
      }
}

template <int NS>
__device__ __forceinline__ float block_median(const float* depth, int W, int y0, int x0, int bh,
                                              int bw, bool* has_valid) {
  float v[NS];
  int n = 0;
  bool any = false;
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    float d = __int_as_float(0x7f800000);  // +inf pads
    if (k < bh * bw) {
      const int j = k / bw, l = k - j * bw;
      const float x = __ldg(&depth[(size_t)(y0 + j) * W + x0 + l]);
      any |= !(x <= 0.0f);  // has_valid = ~all(blocks <= 0): NaN samples count
      if (x > 0.0f) {       // nanmedian: NaN and <= 0 are missing
        d = x;
        ++n;
      }
    }
    v[k] = d;
  }
  *has_valid = any;
  if (n == 0) return __int_as_float(0x7fc00000);  // all-NaN slice -> NaN
  bitonic<NS>(v);
  const int il = (n - 1) >> 1, ih = n >> 1;
  float lo = v[0], hi = v[0];
#pragma unroll
  for (int k = 1; k < NS; ++k) {
    lo = (k == il) ? v[k] : lo;
    hi = (k == ih) ? v[k] : hi;
  }
  return __fmul_rn(__fadd_rn(lo, hi), 0.5f);  // np.true_divide(lo + hi, 2.)
}

template <int NS>
__global__ void __launch_bounds__(CACHE_THREADS) k_cache_reduce(CacheArgs a) {
  const CacheFrame& f = a.frames[blockIdx.y];
  const int hw = a.low_w * a.low_h;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= hw) return;
  const int y = p / a.low_w, x = p - y * a.low_w;
  const int y0 = y * a.bh, x0 = x * a.bw;
  // intensity: rows of the block in order, each a pairwise row sum
  float acc = 0.0f;
  for (int j = 0; j < a.bh; ++j) {
    const float r = row_sum(f.color, a.W, y0 + j, x0, a.bw, a.luma_order);
    acc = j == 0 ? r : __fadd_rn(acc, r);
  }
  f.intensity[p] = (float)__ddiv_rn((double)acc, (double)(a.bh * a.bw));
  bool has_valid = false;
  const float med = block_median<NS>(f.depth_in, a.W, y0, x0, a.bh, a.bw, &has_valid);
  const float d = has_valid ? med : 0.0f;
  f.depth[p] = d;
  const bool valid = d > 0.0f;
  f.valid[p] = valid ? 1 : 0;
  float px = 0.0f, py = 0.0f, pz = 0.0f;
  if (valid) {
    const double z = (double)d;
    px = (float)__dmul_rn(__ddiv_rn(__dsub_rn((double)x, a.cx), a.fx), z);
    py = (float)__dmul_rn(__ddiv_rn(__dsub_rn((double)y, a.cy), a.fy), z);
    pz = d;
  }
  f.points[3 * p] = px;
  f.points[3 * p + 1] = py;
  f.points[3 * p + 2] = pz;
}

__global__ void __launch_bounds__(CACHE_THREADS) k_cache_normals(CacheArgs a) {
  const CacheFrame& f = a.frames[blockIdx.y];
  const int w = a.low_w, h = a.low_h;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= w * h) return;
  const int y = p / w, x = p - y * w;
  const bool interior = x >= 1 && x < w - 1 && y >= 1 && y < h - 1;
  float n0 = 0.0f, n1 = 0.0f, n2 = 0.0f;
  bool ok = false;
  if (interior) {
    ok = f.valid[p] && f.valid[p + 1] && f.valid[p - 1] && f.valid[p + w] && f.valid[p - w];
    const float* P = f.points;
    float dx[3], dy[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      dx[c] = __fsub_rn(P[3 * (p + 1) + c], P[3 * (p - 1) + c]);
      dy[c] = __fsub_rn(P[3 * (p + w) + c], P[3 * (p - w) + c]);
    }
    // np.cross(dy, dx)
    n0 = __fsub_rn(__fmul_rn(dy[1], dx[2]), __fmul_rn(dy[2], dx[1]));
    n1 = __fsub_rn(__fmul_rn(dy[2], dx[0]), __fmul_rn(dy[0], dx[2]));
    n2 = __fsub_rn(__fmul_rn(dy[0], dx[1]), __fmul_rn(dy[1], dx[0]));
    const float len = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(n0, n0), __fmul_rn(n1, n1)),
                                           __fmul_rn(n2, n2)));
    ok = ok && len > 1e-12f;
    if (ok) {
      n0 = __fdiv_rn(n0, len);
      n1 = __fdiv_rn(n1, len);
      n2 = __fdiv_rn(n2, len);
      const float s = __fadd_rn(__fadd_rn(__fmul_rn(n0, P[3 * p]), __fmul_rn(n1, P[3 * p + 1])),
                                __fmul_rn(n2, P[3 * p + 2]));
      if (s > 0.0f) {
        n0 = -n0;
        n1 = -n1;
        n2 = -n2;
      }
    }
  }
  if (!ok) n0 = n1 = n2 = 0.0f;
  f.normals[3 * p] = n0;
  f.normals[3 * p + 1] = n1;
  f.normals[3 * p + 2] = n2;
  f.valid_n[p] = ok ? 1 : 0;
  const float* I = f.intensity;
  f.grad[2 * p] = (x >= 1 && x < w - 1) ? __fmul_rn(0.5f, __fsub_rn(I[p + 1], I[p - 1])) : 0.0f;
  f.grad[2 * p + 1] = (y >= 1 && y < h - 1) ? __fmul_rn(0.5f, __fsub_rn(I[p + w], I[p - w])) : 0.0f;
}

cudaError_t launch_build_cache(const CacheArgs& a, int n_frames, cudaStream_t s) {
  if (n_frames <= 0) return cudaSuccess;
  const int hw = a.low_w * a.low_h;
  const dim3 grid((hw + CACHE_THREADS - 1) / CACHE_THREADS, n_frames);
  const int ns = a.bh * a.bw;
  sfb_count_launch(2);
  if (ns <= 1) k_cache_reduce<1><<<grid, CACHE_THREADS, 0, s>>>(a);
  else if (ns <= 4) k_cache_reduce<4><<<grid, CACHE_THREADS, 0, s>>>(a);
  else if (ns <= 16) k_cache_reduce<16><<<grid, CACHE_THREADS, 0, s>>>(a);
  else if (ns <= 64) k_cache_reduce<64><<<grid, CACHE_THREADS, 0, s>>>(a);
  else return cudaErrorInvalidValue;
  k_cache_normals<<<grid, CACHE_THREADS, 0, s>>>(a);
  return cudaGetLastError();
}
