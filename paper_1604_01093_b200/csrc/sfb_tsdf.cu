// Hashed TSDF integrate / de-integrate on the device (reference tsdf.py:55-201).
//
//  k_tsdf_touch   one thread per depth pixel: the truncation band's ray
//                 samples -> packed block keys (_touched_blocks, :162-181);
//                 sorted + deduplicated with CUB afterwards (np.unique).
//  k_tsdf_voxels  one CTA per touched 8x8x8 block, one thread per voxel:
//                 voxel centre -> camera (pose.inverse().apply) -> pixel
//                 (project_many, np.round) -> truncated signed distance,
//                 weight and colour (_apply, :98-128), then, by mode:
//                   EVAL    any voxel hit?              (allocation decisions)
//                   CHECK   would a weight go < -eps?   (de-integration errors)
//                   COMMIT  accumulate s*w, s*w*d, s*w*c in float32; on
//                           de-integration snap float dust, clear empty
//                           voxels and report empty blocks (:146-156).
// The block dictionary (key -> pool slot, insertion order, the reference's
// error order) lives on the host side of the library (sfb_abi.cu); the voxel
// accumulators live in a device pool of 512-voxel blocks.
//
// Every quantity that decides a voxel (which pixel, whether it is hit) and
// every accumulated float32 follows NumPy's evaluation: apply() with the
// probed BLAS FMA order, separate mul/div/add in the projection, round half
// to even, double -> float32 rounding of w, w*sdf and w*colour.
#include "sfb_kernels.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#define TSDF_SHIFT (1LL << 20)

__device__ __forceinline__ long long tsdf_key(long long c0, long long c1, long long c2) {
  // tsdf.py:187-189: ((c + 2^20) << 42) | ((c + 2^20) << 21) | (c + 2^20), int64
  const unsigned long long a = (unsigned long long)(c0 + TSDF_SHIFT);
  const unsigned long long b = (unsigned long long)(c1 + TSDF_SHIFT);
  const unsigned long long c = (unsigned long long)(c2 + TSDF_SHIFT);
  return (long long)((a << 42) | (b << 21) | c);
}

__global__ void k_tsdf_touch(TsdfTouchArgs a) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.W * a.H) return;
  long long* out = a.keys + (size_t)p * a.n_samples;
  const float df = __ldg(&a.depth[p]);
  if (!(df > 0.0f)) {
    for (int s = 0; s < a.n_samples; ++s) out[s] = LLONG_MAX;  // dropped after the sort
    return;
  }
  const int y = p / a.W, x = p - y * a.W;
  const double d = df;
  // rays = unproject(pixels, 1): ((u - cx) / fx) * 1.0
  const double r0 = __ddiv_rn(__dsub_rn((double)x, a.cx), a.fx);
  const double r1 = __ddiv_rn(__dsub_rn((double)y, a.cy), a.fy);
  const double sn = fmax(__dsub_rn(d, a.trunc), 1e-3), sf = __dadd_rn(d, a.trunc);
  double wn[3], wf[3];
  xf_apply_exact(a.pose, __dmul_rn(r0, sn), __dmul_rn(r1, sn), sn, a.ord, wn);
  xf_apply_exact(a.pose, __dmul_rn(r0, sf), __dmul_rn(r1, sf), sf, a.ord, wf);
  for (int s = 0; s < a.n_samples; ++s) {
    const double t = a.t[s];
    long long c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double q = __dadd_rn(wn[k], __dmul_rn(t, __dsub_rn(wf[k], wn[k])));
      c[k] = (long long)floor(__ddiv_rn(q, a.extent));
    }
    out[s] = tsdf_key(c[0], c[1], c[2]);
  }
}

template <int MODE>  // 0 EVAL, 1 CHECK, 2 COMMIT
__global__ void __launch_bounds__(512) k_tsdf_voxels(TsdfVoxelArgs a) {
  const int b = a.first + blockIdx.x;
  const long long key = a.keys[b];
  const long long c0 = ((key >> 42) & ((1LL << 21) - 1)) - TSDF_SHIFT;
  const long long c1 = ((key >> 21) & ((1LL << 21) - 1)) - TSDF_SHIFT;
  const long long c2 = (key & ((1LL << 21) - 1)) - TSDF_SHIFT;
  const int slot = a.slots ? a.slots[b] : -1;
  const int v = threadIdx.x;
  const int i = v >> 6, j = (v >> 3) & 7, k = v & 7;  // meshgrid(indexing="ij") order
  // centers = touched * block_extent + (offset + 0.5) * voxel_size
  const double p0 = __dadd_rn(__dmul_rn((double)c0, a.extent), __dmul_rn(i + 0.5, a.vs));
  const double p1 = __dadd_rn(__dmul_rn((double)c1, a.extent), __dmul_rn(j + 0.5, a.vs));
  const double p2 = __dadd_rn(__dmul_rn((double)c2, a.extent), __dmul_rn(k + 0.5, a.vs));
  double cam[3];
  xf_apply_exact(a.inv_pose, p0, p1, p2, a.ord, cam);
  double u, vv;
  bool front;
  project_exact(a.fx, a.fy, a.cx, a.cy, cam, &u, &vv, &front);
  const double xr = rint(u), yr = rint(vv);
  const bool inside = front && xr >= 0.0 && xr < (double)a.W && yr >= 0.0 && yr < (double)a.H;
  const int xi = (int)fmin(fmax(xr, 0.0), (double)(a.W - 1));
  const int yi = (int)fmin(fmax(yr, 0.0), (double)(a.H - 1));
  const int px = yi * a.W + xi;
  const double d = __ldg(&a.depth[px]);
  const double sdf = __dsub_rn(d, cam[2]);
  const bool hit = inside && d > 0.0 && fabs(sdf) <= a.trunc;
  if (MODE == 0) {
    const int any = __syncthreads_or(hit);
    if (v == 0) a.flags[b] = any ? 1 : 0;
    return;
  }
  if (slot < 0) return;  // EVAL-only blocks, or blocks the host did not admit
  double wgt = 1.0;
  if (a.depth_weighting) wgt = cam[2] > 0.0 ? __ddiv_rn(1.0, fmax(cam[2], 1e-6)) : 0.0;
  const float w = (float)wgt;
  const float wd = (float)__dmul_rn(wgt, sdf);
  float wc[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) wc[q] = (float)__dmul_rn(wgt, (double)a.color[3 * px + q]);
  float* W_ = a.weight + (size_t)slot * 512;
  float* D_ = a.wdist + (size_t)slot * 512;
  float* C_ = a.wcolor + (size_t)slot * 1536;
  const float s = a.sign;
  const bool upd = hit;
  float nw = W_[v];
  if (upd) nw = __fadd_rn(nw, __fmul_rn(s, w));
  if (MODE == 1) {
    const int neg = __syncthreads_or(nw < -1e-6f);
    if (v == 0) a.flags[b] = neg ? 1 : 0;
    return;
  }
  // COMMIT
  float nd = D_[v], nc0 = C_[3 * v], nc1 = C_[3 * v + 1], nc2 = C_[3 * v + 2];
  if (upd) {
    nd = __fadd_rn(nd, __fmul_rn(s, wd));
    nc0 = __fadd_rn(nc0, __fmul_rn(s, wc[0]));
    nc1 = __fadd_rn(nc1, __fmul_rn(s, wc[1]));
    nc2 = __fadd_rn(nc2, __fmul_rn(s, wc[2]));
  }
  if (s < 0.0f && a.hit[b] && b < a.snap_end) {  // touched blocks only (tsdf.py:146-155)
    if (fabsf(nw) <= 1e-6f && nw != 0.0f) nw = 0.0f;  // snap float dust only
    if (nw == 0.0f) nd = nc0 = nc1 = nc2 = 0.0f;
  }
  W_[v] = nw;
  D_[v] = nd;
  C_[3 * v] = nc0;
  C_[3 * v + 1] = nc1;
  C_[3 * v + 2] = nc2;
  const int nonzero = __syncthreads_or(nw != 0.0f);
  if (v == 0) a.flags[b] = nonzero ? 0 : 1;  // 1: block is empty
}

// zero pool slots (freed blocks; a fresh slot must read as an empty block)
__global__ void k_tsdf_zero(const int* slots, int n, float* weight, float* wdist, float* wcolor) {
  const int s = slots[blockIdx.x];
  for (int v = threadIdx.x; v < 512; v += blockDim.x) {
    weight[(size_t)s * 512 + v] = 0.0f;
    wdist[(size_t)s * 512 + v] = 0.0f;
  }
  for (int v = threadIdx.x; v < 1536; v += blockDim.x) wcolor[(size_t)s * 1536 + v] = 0.0f;
}

// gather (dir 0: pool -> packed) or scatter (dir 1: packed -> pool) whole blocks
__global__ void k_tsdf_copy(const int* slots, int n, int dir, float* weight, float* wdist,
                            float* wcolor, float* pw, float* pd, float* pc) {
  const int b = blockIdx.x;
  const size_t s = (size_t)slots[b];
  for (int v = threadIdx.x; v < 512; v += blockDim.x) {
    if (dir == 0) {
      pw[(size_t)b * 512 + v] = weight[s * 512 + v];
      pd[(size_t)b * 512 + v] = wdist[s * 512 + v];
    } else {
      weight[s * 512 + v] = pw[(size_t)b * 512 + v];
      wdist[s * 512 + v] = pd[(size_t)b * 512 + v];
    }
  }
  for (int v = threadIdx.x; v < 1536; v += blockDim.x) {
    if (dir == 0) pc[(size_t)b * 1536 + v] = wcolor[s * 1536 + v];
    else wcolor[s * 1536 + v] = pc[(size_t)b * 1536 + v];
  }
}

cudaError_t launch_tsdf_zero(const int* slots, int n, float* w, float* d, float* c, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  sfb_count_launch();
  k_tsdf_zero<<<n, 256, 0, s>>>(slots, n, w, d, c);
  return cudaGetLastError();
}

cudaError_t launch_tsdf_copy(const int* slots, int n, int dir, float* w, float* d, float* c,
                             float* pw, float* pd, float* pc, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  sfb_count_launch();
  k_tsdf_copy<<<n, 256, 0, s>>>(slots, n, dir, w, d, c, pw, pd, pc);
  return cudaGetLastError();
}

cudaError_t launch_tsdf_touch(const TsdfTouchArgs& a, cudaStream_t s) {
  const int n = a.W * a.H;
  if (n <= 0) return cudaSuccess;
  sfb_count_launch();
  k_tsdf_touch<<<(n + 255) / 256, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_tsdf_voxels(const TsdfVoxelArgs& a, int mode, int n_blocks, cudaStream_t s) {
  if (n_blocks <= 0) return cudaSuccess;
  sfb_count_launch();
  if (mode == 0) k_tsdf_voxels<0><<<n_blocks, 512, 0, s>>>(a);
  else if (mode == 1) k_tsdf_voxels<1><<<n_blocks, 512, 0, s>>>(a);
  else k_tsdf_voxels<2><<<n_blocks, 512, 0, s>>>(a);
  return cudaGetLastError();
}

// np.unique of the packed keys: radix sort + run-length dedup (CUB).
cudaError_t tsdf_sort_unique(long long* keys, long long* tmp_keys, int n, void* temp,
                             size_t* temp_bytes, int* d_count, cudaStream_t s) {
  size_t b1 = 0, b2 = 0;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, b1, keys, tmp_keys, n, 0, 64, s);
  if (e != cudaSuccess) return e;
  e = cub::DeviceSelect::Unique(nullptr, b2, tmp_keys, keys, d_count, n, s);
  if (e != cudaSuccess) return e;
  const size_t need = b1 > b2 ? b1 : b2;
  if (temp == nullptr) {
    *temp_bytes = need;
    return cudaSuccess;
  }
  if (*temp_bytes < need) return cudaErrorInvalidValue;
  e = cub::DeviceRadixSort::SortKeys(temp, b1, keys, tmp_keys, n, 0, 64, s);
  if (e != cudaSuccess) return e;
  sfb_count_launch(2);
  return cub::DeviceSelect::Unique(temp, b2, tmp_keys, keys, d_count, n, s);
}
