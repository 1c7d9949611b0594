// Frame-pair filter: build_dense_edges (solver.py:130-148) with
// view_angle_deg and frustum_overlap (frames.py:154-188), bit-exact.
//
//  k_angle_gate  one thread per pair a<b: clip(z_a . z_b) >= cos_min, the dot
//                in NumPy's np.dot FMA order.  cos_min is the exact preimage
//                of `degrees(arccos(c)) < view_angle_max_deg` (host bisection).
//  k_overlap_prefilter + k_overlap_culled   the solver's path: a thread per
//                candidate classifies bounding spheres of 16x16 tiles, and only
//                the undecided pairs get the exact per-point test (queue).
//  k_overlap     one CTA per candidate pair, both directions; each direction
//                maps the source's valid points through pose_b^-1 o pose_a
//                with NumPy's rounding and stops at the first point inside
//                the target frustum (overlap > 0 <=> at least one inside),
//                __syncthreads_or per 256-pixel chunk.  full_count mode counts
//                every point instead (frustum_overlap's fraction).
#include "sfb_kernels.cuh"

#include <algorithm>

__global__ void k_angle_gate(const PoseDev* poses, int n, Rounding rd, double cos_min,
                             uint8_t* flags) {
  const int a = blockIdx.y;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b <= a || b >= n) return;
  const PoseDev& A = poses[a];
  const PoseDev& B = poses[b];
  // z axes = rotation[:, 2]
  double d = dot3o(A.R[2], A.R[5], A.R[8], B.R[2], B.R[5], B.R[8], rd.dot3);
  d = fmin(fmax(d, -1.0), 1.0);
  const int64_t q = (int64_t)a * n - ((int64_t)a * (a + 1)) / 2 + (b - a - 1);
  flags[q] = d >= cos_min ? 1 : 0;
}

void launch_angle_gate(const PoseDev* poses, int n, Rounding rd, double cos_min, uint8_t* flags,
                       cudaStream_t s) {
  if (n < 2) return;
  dim3 grid((n + 255) / 256, n - 1);
  sfb_count_launch();
  k_angle_gate<<<grid, 256, 0, s>>>(poses, n, rd, cos_min, flags);
}

__device__ __forceinline__ bool point_inside(const Xf& rel, const FrameDev& Fb, const float4 P,
                                             int ord) {
  double q[3], u, v;
  bool front;
  xf_apply_exact(rel, (double)P.x, (double)P.y, (double)P.z, ord, q);
  project_exact(Fb.fx, Fb.fy, Fb.cx, Fb.cy, q, &u, &v, &front);
  return front && u >= 0.0 && u <= (double)(Fb.w - 1) && v >= 0.0 && v <= (double)(Fb.h - 1);
}

__global__ void __launch_bounds__(256) k_overlap(const FrameDev* frames, const PoseDev* poses,
                                                 const int2* cand, Rounding rd, int full_count,
                                                 uint8_t* pass, int* counts) {
  __shared__ Xf rel[2];
  __shared__ int red[8];
  const int2 ab = cand[blockIdx.x];
  if (threadIdx.x < 2) {
    const int s = threadIdx.x == 0 ? ab.x : ab.y;
    const int t = threadIdx.x == 0 ? ab.y : ab.x;
    rel[threadIdx.x] = xf_relative_exact(poses[s], poses[t], rd);
  }
  __syncthreads();
  bool ok = true;
  for (int dir = 0; dir < 2 && ok; ++dir) {
    const FrameDev Fa = frames[dir == 0 ? ab.x : ab.y];
    const FrameDev Fb = frames[dir == 0 ? ab.y : ab.x];
    const int hw = Fa.w * Fa.h;
    const int ord = Fa.n_valid_depth == 1 ? rd.apply_1 : rd.apply_n;
    if (full_count) {
      int c = 0;
      for (int p = threadIdx.x; p < hw; p += blockDim.x) {
        const float4 P = __ldg(&Fa.P[p]);
        if ((__float_as_uint(P.w) & SFB_FLAG_VD) && point_inside(rel[dir], Fb, P, ord)) ++c;
      }
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
      __syncthreads();
      if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < 8; ++w) t += red[w];
        counts[2 * blockIdx.x + dir] = t;
      }
      __syncthreads();
      continue;
    }
    bool found = false;
    for (int base = 0; base < hw; base += blockDim.x) {
      const int p = base + threadIdx.x;
      bool in = false;
      if (p < hw) {
        const float4 P = __ldg(&Fa.P[p]);
        in = (__float_as_uint(P.w) & SFB_FLAG_VD) && point_inside(rel[dir], Fb, P, ord);
      }
      if (__syncthreads_or(in)) {
        found = true;
        break;
      }
    }
    ok = found;
  }
  if (!full_count && threadIdx.x == 0) pass[blockIdx.x] = ok ? 1 : 0;
}

// Tile culling.  A tile's bounding sphere, moved by the (plainly rounded)
// relative pose, is classified against the target frustum's five half-spaces
// n.q >= 0 (n = (fx,0,cx), (-fx,0,w-1-cx), (0,fy,cy), (0,-fy,h-1-cy)) and
// q_z > 0.  The radius carries a 1e-7 m margin, far above the ~1e-13 m error
// of the plain transform and of NumPy's own rounding, so "no point inside"
// and "every point inside" hold for the exactly-rounded per-point test too:
// culling never changes a decision, it only skips work.
__device__ __forceinline__ int classify_tile(const Xf& rel, const double4 s, const FrameDev& Fb) {
  if (s.w < 0.0) return 0;
  double c[3];
  xf_apply(rel.R, rel.t, s.x, s.y, s.z, c);
  const double r = s.w * (1.0 + 1e-7) + 1e-7;
  const double wm1 = (double)(Fb.w - 1), hm1 = (double)(Fb.h - 1);
  const double n[4][3] = {{Fb.fx, 0.0, Fb.cx}, {-Fb.fx, 0.0, wm1 - Fb.cx},
                          {0.0, Fb.fy, Fb.cy}, {0.0, -Fb.fy, hm1 - Fb.cy}};
  bool all_in = c[2] - r > 0.0;
  if (c[2] + r <= 0.0) return 0;
  for (int k = 0; k < 4; ++k) {
    const double d = n[k][0] * c[0] + n[k][1] * c[1] + n[k][2] * c[2];
    const double nn = sqrt(n[k][0] * n[k][0] + n[k][1] * n[k][1] + n[k][2] * n[k][2]);
    if (d + r * nn < 0.0) return 0;
    if (d - r * nn <= 0.0) all_in = false;
  }
  return all_in ? 1 : 2;
}

// Stage 1, one thread per candidate: both directions' tiles classified with a
// plainly rounded relative pose (error ~1e-15 m << the 1e-7 m margin), which
// settles most pairs for good - every tile of a direction outside the target
// frustum (no overlap), or a fully-inside tile holding a valid point in both
// directions (overlap both ways).  The rest are queued for stage 2.
__global__ void __launch_bounds__(256) k_overlap_prefilter(const FrameDev* frames,
                                                           const PoseDev* poses, const int2* cand,
                                                           int n_cand, uint8_t* pass, int* need,
                                                           int* n_need, int rank, int world) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cand) return;
  if (world > 1 && c % world != rank) {  // another rank's candidate
    pass[c] = 0;
    return;
  }
  const int2 ab = cand[c];
  int verdict = 1;  // 1 pass, 0 fail, 2 undecided
  for (int dir = 0; dir < 2 && verdict != 0; ++dir) {
    const int sa = dir == 0 ? ab.x : ab.y, sb = dir == 0 ? ab.y : ab.x;
    const PoseDev& Pa = poses[sa];
    const PoseDev& Pb = poses[sb];
    // rel = pose_b^-1 o pose_a, plain rounding
    Xf rel;
    double iR[9], it[3];
    xf_inverse_plain(Pb.R, Pb.t, iR, it);
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
      for (int q = 0; q < 3; ++q)
        rel.R[r * 3 + q] = iR[r * 3] * Pa.R[q] + iR[r * 3 + 1] * Pa.R[3 + q] + iR[r * 3 + 2] * Pa.R[6 + q];
      rel.t[r] = iR[r * 3] * Pa.t[0] + iR[r * 3 + 1] * Pa.t[1] + iR[r * 3 + 2] * Pa.t[2] + it[r];
    }
    const FrameDev& Fa = frames[sa];
    const FrameDev& Fb = frames[sb];
    const int nt = Fa.tiles_x * Fa.tiles_y;
    bool in_dir = false, partial = false;
    for (int t = 0; t < nt && !in_dir; ++t) {
      const int cls = classify_tile(rel, Fa.tiles[t], Fb);
      if (cls == 1 && Fa.tile_count[t] > 0) in_dir = true;
      else if (cls == 2) partial = true;
    }
    if (!in_dir) verdict = partial ? 2 : 0;
  }
  if (verdict == 2) {
    need[atomicAdd(n_need, 1)] = c;
  } else {
    pass[c] = verdict ? 1 : 0;
  }
}

// Stage 2 (persistent CTAs over the queue): the exact per-point test in the
// partially visible tiles, as frustum_overlap with NumPy's rounding.
__global__ void __launch_bounds__(256) k_overlap_culled(const FrameDev* frames, const PoseDev* poses,
                                                        const int2* cand, Rounding rd,
                                                        uint8_t* pass, const int* need,
                                                        const int* n_need) {
  __shared__ Xf rel[2];
  __shared__ int partial[1024];
  __shared__ int n_partial;
  const int nq = *n_need;
  for (int k = blockIdx.x; k < nq; k += gridDim.x) {
    const int c = need[k];
    const int2 ab = cand[c];
    if (threadIdx.x < 2) {
      const int s = threadIdx.x == 0 ? ab.x : ab.y;
      const int t = threadIdx.x == 0 ? ab.y : ab.x;
      rel[threadIdx.x] = xf_relative_exact(poses[s], poses[t], rd);
    }
    __syncthreads();
    bool ok = true;
    for (int dir = 0; dir < 2 && ok; ++dir) {
      const FrameDev Fa = frames[dir == 0 ? ab.x : ab.y];
      const FrameDev Fb = frames[dir == 0 ? ab.y : ab.x];
      const int ord = Fa.n_valid_depth == 1 ? rd.apply_1 : rd.apply_n;
      const int nt = Fa.tiles_x * Fa.tiles_y;
      bool found = false;
      for (int t0 = 0; t0 < nt && !found; t0 += 1024) {
        if (threadIdx.x == 0) n_partial = 0;
        __syncthreads();
        bool any_in = false;
        for (int t = t0 + threadIdx.x; t < min(nt, t0 + 1024); t += blockDim.x) {
          const int cls = classify_tile(rel[dir], Fa.tiles[t], Fb);
          if (cls == 1 && Fa.tile_count[t] > 0) any_in = true;
          if (cls == 2) partial[atomicAdd(&n_partial, 1)] = t;
        }
        if (__syncthreads_or(any_in)) {
          found = true;
          break;
        }
        const int np = n_partial;
        for (int q = 0; q < np && !found; ++q) {
          const int t = partial[q];
          const int x = (t % Fa.tiles_x) * SFB_TILE + (threadIdx.x % SFB_TILE);
          const int y = (t / Fa.tiles_x) * SFB_TILE + (threadIdx.x / SFB_TILE);
          bool in = false;
          if (x < Fa.w && y < Fa.h) {
            const float4 P = __ldg(&Fa.P[y * Fa.w + x]);
            in = (__float_as_uint(P.w) & SFB_FLAG_VD) && point_inside(rel[dir], Fb, P, ord);
          }
          if (__syncthreads_or(in)) found = true;
        }
        __syncthreads();
      }
      ok = found;
    }
    if (threadIdx.x == 0) pass[c] = ok ? 1 : 0;
    __syncthreads();  // rel / partial are rewritten by the next queued candidate
  }
}

void launch_overlap(const FrameDev* frames, const PoseDev* poses, const int2* cand, int n_cand,
                    Rounding rd, int full_count, uint8_t* pass, int* counts, cudaStream_t s,
                    int rank, int world, int* need, int* n_need, int n_sm) {
  if (n_cand <= 0) return;
  if (full_count) {
    sfb_count_launch();
    k_overlap<<<n_cand, 256, 0, s>>>(frames, poses, cand, rd, full_count, pass, counts);
    return;
  }
  cudaMemsetAsync(n_need, 0, sizeof(int), s);
  sfb_count_launch(2);
  k_overlap_prefilter<<<(n_cand + 255) / 256, 256, 0, s>>>(frames, poses, cand, n_cand, pass, need,
                                                           n_need, rank, world);
  const int grid = std::min(n_cand, 8 * n_sm);  // persistent over the (device-sized) queue
  k_overlap_culled<<<grid, 256, 0, s>>>(frames, poses, cand, rd, pass, need, n_need);
}
