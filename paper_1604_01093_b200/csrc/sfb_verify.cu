// Dense two-sided consistency check of a relative transform (dense_verify,
// reference filters.py:216-277), one CTA per (frame pair, direction).
//
// A direction reprojects every source pixel with valid_depth & valid_normal
// into the destination frame (RigidTransform.apply + project_many + np.round,
// geometry.py:139-146,219-227), gathers the destination point / normal at the
// rounded pixel and the bilinear destination intensity at the continuous one
// (interp.py:8-33), and keeps the pixel when all three gates pass.  Every
// decision reproduces NumPy's rounding (separate mul/div/add, BLAS FMA chain
// orders passed in by the host probe, round-half-even, sequential 3-term
// norm/sum), so the per-direction counts are bit-exact; the mean error is the
// NumPy pairwise sum (numpy pairwise_sum: blocks of <= 128 with 8
// accumulators, halves split at n/2 rounded down to a multiple of 8) of the
// good distances in row-major order, so it is bit-exact too.
//
// Layout: each warp scans a contiguous pixel segment and appends its good
// distances in order to its own shared-memory segment (no CTA barrier in the
// scan); the pairwise tree (leaves in parallel, the combine on one thread)
// then reads the segments in global order.  <= 25,600 source pixels (200 KB).
#include "sfb_kernels.cuh"

#define VERIFY_THREADS 512
#define VERIFY_WARPS (VERIFY_THREADS / 32)
#define VERIFY_MAX_LEAVES 512

// bilinear_sample (interp.py:17-33) of a single-channel f32 image, NumPy
// evaluation order, no contraction.
__device__ __forceinline__ double bilinear1_exact(const float* img, int w, int h, double x,
                                                  double y) {
  x = fmin(fmax(x, 0.0), (double)w - 1.0);  // np.clip(x, 0.0, w - 1.0)
  y = fmin(fmax(y, 0.0), (double)h - 1.0);
  const int x0 = min((int)floor(x), w - 2);
  const int y0 = min((int)floor(y), h - 2);
  const double fx = __dsub_rn(x, (double)x0), fy = __dsub_rn(y, (double)y0);
  const double v00 = __ldg(&img[y0 * w + x0]), v01 = __ldg(&img[y0 * w + x0 + 1]);
  const double v10 = __ldg(&img[(y0 + 1) * w + x0]), v11 = __ldg(&img[(y0 + 1) * w + x0 + 1]);
  const double gx = __dsub_rn(1.0, fx), gy = __dsub_rn(1.0, fy);
  const double a = __dmul_rn(__dmul_rn(v00, gx), gy);
  const double b = __dmul_rn(__dmul_rn(v01, fx), gy);
  const double c = __dmul_rn(__dmul_rn(v10, gx), fy);
  const double d = __dmul_rn(__dmul_rn(v11, fx), fy);
  return __dadd_rn(__dadd_rn(__dadd_rn(a, b), c), d);
}

// Sequential reader of the compacted good distances stored as per-warp
// segments: global index i lives at gd[w*seg + i - off[w]].
struct SegReader {
  const double* gd;
  const int* off;
  int seg;
  int i;
  int w = 0;
  __device__ __forceinline__ double next() {
    while (i >= off[w + 1]) ++w;
    return gd[w * seg + (i++ - off[w])];
  }
};

// NumPy pairwise_sum leaf: n < 8 sequential from 0.0; n <= 128 eight strided
// accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail.
__device__ double pairwise_leaf(SegReader a, int n) {
  if (n < 8) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = __dadd_rn(s, a.next());
    return s;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a.next();
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a.next());
  double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                       __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) s = __dadd_rn(s, a.next());
  return s;
}

__global__ void __launch_bounds__(VERIFY_THREADS) k_dense_verify(const VerifyItem* items,
                                                                 VerifyCfg cfg, double* err_out,
                                                                 long long* cnt_out) {
  extern __shared__ double gd[];  // good distances, row-major order
  __shared__ int warp_cnt[VERIFY_WARPS];
  __shared__ int leaf_lo[VERIFY_MAX_LEAVES], leaf_n[VERIFY_MAX_LEAVES];
  __shared__ double leaf_v[VERIFY_MAX_LEAVES];
  __shared__ short ops[2 * VERIFY_MAX_LEAVES];  // post-order: >= 0 leaf id, -1 add
  __shared__ int n_leaves, n_ops;
  const VerifyItem& it = items[blockIdx.x];
  const FrameDev S = it.src, D = it.dst;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int hw = S.w * S.h;
  // (m, 3) @ R.T: NumPy takes the gemv path when m == 1 (eligible pixels)
  const int ord = S.n_valid_geo == 1 ? it.ord_1 : it.ord_n;
  Xf X;
#pragma unroll
  for (int k = 0; k < 9; ++k) X.R[k] = it.R[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) X.t[k] = it.t[k];
  const unsigned both = SFB_FLAG_VD | SFB_FLAG_VN;
  // warp w owns the contiguous pixel segment [w*seg, (w+1)*seg) and appends
  // its good distances, in order, at gd[w*seg ...]: no CTA barrier in the loop
  const int seg = ((hw + VERIFY_WARPS - 1) / VERIFY_WARPS + 31) & ~31;
  const int p_begin = wid * seg, p_end = min(hw, p_begin + seg);
  int wcount = 0;  // warp-uniform
  for (int p0 = p_begin; p0 < p_end; p0 += 32) {
    const int p = p0 + lane;
    bool good = false;
    double dist = 0.0;
    if (p < p_end) {
      const float4 P = __ldg(&S.P[p]);
      if ((__float_as_uint(P.w) & both) == both) {
        double q[3], u, v;
        bool front;
        xf_apply_exact(X, P.x, P.y, P.z, ord, q);  // transform.apply(points)
        project_exact(D.fx, D.fy, D.cx, D.cy, q, &u, &v, &front);
        const double xr = rint(u), yr = rint(v);  // np.round: half to even
        if (front && xr >= 0.0 && xr < (double)D.w && yr >= 0.0 && yr < (double)D.h) {
          const int ti = (int)yr * D.w + (int)xr;
          const float4 PT = __ldg(&D.P[ti]);
          if ((__float_as_uint(PT.w) & both) == both) {
            const float4 N = __ldg(&S.N[p]);
            const float4 NT = __ldg(&D.N[ti]);
            // distance = np.linalg.norm(moved - dst_points, axis=1)
            const double x0 = __dsub_rn(q[0], (double)PT.x);
            const double x1 = __dsub_rn(q[1], (double)PT.y);
            const double x2 = __dsub_rn(q[2], (double)PT.z);
            dist = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x0, x0), __dmul_rn(x1, x1)),
                                        __dmul_rn(x2, x2)));
            // normal_dot = np.sum(transform.rotate(normals) * dst_normals, axis=1)
            double nr[3];
            xf_rotate_exact(X, N.x, N.y, N.z, ord, nr);
            const double nd = __dadd_rn(__dadd_rn(__dmul_rn(nr[0], (double)NT.x),
                                                  __dmul_rn(nr[1], (double)NT.y)),
                                        __dmul_rn(nr[2], (double)NT.z));
            // color_diff = |intensity - bilinear_sample(intensity_dst, u, v)|
            const double cd =
                fabs(__dsub_rn((double)__ldg(&S.I[p]), bilinear1_exact(D.I, D.w, D.h, u, v)));
            good = dist < cfg.depth_max && nd > cfg.normal_min && cd < cfg.color_max;
          }
        }
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, good);
    if (good) gd[p_begin + wcount + __popc(bal & ((1u << lane) - 1u))] = dist;
    wcount += __popc(bal);
  }
  if (lane == 0) warp_cnt[wid] = wcount;
  __syncthreads();
  __shared__ int seg_off[VERIFY_WARPS + 1];
  if (tid == 0) {
    int acc = 0;
    for (int w = 0; w < VERIFY_WARPS; ++w) {
      seg_off[w] = acc;
      acc += warp_cnt[w];
    }
    seg_off[VERIFY_WARPS] = acc;
  }
  __syncthreads();
  const int base = seg_off[VERIFY_WARPS];
  const int n = base;
  // numpy pairwise_sum tree over gd[0..n): leaves and post-order ops
  if (tid == 0) {
    int st_lo[40], st_n[40];
    bool st_x[40];
    int sp = 0, nl = 0, no = 0;
    st_lo[0] = 0;
    st_n[0] = n;
    st_x[0] = false;
    sp = 1;
    while (sp > 0) {
      --sp;
      const int lo = st_lo[sp], m = st_n[sp];
      const bool expanded = st_x[sp];
      if (m <= 128) {
        leaf_lo[nl] = lo;
        leaf_n[nl] = m;
        ops[no++] = (short)nl++;
      } else if (expanded) {
        ops[no++] = -1;
      } else {
        int n2 = m / 2;
        n2 -= n2 % 8;
        st_lo[sp] = lo; st_n[sp] = m; st_x[sp] = true; ++sp;                // the add, last
        st_lo[sp] = lo + n2; st_n[sp] = m - n2; st_x[sp] = false; ++sp;     // right
        st_lo[sp] = lo; st_n[sp] = n2; st_x[sp] = false; ++sp;              // left, first
      }
    }
    n_leaves = nl;
    n_ops = no;
  }
  __syncthreads();
  for (int k = tid; k < n_leaves; k += VERIFY_THREADS)
    leaf_v[k] = pairwise_leaf(SegReader{gd, seg_off, seg, leaf_lo[k]}, leaf_n[k]);
  __syncthreads();
  if (tid == 0) {
    double vs[40];
    int sp = 0;
    for (int k = 0; k < n_ops; ++k) {
      if (ops[k] >= 0) {
        vs[sp++] = leaf_v[ops[k]];
      } else {
        const double r = vs[--sp];
        const double l = vs[--sp];
        vs[sp++] = __dadd_rn(l, r);
      }
    }
    const double sum = sp ? vs[0] : 0.0;
    err_out[blockIdx.x] = n ? __ddiv_rn(sum, (double)n) : 0.0;
    cnt_out[blockIdx.x] = n;
  }
}

int verify_max_pixels() { return (200 * 1024) / 8; }

cudaError_t launch_dense_verify(const VerifyItem* items, int n_items, int max_src_hw,
                                const VerifyCfg& cfg, double* err, long long* cnt,
                                cudaStream_t s) {
  if (n_items <= 0) return cudaSuccess;
  // per-warp segments of ceil(hw / warps) rounded up to 32 pixels
  const int seg = ((max_src_hw + VERIFY_WARPS - 1) / VERIFY_WARPS + 31) & ~31;
  const size_t smem = (size_t)VERIFY_WARPS * seg * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_dense_verify, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  sfb_count_launch();
  k_dense_verify<<<n_items, VERIFY_THREADS, smem, s>>>(items, cfg, err, cnt);
  return cudaGetLastError();
}
