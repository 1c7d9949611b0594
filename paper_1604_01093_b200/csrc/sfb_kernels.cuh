// sfb_kernels.cuh — launcher declarations shared by the kernel TUs and the ABI.
#pragma once
#include "sfb_internal.cuh"

struct PackArgs {
  const uint8_t* vd;
  const uint8_t* vn;
  const float* pts;
  const float* nrm;
  const float* grad;
  float4* P;
  float4* N;
  float2* G;
  float4* T;
  int w, h;
  int* counts;  // [0] valid_depth, [1] valid_depth & valid_normal, [2] non-finite
  int tiles_x, tiles_y;
  double4* tiles;
  int* tile_count;
};

struct SparseArgs {
  const PoseDev* poses;
  const int* set_fi;
  const int* set_fj;
  const int64_t* set_off;   // set s covers [set_off[s], set_end[s])
  const int64_t* set_end;
  const double* pts_i;
  const double* pts_j;
  double* world_i;     // may be null (energy-only)
  double* world_j;
  double* set_out;     // SFB_SET_STRIDE per set
  int n_sets;
  double w_sparse;
  int energy_only;
};

struct DenseArgs {
  const FrameDev* frames;
  const PoseDev* poses;
  const int4* items;        // (dir edge, begin, end, 0)
  const int2* dir_edges;    // (src frame, dst frame)
  double* edge_rel;         // scratch: 12 f64 per directed edge (relative transforms), or null
  int n_dir;
  const int64_t* photo_off; // per dir edge: u32-word offset
  const int64_t* geo_off;   // per dir edge: u16 offset
  uint32_t* photo_mask;
  uint16_t* geo_tgt;
  const uint32_t* photo_mask_prev;  // previous linearisation's frozen sets (fused
  const uint16_t* geo_tgt_prev;     // energy-after), or null
  int prev_photo, prev_geo;         // which frozen terms the previous pass produced
  uint8_t* tile_any;                // per (edge, source tile): any frozen association
  const uint8_t* tile_any_prev;
  double* item_out;         // SFB_ITEM_STRIDE per item
  Rounding rd;
  double s_photo, s_geo;
  int do_photo, do_geo;
  double geo_dmax, geo_nmin;
  int stride;
  // per frame, valid_depth / geo pixel counts on the stride grid (stride > 1;
  // the m == 1 NumPy rounding case of _source_pixel_data, solver.py:158-167)
  const int2* stride_counts;
  int n_items;
};

struct AssembleArgs {
  int n_blk;
  int n_pairs;
  const double* set_out;
  const double* edge_out;
  const int* d_ptr;   // per var: D/g contribution list
  const int* d_ent;
  const int* b_ptr;   // per pair: B contribution list
  const int* b_ent;
  double* D;          // n_blk * 36
  double* B;          // n_pairs * 36
  double* g;          // n_blk * 6
  const int* row_ptr;    // matvec slots: row_ptr[v] is v's diagonal slot
  const int* pair_slot;  // 2 per pair: slot in row a (as is), in row b (transposed)
  double* Brow;          // slots * 36
  double* jdiag;         // n_blk * 6 Jacobi diagonal (solver.py:412-428), or null
  int dense_on;
};

struct PcgArgs {
  int n_blk;
  const double* Brow;  // slot blocks, row-major, oriented for their row
  const int* row_ptr;  // slots of row v: [row_ptr[v], row_ptr[v+1]), first = diagonal
  const int* row_col;  // column block of each slot
  const double* g;
  double* x;
  double* r;
  double* z;
  double* p;
  double* p2;          // ping-pong partner of p
  double* Ap;
  double* inv_diag;
  double* b;
  const double* jdiag; // _jacobi_diagonal (solver.py:412-428)
  double* part;        // 4 * gridDim
  int* flags;          // scratch
  int max_it;
  double tol;
  int restart;
  double* out_scalars; // [0] iterations, [1] relative, [2] status
  const double* skip;  // optional: skip when *skip != 0
  const double* bj_inv;  // block-Jacobi inverses (n_blk x 36) or null: scalar Jacobi
};

// dense_verify (filters.py:216-277): one item = one direction of one pair
struct VerifyItem {
  FrameDev src, dst;
  double R[9], t[3];  // transform src -> dst (row-major R)
  int ord_n, ord_1;   // NumPy (m,3) @ R.T FMA chain order for m > 1 / m == 1
};
struct VerifyCfg {
  double depth_max, normal_min, color_max;
};

// build_cache (frames.py:75-151): per-frame device planes
struct CacheFrame {
  const uint8_t* color;   // (H, W, 3)
  const float* depth_in;  // (H, W)
  float* intensity;       // (h, w)       -- the host image layout, in order:
  float* depth;           // (h, w)          intensity, depth, points, normals,
  float* points;          // (h, w, 3)       grad (f32), valid, valid_n (u8)
  float* normals;         // (h, w, 3)
  float* grad;            // (h, w, 2)
  uint8_t* valid;         // (h, w)
  uint8_t* valid_n;       // (h, w)
};
struct CacheArgs {
  const CacheFrame* frames;
  int W, H, low_w, low_h, bw, bh;
  double fx, fy, cx, cy;  // intrinsics.scaled(low_w, low_h)
  int luma_order;
};

// hashed TSDF (tsdf.py:55-201)
struct TsdfTouchArgs {
  const float* depth;  // (H, W)
  int W, H;
  double fx, fy, cx, cy;
  Xf pose;             // camera -> world
  int ord;             // NumPy order of (m,3) @ pose.rotation.T
  double trunc, extent;
  const double* t;     // np.linspace(0, 1, n_samples), from the host
  int n_samples;
  long long* keys;     // W*H*n_samples
};
struct TsdfVoxelArgs {
  const long long* keys;  // sorted unique touched block keys
  const int* slots;       // pool slot per touched block (-1: skip)
  const unsigned char* hit;  // EVAL result per touched block
  unsigned char* flags;   // per touched block: EVAL hit / CHECK negative / COMMIT empty
  int first;              // first touched block of this launch
  int snap_end;           // de-integration snaps/clears only touched blocks below this
  double extent, vs, trunc;
  Xf inv_pose;            // pose.inverse(), NumPy rounding (host)
  int ord;
  double fx, fy, cx, cy;
  int W, H;
  const float* depth;
  const uint8_t* color;   // (H, W, 3)
  int depth_weighting;
  float sign;
  float* weight;          // pool: slot * 512
  float* wdist;
  float* wcolor;          // slot * 1536
};

// one host -> device byte copy (pinned source, read through UVA)
struct CopyJob {
  const uint8_t* src;
  uint8_t* dst;
  size_t n;
};
cudaError_t launch_stage_copy(const CopyJob* jobs, int n_jobs, cudaStream_t s);

// Library-wide kernel launch counter (sfb_launch_count).
void sfb_count_launch(int n = 1);

// every frame of an upload in two launches (planes, then tile spheres)
void launch_pack_batch(const PackArgs* args_dev, int n, int max_hw, int max_tiles, cudaStream_t s);
void launch_sparse(const SparseArgs& a, cudaStream_t s);
void launch_dense_linearize(const DenseArgs& a, cudaStream_t s);
void launch_stride_counts(const FrameDev* frames, int n, int stride, int2* out, cudaStream_t s);
void launch_dense_energy(const DenseArgs& a, double* item_e2, cudaStream_t s);
void launch_block_jacobi_inv(const double* D, const double* jdiag, int n_blk, double* out,
                             cudaStream_t s);
// block-system structure (sfb_struct.cu)
void launch_struct_edges(const int2* edges, int n_e, int bidir, const FrameDev* frames,
                         int shard_rank, int shard_world, int target, int2* dir, int* icount,
                         int64_t* pcount, int64_t* gcount, int* per, cudaStream_t s);
void launch_struct_items(const int2* dir, int n_dir, const FrameDev* frames, const int* eptr,
                         const int* per, int4* items, cudaStream_t s);
void launch_struct_count(const int* set_fi, const int* set_fj, const int64_t* set_off,
                         const int64_t* set_end, int n_sets, const int2* dir, int n_dir,
                         int* dcount, int* bcount, cudaStream_t s);
void launch_struct_fill(const int* set_fi, const int* set_fj, const int64_t* set_off,
                        const int64_t* set_end, int n_sets, const int2* dir, int n_dir, int nb,
                        const int* doff, const int* boff, unsigned* dkey, int* dval, unsigned* bkey,
                        int* bval, cudaStream_t s);
void launch_struct_ptr(const unsigned* keys, int n, int rows, int* ptr, cudaStream_t s);
void launch_struct_pairs_count(const unsigned* unique_keys, const int* n_runs, int* n_pairs,
                               cudaStream_t s);
void launch_rows_keys(const unsigned* pair_key, const int* n_pairs_d, int nb, int n_max,
                      unsigned* hkey, int* hval, cudaStream_t s);
void launch_rows_out(const unsigned* hkey, const int* hval, const int* n_pairs_d, int nb, int n_max,
                     int* row_ptr, int* row_col, int* pair_slot, cudaStream_t s);
// sharded PCG (sfb_pcg_sharded.cu)
void launch_pcgs_init(const PcgArgs& a, double* st, cudaStream_t s);
void launch_pcgs_step(const PcgArgs& a, double* st, int k, int restart, cudaStream_t s);
void launch_pcgs_restart(const PcgArgs& a, double* st, cudaStream_t s);
int sys_pack_len(int n6, int with_d);
void launch_sys_pack(double* g, double* jdiag, double* dscal, double* D, int n6, int with_d,
                     double* buf, int unpack, cudaStream_t s);
void launch_matvec(const PcgArgs& a, const double* xin, double* yout, cudaStream_t s);
void launch_edge_reduce2(const int* edge_item_ptr, const double* item_e2, double* edge_e2, int n_dir,
                         cudaStream_t s);
void launch_edge_reduce(const int* edge_item_ptr, const double* item_out, double* edge_out,
                        int n_dir, const int2* dir_edges, const PoseDev* poses, cudaStream_t s,
                        double* const* peer_dst = nullptr, int rank = 0, int world = 1);
void launch_p2p_sync(unsigned* const* peer_flags, unsigned* my_flags, int rank, int world,
                     unsigned epoch, cudaStream_t s);
void launch_assemble(const AssembleArgs& a, cudaStream_t s);
// scratch: SUM_ENERGY_SCRATCH doubles, zero before the first launch
#define SUM_ENERGY_SCRATCH 168
void launch_sum_energies(const double* set_out, int n_sets, const double* edge_out, int n_dir,
                         const double* item_e2, int n_items, double* out3, int mode,
                         double* scratch, cudaStream_t s);
cudaError_t launch_pcg(const PcgArgs& a, int n_sm, cudaStream_t s);
cudaError_t launch_pcg_dense(const PcgArgs& a, const double* A, int n_sm, cudaStream_t s);
void launch_matvec(const PcgArgs& a, const double* xin, double* yout, cudaStream_t s);
void launch_pose_update(PoseDev* poses, int n_frames, const double* dx, double* step_norm,
                        const double* skip, cudaStream_t s);
void launch_angle_gate(const PoseDev* poses, int n, Rounding rd, double cos_min, uint8_t* flags,
                       cudaStream_t s);
void launch_overlap(const FrameDev* frames, const PoseDev* poses, const int2* cand, int n_cand,
                    Rounding rd, int full_count, uint8_t* pass, int* counts, cudaStream_t s,
                    int rank = 0, int world = 1, int* need = nullptr, int* n_need = nullptr,
                    int n_sm = 148);
void launch_associate(const DenseArgs& a, int src, int dst, int kind, uint8_t* sel, int* tgt,
                      cudaStream_t s);
void launch_point_eval(const FrameDev* frames, const PoseDev* poses, int src, int dst, int kind,
                       int64_t m, const double* pts, const double* aux, const double* tgts,
                       double* res, double* jac, cudaStream_t s);
cudaError_t launch_build_cache(const CacheArgs& a, int n_frames, cudaStream_t s);
cudaError_t launch_tsdf_touch(const TsdfTouchArgs& a, cudaStream_t s);
cudaError_t launch_tsdf_zero(const int* slots, int n, float* w, float* d, float* c, cudaStream_t s);
cudaError_t launch_tsdf_copy(const int* slots, int n, int dir, float* w, float* d, float* c,
                             float* pw, float* pd, float* pc, cudaStream_t s);
cudaError_t launch_tsdf_voxels(const TsdfVoxelArgs& a, int mode, int n_blocks, cudaStream_t s);
cudaError_t tsdf_sort_unique(long long* keys, long long* tmp_keys, int n, void* temp,
                             size_t* temp_bytes, int* d_count, cudaStream_t s);
int verify_max_pixels();
cudaError_t launch_dense_verify(const VerifyItem* items, int n_items, int max_src_hw,
                                const VerifyCfg& cfg, double* err, long long* cnt, cudaStream_t s);
void launch_sparse_residuals(const SparseArgs& a, double* res, double* set_max, cudaStream_t s);
