// sfb_abi.cu — extern "C" entry points of libsfb.so (see include/sfb.h) and
// the host-side bookkeeping behind them: frame store, problem handles, the
// block-system structure (which frame pairs couple), work decomposition of
// the dense term into (directed edge, pixel tile) items.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdlib>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "../../include/sfb.h"
#include "sfb_kernels.cuh"

static std::atomic<long long> g_launches{0};
void sfb_count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

#include "sfb_host.cuh"


struct sfb_problem : Handle {
  sfb_ctx* ctx = nullptr;
  cudaStream_t stream = nullptr;
  int n = 0;          // frames
  int n_blk = 0;      // variable blocks = n - 1
  bool has_frames = false;
  std::vector<int> slots;
  std::vector<FrameDev> frames_h;
  DBuf<FrameDev> frames;
  DBuf<PoseDev> poses, best;
  // sparse
  int n_sets = 0;
  int64_t n_corr = 0;
  std::vector<int> set_fi_h, set_fj_h;
  std::vector<int64_t> set_beg_h, set_end_h;  // per set [begin, end) into the correspondences
  DBuf<int> set_fi, set_fj;
  DBuf<int64_t> set_off;   // per set: first correspondence
  DBuf<int64_t> set_end;   // per set: one past its last correspondence
  DBuf<double> pts_i, pts_j, world_i, world_j, set_out;
  // dense
  std::vector<int2> edges;  // undirected (a < b in frame order)
  int struct_bidir = -1;
  int n_dir = 0, n_items = 0;
  DBuf<int2> dir_edges;
  DBuf<int4> items;
  DBuf<int> edge_item_ptr;
  DBuf<int64_t> photo_off, geo_off;
  DBuf<uint32_t> photo_mask[2];  // frozen associations, double-buffered so the
  DBuf<uint16_t> geo_tgt[2];     // next linearisation can evaluate the last one
  DBuf<uint8_t> tile_any[2];     // per (edge, source tile): any frozen association
  int cur = 0;                   // buffer holding the latest linearisation
  DBuf<double> item_out, edge_out, item_e2;
  DBuf<double> edge_rel;         // per directed edge: pose_j^-1 o pose_i (12 f64), per dense pass
  DBuf<int2> stride_counts;      // per frame source counts on the stride grid
  int stride_counts_for = 0;     // stride they were computed for (0: none)
  DBuf<double> edge_e2;          // frozen-energy sums per directed edge (2 each)
  bool dense_active = false;
  // between the two halves of a (possibly sharded) linearisation / energy
  bool pending_dense_on = false;
  int pending_prev_mode = 0;
  bool pending_gn_relin = false;
  // speculative PCG of the next GN iteration (sfb_gn_step_end)
  bool spec_pcg = false;
  int spec_pcg_args[2] = {0, 0};
  double spec_pcg_tol = 0.0;
  int spec_max_it = 0, spec_restart = 1;
  double spec_tol = 0.0;
  cudaEvent_t d2h_done = nullptr;
  bool pending_energy_dense = false;
  // data-parallel sharding over directed dense edges
  int shard_rank = 0, shard_world = 1;
  int shard_mode = 0;            // 0: exchange per-edge sums; 1: partial systems + sharded PCG
  // peer-memory exchange of the per-edge sums (sfb_set_p2p): IPC-mapped
  // edge_out / flag buffers of the other ranks
  bool p2p_on = false;
  DBuf<unsigned> p2p_flags;      // 64 slots: peers store their epochs here
  unsigned p2p_epoch = 0;
  std::vector<void*> p2p_open[2];  // opened peer pointers (edge_out, flags)
  DBuf<double*> peer_edge_d;
  DBuf<unsigned*> peer_flags_d;
  bool p2p_ready[2] = {false, false};
  DBuf<double> xsys;             // mode 1: packed [g | jdiag | dense energies | D]
  DBuf<double> pcgs_state;       // mode 1: PCG scalars (sfb_pcg_sharded)
  int n_cand = 0;                // pair-filter candidates of the last filter pass
  int last_do_photo = 0, last_do_geo = 0;
  // system
  int n_pairs = 0;
  DBuf<int> d_ptr, d_ent, b_ptr, b_ent, row_ptr, row_ent, row_col;
  DBuf<unsigned> pair_key;     // pair q = (a, b): a * n_blk + b, increasing
  DBuf<int2> edges_d;          // the undirected edges on the device
  struct {                     // rebuild_structure scratch
    DBuf<int> icount, per, dcount, bcount, doff, boff, dval, bval, runs, hval, hval2;
    DBuf<int64_t> pcount, gcount;
    DBuf<unsigned> dkey, dkey2, bkey, bkey2, hkey, hkey2;
    DBuf<double> scal;
    DBuf<uint8_t> temp;
  } sc;
  DBuf<double> D, B, g, Brow;  // Brow: row-major pre-oriented blocks for the matvec
  DBuf<double> pv2;            // second search-direction buffer (PCG ping-pong)
  DBuf<double> x, r, z, pv, Ap, inv_diag, bvec, part, tmp, jdiag;
  DBuf<int> flags;
  int precond = 0;             // 0: scalar Jacobi (reference), 1: block Jacobi (opt-in)
  DBuf<double> bj_inv;         // block-Jacobi inverses, n_blk x 36
  bool have_system = false;
  bool have_solution = false;
  // scalars
  DBuf<double> dscal;       // device scalars
  DBuf<double> esum;        // k_sum_energies scratch (CTA partials + ticket)
  double* hscal = nullptr;  // pinned mirror
  Prof prof;
  // pair-filter scratch
  DBuf<int2> f_all, f_cand, f_sel;
  DBuf<uint8_t> f_fl, f_pass, f_temp;
  DBuf<int> f_cnt;
  DBuf<int> f_need;  // [0] queue length, then the undecided candidates (pair filter stage 2)
};

namespace {


// Stable compaction of flagged elements (cub::DeviceSelect::Flagged).
template <class T>
cudaError_t select_flagged(const T* in, const uint8_t* flags, T* out, int* d_count, int n,
                           DBuf<uint8_t>& temp, cudaStream_t s) {
  size_t bytes = 0;
  cudaError_t e = cub::DeviceSelect::Flagged(nullptr, bytes, in, flags, out, d_count, n, s);
  if (e != cudaSuccess) return e;
  if ((e = temp.ensure(bytes)) != cudaSuccess) return e;
  return cub::DeviceSelect::Flagged(temp.p, bytes, in, flags, out, d_count, n, s);
}

__global__ void k_enumerate_pairs(int n, int2* out) {
  const int a = blockIdx.y;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b <= a || b >= n) return;
  const int64_t q = (int64_t)a * n - ((int64_t)a * (a + 1)) / 2 + (b - a - 1);
  out[q] = make_int2(a, b);
}

PcgArgs pcg_args(sfb_problem* p) {
  PcgArgs a{};
  a.n_blk = p->n_blk;
  a.Brow = p->Brow.p;
  a.row_ptr = p->row_ptr.p;
  a.row_col = p->row_col.p;
  a.p2 = p->pv2.p;
  a.g = p->g.p;
  a.x = p->x.p;
  a.r = p->r.p;
  a.z = p->z.p;
  a.p = p->pv.p;
  a.Ap = p->Ap.p;
  a.inv_diag = p->inv_diag.p;
  a.b = p->bvec.p;
  a.jdiag = p->jdiag.p;
  a.part = p->part.p;
  a.flags = p->flags.p;
  a.bj_inv = p->precond ? p->bj_inv.p : nullptr;
  return a;
}

template <class T>
cudaError_t upload_vec(DBuf<T>& d, const std::vector<T>& h, cudaStream_t s) {
  cudaError_t e = d.ensure(h.size(), s);
  if (e != cudaSuccess || h.empty()) return e;
  return cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s);
}

// CUB device-wide primitives with the problem's shared temp storage.
template <class F>
cudaError_t cub_call(DBuf<uint8_t>& temp, cudaStream_t s, F f) {
  size_t bytes = 0;
  cudaError_t e = f(nullptr, bytes);
  if (e != cudaSuccess) return e;
  if ((e = temp.ensure(bytes, s)) != cudaSuccess) return e;
  return f(temp.p, bytes);
}

// Which frame pairs couple, the contribution lists, the dense work items
// (built on the device, sfb_struct.cu).  One host sync at the end reads the
// sizes the later allocations need.
int rebuild_structure(sfb_problem* p, int bidir) {
  const auto t_start = std::chrono::steady_clock::now();
  const int nb = p->n_blk;
  cudaStream_t s = p->stream;
  const int n_e = (int)p->edges.size();
  const int n_dir = n_e * (bidir ? 2 : 1);
  // sharded PCG mode: the correspondence sets belong to rank 0's partial system
  const int n_sets_s = (p->shard_mode == 1 && p->shard_world > 1 && p->shard_rank != 0) ? 0 : p->n_sets;
  const int n_units = n_sets_s + n_dir;
  p->n_dir = n_dir;
  if ((int64_t)nb * (nb + 1) >= ((int64_t)1 << 32) - 1)
    return fail(p, SFB_E_ARG, "too many frames for 32-bit structure keys");
  // directed dense edges (solver.py:151-155) and the work decomposition:
  // enough (edge, tile range) items to fill the GPU, at most 1024 tiles each;
  // frozen associations in tile-major slots (8 photo-mask words and 256 geo
  // targets per 16x16 tile)
  const int target = 148 * 8;
  int max_nt = 1;
  for (const FrameDev& F : p->frames_h) max_nt = std::max(max_nt, F.tiles_x * F.tiles_y);
  const int64_t items_bound =
      (int64_t)n_dir * std::max((target + std::max(1, n_dir) - 1) / std::max(1, n_dir), (max_nt + 1023) / 1024) + 1;
  const int64_t nd_bound = 3 * (int64_t)n_sets_s + 2 * (int64_t)n_dir;  // D entries
  const int64_t np_bound = (int64_t)n_sets_s + n_dir;                     // B entries >= pairs
  const int64_t nh_bound = nb + 2 * np_bound;                               // row slots
  auto& sc = p->sc;
  CK(p, upload_vec(p->edges_d, p->edges, s));
  CK(p, p->dir_edges.ensure((size_t)std::max(1, n_dir), s));
  CK(p, sc.icount.ensure((size_t)n_dir + 1, s));
  CK(p, sc.per.ensure((size_t)std::max(1, n_dir), s));
  CK(p, sc.pcount.ensure((size_t)n_dir + 1, s));
  CK(p, sc.gcount.ensure((size_t)n_dir + 1, s));
  CK(p, p->edge_item_ptr.ensure((size_t)n_dir + 1, s));
  CK(p, p->photo_off.ensure((size_t)n_dir + 1, s));
  CK(p, p->geo_off.ensure((size_t)n_dir + 1, s));
  CK(p, p->items.ensure((size_t)items_bound, s));
  CK(p, sc.dcount.ensure((size_t)n_units + 1, s));
  CK(p, sc.bcount.ensure((size_t)n_units + 1, s));
  CK(p, sc.doff.ensure((size_t)n_units + 1, s));
  CK(p, sc.boff.ensure((size_t)n_units + 1, s));
  CK(p, sc.dkey.ensure((size_t)std::max<int64_t>(1, nd_bound), s));
  CK(p, sc.dkey2.ensure((size_t)std::max<int64_t>(1, nd_bound), s));
  CK(p, sc.dval.ensure((size_t)std::max<int64_t>(1, nd_bound), s));
  CK(p, p->d_ent.ensure((size_t)std::max<int64_t>(1, nd_bound), s));
  CK(p, p->d_ptr.ensure((size_t)nb + 1, s));
  CK(p, sc.bkey.ensure((size_t)std::max<int64_t>(1, np_bound), s));
  CK(p, sc.bkey2.ensure((size_t)std::max<int64_t>(1, np_bound), s));
  CK(p, sc.bval.ensure((size_t)std::max<int64_t>(1, np_bound), s));
  CK(p, p->b_ent.ensure((size_t)std::max<int64_t>(1, np_bound), s));
  CK(p, p->pair_key.ensure((size_t)std::max<int64_t>(1, np_bound), s));
  CK(p, sc.runs.ensure((size_t)np_bound + 1, s));
  CK(p, p->b_ptr.ensure((size_t)np_bound + 1, s));
  CK(p, sc.hkey.ensure((size_t)nh_bound, s));
  CK(p, sc.hkey2.ensure((size_t)nh_bound, s));
  CK(p, sc.hval.ensure((size_t)nh_bound, s));
  CK(p, sc.hval2.ensure((size_t)nh_bound, s));
  CK(p, p->row_ptr.ensure((size_t)nb + 1, s));
  CK(p, p->row_col.ensure((size_t)nh_bound, s));
  CK(p, p->row_ent.ensure((size_t)std::max<int64_t>(2, 2 * np_bound), s));
  CK(p, sc.scal.ensure(8, s));
  const auto t_alloc = std::chrono::steady_clock::now();

  // work items
  launch_struct_edges(p->edges_d.p, n_e, bidir, p->frames.p, p->shard_rank, p->shard_world, target,
                      p->dir_edges.p, sc.icount.p, sc.pcount.p, sc.gcount.p, sc.per.p, s);
  CKL(p);
  CK(p, cub_call(sc.temp, s, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, sc.icount.p, p->edge_item_ptr.p, n_dir + 1, s);
  }));
  CK(p, cub_call(sc.temp, s, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, sc.pcount.p, p->photo_off.p, n_dir + 1, s);
  }));
  CK(p, cub_call(sc.temp, s, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, sc.gcount.p, p->geo_off.p, n_dir + 1, s);
  }));
  launch_struct_items(p->dir_edges.p, n_dir, p->frames.p, p->edge_item_ptr.p, sc.per.p, p->items.p, s);
  CKL(p);

  // contribution lists: sets in set order, then directed edges; stable
  // sorts keep that order within a variable / pair.  Unused tail keys are
  // 0xFFFFFFFF (after every real key).
  launch_struct_count(p->set_fi.p, p->set_fj.p, p->set_off.p, p->set_end.p, n_sets_s,
                      p->dir_edges.p, n_dir, sc.dcount.p, sc.bcount.p, s);
  CKL(p);
  CK(p, cub_call(sc.temp, s, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, sc.dcount.p, sc.doff.p, n_units + 1, s);
  }));
  CK(p, cub_call(sc.temp, s, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, sc.bcount.p, sc.boff.p, n_units + 1, s);
  }));
  CK(p, cudaMemsetAsync(sc.dkey.p, 0xFF, sizeof(unsigned) * std::max<int64_t>(1, nd_bound), s));
  CK(p, cudaMemsetAsync(sc.bkey.p, 0xFF, sizeof(unsigned) * std::max<int64_t>(1, np_bound), s));
  launch_struct_fill(p->set_fi.p, p->set_fj.p, p->set_off.p, p->set_end.p, n_sets_s,
                     p->dir_edges.p, n_dir, nb, sc.doff.p, sc.boff.p, sc.dkey.p, sc.dval.p, sc.bkey.p,
                     sc.bval.p, s);
  CKL(p);
  const int nd = (int)std::max<int64_t>(1, nd_bound), npb = (int)std::max<int64_t>(1, np_bound);
  CK(p, cub_call(sc.temp, s, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, sc.dkey.p, sc.dkey2.p, sc.dval.p, p->d_ent.p, nd, 0, 32, s);
  }));
  launch_struct_ptr(sc.dkey2.p, nd, nb, p->d_ptr.p, s);
  CKL(p);
  CK(p, cub_call(sc.temp, s, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, sc.bkey.p, sc.bkey2.p, sc.bval.p, p->b_ent.p, npb, 0, 32, s);
  }));
  int* n_runs = reinterpret_cast<int*>(sc.scal.p);
  CK(p, cub_call(sc.temp, s, [&](void* t, size_t& b) {
    return cub::DeviceRunLengthEncode::Encode(t, b, sc.bkey2.p, p->pair_key.p, sc.runs.p, n_runs, npb, s);
  }));
  // drop the sentinel run: pairs = runs whose key is real
  launch_struct_pairs_count(p->pair_key.p, n_runs, n_runs + 1, s);
  CKL(p);
  CK(p, cub_call(sc.temp, s, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, sc.runs.p, p->b_ptr.p, npb + 1, s);
  }));
  // matvec rows
  const int nh = (int)nh_bound;
  CK(p, cudaMemsetAsync(sc.hkey.p, 0xFF, sizeof(unsigned) * nh, s));
  launch_rows_keys(p->pair_key.p, n_runs + 1, nb, nh, sc.hkey.p, sc.hval.p, s);
  CKL(p);
  CK(p, cub_call(sc.temp, s, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, sc.hkey.p, sc.hkey2.p, sc.hval.p, sc.hval2.p, nh, 0, 32, s);
  }));
  launch_rows_out(sc.hkey2.p, sc.hval2.p, n_runs + 1, nb, nh, p->row_ptr.p, p->row_col.p, p->row_ent.p, s);
  CKL(p);
  // sizes for the allocations below
  int64_t hsz[4] = {0, 0, 0, 0};
  CK(p, cudaMemcpyAsync(&hsz[0], p->edge_item_ptr.p + n_dir, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(p, cudaMemcpyAsync(&hsz[1], p->photo_off.p + n_dir, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(p, cudaMemcpyAsync(&hsz[2], p->geo_off.p + n_dir, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(p, cudaMemcpyAsync(&hsz[3], n_runs + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(p, cudaStreamSynchronize(s));
  const auto t_dev = std::chrono::steady_clock::now();
  p->n_items = (int)(hsz[0] & 0xFFFFFFFF);
  const int64_t pw = hsz[1], gw = hsz[2];
  p->n_pairs = (int)(hsz[3] & 0xFFFFFFFF);
  for (int b = 0; b < 2; ++b) {
    CK(p, p->photo_mask[b].ensure((size_t)std::max<int64_t>(pw, 1), s));
    CK(p, p->geo_tgt[b].ensure((size_t)std::max<int64_t>(gw, 1), s));
    CK(p, p->tile_any[b].ensure((size_t)std::max<int64_t>(gw / 256, 1), s));
  }
  CK(p, p->item_out.ensure((size_t)std::max(1, p->n_items) * SFB_ITEM_STRIDE, s));
  CK(p, p->edge_out.ensure((size_t)std::max(1, p->n_dir) * SFB_ITEM_STRIDE, s));
  CK(p, p->edge_rel.ensure((size_t)std::max(1, p->n_dir) * 12, s));
  CK(p, p->item_e2.ensure((size_t)std::max(1, p->n_items) * 2, s));
  CK(p, p->edge_e2.ensure((size_t)std::max(1, p->n_dir) * 2, s));
  CK(p, p->D.ensure((size_t)std::max(1, nb) * 36, s));
  CK(p, p->B.ensure((size_t)std::max(1, p->n_pairs) * 36, s));
  CK(p, p->Brow.ensure((size_t)std::max(1, nb + 2 * p->n_pairs) * 36, s));
  if (trace_on()) {
    const auto t_end = std::chrono::steady_clock::now();
    fprintf(stderr, "sfb rebuild_structure (device): buffers %.2f ms, build+sync %.2f ms, alloc %.2f ms "
            "(%d dir edges, %d pairs, %d items)\n",
            std::chrono::duration<double, std::milli>(t_alloc - t_start).count(),
            std::chrono::duration<double, std::milli>(t_dev - t_alloc).count(),
            std::chrono::duration<double, std::milli>(t_end - t_dev).count(), p->n_dir, p->n_pairs,
            p->n_items);
  }
  p->struct_bidir = bidir;
  p->have_system = false;
  p->dense_active = false;
  return SFB_OK;
}

DenseArgs dense_args(sfb_problem* p) {
  DenseArgs a{};
  a.frames = p->frames.p;
  a.poses = p->poses.p;
  a.items = p->items.p;
  a.dir_edges = p->dir_edges.p;
  a.edge_rel = p->edge_rel.p;
  a.n_dir = p->n_dir;
  a.photo_off = p->photo_off.p;
  a.geo_off = p->geo_off.p;
  a.photo_mask = p->photo_mask[p->cur].p;
  a.geo_tgt = p->geo_tgt[p->cur].p;
  a.tile_any = p->tile_any[p->cur].p;
  a.item_out = p->item_out.p;
  a.rd = p->ctx->rd;
  a.n_items = p->n_items;
  a.stride = 1;
  return a;
}

// Per-frame source-pixel counts on a stride grid (> 1), computed once per stride.
int ensure_stride_counts(sfb_problem* p, int stride, DenseArgs* a) {
  a->stride = stride;
  a->stride_counts = nullptr;
  if (stride <= 1 || !p->has_frames) return SFB_OK;
  if (p->stride_counts_for != stride) {
    CK(p, p->stride_counts.ensure(p->n, p->stream));
    launch_stride_counts(p->frames.p, p->n, stride, p->stride_counts.p, p->stream);
    CKL(p);
    p->stride_counts_for = stride;
  }
  a->stride_counts = p->stride_counts.p;
  return SFB_OK;
}

SparseArgs sparse_args(sfb_problem* p) {
  SparseArgs a{};
  a.poses = p->poses.p;
  a.set_fi = p->set_fi.p;
  a.set_fj = p->set_fj.p;
  a.set_off = p->set_off.p;
  a.set_end = p->set_end.p;
  a.pts_i = p->pts_i.p;
  a.pts_j = p->pts_j.p;
  a.set_out = p->set_out.p;
  a.n_sets = p->n_sets;
  return a;
}

// Enqueue linearize (no sync).  dense_on decided on the host.
int enqueue_energy_frozen(sfb_problem* p, int dense, double* dout3, int dense_only = 0);
int enqueue_dense_energy_edges(sfb_problem* p);
int enqueue_linearize_end(sfb_problem* p);

// Linearisation at the current poses.  With fuse_prev, the previous
// linearisation's frozen dense energy is evaluated in the same pass when one
// exists (*prev_mode = 1: sums in dscal[3..4]; 2: separate pass, dscal[17..18];
// 0: none).
int enqueue_linearize(sfb_problem* p, const sfb_weights* w, double w_dense, const sfb_config* cfg,
                      int fuse_prev = 0, int* prev_mode = nullptr) {
  if (cfg->dense_pixel_stride < 1) return fail(p, SFB_E_ARG, "dense_pixel_stride must be >= 1");
  const int bidir = cfg->dense_bidirectional ? 1 : 0;
  if (p->struct_bidir != bidir) {
    int rc = rebuild_structure(p, bidir);
    if (rc) return rc;
  }
  cudaStream_t s = p->stream;
  SparseArgs sa = sparse_args(p);
  sa.world_i = p->world_i.p;
  sa.world_j = p->world_j.p;
  sa.w_sparse = w->sparse;
  sa.energy_only = 0;
  {
    ProfScope ps(p->prof, 4, s);
    launch_sparse(sa, s);
  }
  CKL(p);
  const bool dense_on = p->has_frames && w_dense > 0.0 && !p->edges.empty();
  const bool prev_avail = fuse_prev && p->dense_active && p->n_items > 0;
  if (prev_mode) *prev_mode = 0;
  const bool lin = dense_on && (w->photo > 0.0 || w->geo > 0.0);
  if (prev_avail && !lin) {
    int rc = enqueue_dense_energy_edges(p);
    if (rc) return rc;
    if (prev_mode) *prev_mode = 2;
  }
  if (dense_on) {
    DenseArgs da = dense_args(p);
    da.do_photo = w->photo > 0.0;
    da.do_geo = w->geo > 0.0;
    da.s_photo = w_dense * w->photo;
    da.s_geo = w_dense * w->geo;
    da.geo_dmax = cfg->geo_distance_max;
    da.geo_nmin = cfg->geo_normal_min;
    {
      int rc = ensure_stride_counts(p, cfg->dense_pixel_stride, &da);
      if (rc) return rc;
    }
    if (lin) {
      const int nxt = 1 - p->cur;
      da.photo_mask = p->photo_mask[nxt].p;
      da.geo_tgt = p->geo_tgt[nxt].p;
      da.tile_any = p->tile_any[nxt].p;
      if (prev_avail) {
        da.photo_mask_prev = p->photo_mask[p->cur].p;
        da.geo_tgt_prev = p->geo_tgt[p->cur].p;
        da.tile_any_prev = p->tile_any[p->cur].p;
        da.prev_photo = p->last_do_photo;
        da.prev_geo = p->last_do_geo;
        if (prev_mode) *prev_mode = 1;
      }
      {
        ProfScope ps(p->prof, 0, s);
        launch_dense_linearize(da, s);
      }
      CKL(p);
      p->cur = nxt;
      ProfScope ps(p->prof, 5, s);
      const bool p2p = p->p2p_on && p->shard_world > 1 && p->p2p_ready[0] && p->p2p_ready[1];
      if (p2p) {  // every rank is done reading the previous sums before anyone pushes new ones
        launch_p2p_sync(p->peer_flags_d.p, p->p2p_flags.p, p->shard_rank, p->shard_world,
                        ++p->p2p_epoch, s);
        CKL(p);
      }
      launch_edge_reduce(p->edge_item_ptr.p, p->item_out.p, p->edge_out.p, p->n_dir, p->dir_edges.p,
                         p->poses.p, s, p2p ? p->peer_edge_d.p : nullptr, p->shard_rank,
                         p->shard_world);
      CKL(p);
      if (p2p) {  // every rank's pushes have landed before the assembly reads them
        launch_p2p_sync(p->peer_flags_d.p, p->p2p_flags.p, p->shard_rank, p->shard_world,
                        ++p->p2p_epoch, s);
        CKL(p);
      }
    } else {
      CK(p, cudaMemsetAsync(p->edge_out.p, 0, sizeof(double) * p->n_dir * SFB_ITEM_STRIDE, s));
    }
    p->last_do_photo = da.do_photo;
    p->last_do_geo = da.do_geo;
  }
  p->pending_dense_on = dense_on;
  p->pending_prev_mode = prev_mode ? *prev_mode : 0;
  return SFB_OK;
}

// Second half of a linearisation, after the per-edge sums are complete on
// every rank (sharded runs all-reduce edge_out / edge_e2 in between).
int enqueue_linearize_end(sfb_problem* p) {
  cudaStream_t s = p->stream;
  const bool dense_on = p->pending_dense_on;
  AssembleArgs aa{};
  aa.n_blk = p->n_blk;
  aa.n_pairs = p->n_pairs;
  aa.set_out = p->set_out.p;
  aa.edge_out = p->edge_out.p;
  aa.d_ptr = p->d_ptr.p;
  aa.d_ent = p->d_ent.p;
  aa.b_ptr = p->b_ptr.p;
  aa.b_ent = p->b_ent.p;
  aa.D = p->D.p;
  aa.B = p->B.p;
  aa.g = p->g.p;
  aa.dense_on = dense_on ? 1 : 0;
  aa.row_ptr = p->row_ptr.p;
  aa.pair_slot = p->row_ent.p;
  aa.Brow = p->Brow.p;
  aa.jdiag = p->jdiag.p;  // the Jacobi diagonal, fused into the assembly
  ProfScope ps(p->prof, 5, s);
  launch_assemble(aa, s);
  CKL(p);
  if (p->n_blk > 0) {
    if (p->precond) {
      CK(p, p->bj_inv.ensure((size_t)p->n_blk * 36, s));
      launch_block_jacobi_inv(p->D.p, p->jdiag.p, p->n_blk, p->bj_inv.p, s);
      CKL(p);
    }
  }
  launch_sum_energies(p->set_out.p, p->n_sets, p->edge_out.p, dense_on ? p->n_dir : 0, nullptr, 0,
                      p->dscal.p, 0, p->esum.p, s);
  CKL(p);
  if (p->pending_prev_mode == 2) {  // separate frozen-energy pass: sums -> dscal[16..18]
    launch_sum_energies(nullptr, 0, nullptr, 0, p->edge_e2.p, p->n_dir, p->dscal.p + 16, 1, p->esum.p, s);
    CKL(p);
  }
  p->dense_active = dense_on;
  p->have_system = true;
  p->spec_pcg = false;  // a speculative PCG belongs to the previous system
  p->have_solution = false;
  return SFB_OK;
}

// Frozen-association dense energy at the current poses -> per-edge sums
// (edge_e2, 2 per directed edge; zero for edges this rank does not own).
int enqueue_dense_energy_edges(sfb_problem* p) {
  cudaStream_t s = p->stream;
  DenseArgs da = dense_args(p);
  da.do_photo = p->last_do_photo;
  da.do_geo = p->last_do_geo;
  {
    ProfScope ps(p->prof, 1, s);
    launch_dense_energy(da, p->item_e2.p, s);
  }
  CKL(p);
  launch_edge_reduce2(p->edge_item_ptr.p, p->item_e2.p, p->edge_e2.p, p->n_dir, s);
  CKL(p);
  return SFB_OK;
}

int enqueue_energy_frozen_begin(sfb_problem* p, int dense) {
  cudaStream_t s = p->stream;
  SparseArgs sa = sparse_args(p);
  sa.energy_only = 1;
  sa.w_sparse = 1.0;
  {
    ProfScope ps(p->prof, 4, s);
    launch_sparse(sa, s);
  }
  CKL(p);
  p->pending_energy_dense = dense && p->dense_active && p->n_items > 0;
  if (p->pending_energy_dense) return enqueue_dense_energy_edges(p);
  return SFB_OK;
}

int enqueue_energy_frozen_end(sfb_problem* p, double* dout3) {
  const bool d = p->pending_energy_dense;
  launch_sum_energies(p->set_out.p, p->n_sets, nullptr, 0, p->edge_e2.p, d ? p->n_dir : 0, dout3,
                      1, p->esum.p, p->stream);
  CKL(p);
  return SFB_OK;
}

int enqueue_energy_frozen(sfb_problem* p, int dense, double* dout3, int /*dense_only*/) {
  int rc = enqueue_energy_frozen_begin(p, dense);
  if (rc) return rc;
  return enqueue_energy_frozen_end(p, dout3);
}

}  // namespace

// ===========================================================================
extern "C" {

const char* sfb_last_error(const void* handle) {
  if (handle) return static_cast<const Handle*>(handle)->err.c_str();
  return g_tls_err.c_str();
}

int sfb_abi_version(void) { return SFB_ABI_VERSION; }

int sfb_ctx_create(int32_t device, sfb_ctx** out) {
  if (!out) return fail(nullptr, SFB_E_ARG, "out is null");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, SFB_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(nullptr, SFB_E_ARG, "bad device index");
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(nullptr, SFB_E_CUDA, cudaGetErrorString(e));
  sfb_ctx* c = new sfb_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, device);
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(nullptr, SFB_E_CUDA, cudaGetErrorString(e));
  }
  *out = c;
  return SFB_OK;
}

int sfb_ctx_destroy(sfb_ctx* c) {
  if (!c) return SFB_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& kv : c->block_refs) cudaFree(kv.first);
  for (auto& kv : c->free_blocks) cudaFree(kv.second);
  for (auto& sl : c->slots)
    if (sl.intensity) dev_cache().release(sl.intensity, sl.intensity_bytes);
  c->verify_items.release();
  c->copy_jobs.release();
  c->cache_raw.release();
  c->cache_out.release();
  c->cache_frames.release();
  c->verify_err.release();
  c->verify_cnt.release();
  c->pack_args.release();
  c->staging.release();
  c->counts.release();
  cudaStreamDestroy(c->stream);
  delete c;
  return SFB_OK;
}

int sfb_ctx_set_rounding(sfb_ctx* c, const sfb_rounding* r) {
  if (!c || !r) return fail(c, SFB_E_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  const int32_t v[6] = {r->matvec_c, r->matvec_f, r->gemm33, r->apply_n, r->apply_1, r->dot3};
  for (int k = 0; k < 6; ++k)
    if (v[k] < 0 || v[k] > 5) return fail(c, SFB_E_ARG, "rounding code out of range");
  c->rd = Rounding{r->matvec_c, r->matvec_f, r->gemm33, r->apply_n, r->apply_1, r->dot3};
  return SFB_OK;
}

int sfb_frames_upload(sfb_ctx* c, int32_t n, const sfb_frame_desc* d, int32_t* slots_out) {
  if (!c || n < 0 || (n > 0 && (!d || !slots_out))) return fail(c, SFB_E_ARG, "bad arguments");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  if (n == 0) return SFB_OK;
  const auto t_start = std::chrono::steady_clock::now();
  CK(c, cudaSetDevice(c->device));
  size_t total = 0, stage = 0;
  for (int k = 0; k < n; ++k) {
    const int64_t hw = (int64_t)d[k].width * d[k].height;
    if (d[k].width < 2 || d[k].height < 2)
      return fail(c, SFB_E_ARG, "frames must be at least 2x2 (bilinear sampling)");
    if (!d[k].valid_depth || !d[k].valid_normal || !d[k].points || !d[k].normals || !d[k].grad)
      return fail(c, SFB_E_ARG, "null frame plane");
    const int64_t nt = (int64_t)((d[k].width + SFB_TILE - 1) / SFB_TILE) *
                       ((d[k].height + SFB_TILE - 1) / SFB_TILE);
    total += align256(hw * 16) * 2 + align256(hw * 8) + align256(hw * 32) + align256(nt * 32) +
             align256(nt * 4);
    stage += align256(hw * 2) + align256(hw * 24) + align256(hw * 8);
  }
  // frame blocks come from a per-context cache (released blocks are kept for
  // reuse, like a caching allocator): no cudaMalloc/cudaFree on the hot path
  void* block = nullptr;
  size_t block_bytes = 0;
  {
    auto it = c->free_blocks.lower_bound(total);
    if (it != c->free_blocks.end() && it->first <= 2 * total + (64u << 20)) {
      block = it->second;
      block_bytes = it->first;
      c->cached_bytes -= it->first;
      c->free_blocks.erase(it);
    } else {
      CK(c, cudaMalloc(&block, total));
      block_bytes = total;
    }
  }
  CK(c, c->staging.ensure(stage));
  CK(c, c->counts.ensure(3 * (size_t)n));
  CK(c, c->pack_args.ensure((size_t)n));
  CK(c, cudaMemsetAsync(c->counts.p, 0, sizeof(int) * 3 * n, c->stream));
  char* dst = static_cast<char*>(block);
  char* stg = reinterpret_cast<char*>(c->staging.p);
  std::vector<FrameDev> devs(n);
  std::vector<PackArgs> pargs(n);
  std::vector<void*> cdst, csrc;
  std::vector<size_t> csz;
  std::vector<CopyJob> jobs;
  cdst.reserve(5 * (size_t)n);
  csrc.reserve(5 * (size_t)n);
  csz.reserve(5 * (size_t)n);
  int max_hw = 0, max_nt = 0;
  for (int k = 0; k < n; ++k) {
    const int w = d[k].width, h = d[k].height;
    const size_t hw = (size_t)w * h;
    FrameDev f{};
    f.P = reinterpret_cast<float4*>(dst); dst += align256(hw * 16);
    f.N = reinterpret_cast<float4*>(dst); dst += align256(hw * 16);
    f.G = reinterpret_cast<float2*>(dst); dst += align256(hw * 8);
    f.T = reinterpret_cast<float4*>(dst); dst += align256(hw * 32);
    f.tiles_x = (w + SFB_TILE - 1) / SFB_TILE;
    f.tiles_y = (h + SFB_TILE - 1) / SFB_TILE;
    const size_t nt = (size_t)f.tiles_x * f.tiles_y;
    f.tiles = reinterpret_cast<double4*>(dst); dst += align256(nt * 32);
    f.tile_count = reinterpret_cast<int*>(dst); dst += align256(nt * 4);
    f.fx = d[k].fx; f.fy = d[k].fy; f.cx = d[k].cx; f.cy = d[k].cy;
    f.w = w; f.h = h;
    uint8_t* svd = reinterpret_cast<uint8_t*>(stg);
    uint8_t* svn = svd + hw;
    stg += align256(hw * 2);
    float* spt = reinterpret_cast<float*>(stg);
    float* snr = spt + 3 * hw;
    stg += align256(hw * 24);
    float* sgr = reinterpret_cast<float*>(stg);
    stg += align256(hw * 8);
    const void* srcs[5] = {d[k].valid_depth, d[k].valid_normal, d[k].points, d[k].normals, d[k].grad};
    void* dsts[5] = {svd, svn, spt, snr, sgr};
    const size_t szs[5] = {hw, hw, hw * 12, hw * 12, hw * 8};
    const void* use[5];
    for (int q = 0; q < 5; ++q) {
      // device-resident planes (sfb_build_cache) are read in place; page-locked
      // host planes are pulled by one wide-load copy kernel (16 B per thread,
      // coalesced over the host link) into staging; pageable ones go by DMA
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, srcs[q]) == cudaSuccess) {
        if (at.type == cudaMemoryTypeDevice && at.device == c->device) {
          use[q] = at.devicePointer;
          continue;
        }
        if (at.type == cudaMemoryTypeHost && at.devicePointer != nullptr) {
          jobs.push_back(CopyJob{static_cast<const uint8_t*>(at.devicePointer),
                                 static_cast<uint8_t*>(dsts[q]), szs[q]});
          use[q] = dsts[q];
          continue;
        }
      }
      cudaGetLastError();
      cdst.push_back(dsts[q]);
      csrc.push_back(const_cast<void*>(srcs[q]));
      csz.push_back(szs[q]);
      use[q] = dsts[q];
    }
    svd = (uint8_t*)use[0];
    svn = (uint8_t*)use[1];
    spt = (float*)use[2];
    snr = (float*)use[3];
    sgr = (float*)use[4];
    pargs[k] = PackArgs{svd, svn, spt, snr, sgr, const_cast<float4*>(f.P), const_cast<float4*>(f.N),
                        const_cast<float2*>(f.G), const_cast<float4*>(f.T), w, h,
                        c->counts.p + 3 * k, f.tiles_x, f.tiles_y, const_cast<double4*>(f.tiles),
                        const_cast<int*>(f.tile_count)};
    max_hw = std::max(max_hw, (int)hw);
    max_nt = std::max(max_nt, (int)nt);
    devs[k] = f;
  }
  const auto t_scan = std::chrono::steady_clock::now();
  // pageable planes by DMA, one cudaMemcpyAsync per plane (the batched copy
  // API is not used)
  for (size_t q = 0; q < cdst.size(); ++q)
    CK(c, cudaMemcpyAsync(cdst[q], csrc[q], csz[q], cudaMemcpyHostToDevice, c->stream));
  if (!jobs.empty()) {
    CK(c, c->copy_jobs.ensure(jobs.size(), c->stream));
    CK(c, cudaMemcpyAsync(c->copy_jobs.p, jobs.data(), sizeof(CopyJob) * jobs.size(),
                          cudaMemcpyHostToDevice, c->stream));
    CK(c, launch_stage_copy(c->copy_jobs.p, (int)jobs.size(), c->stream));
  }
  CK(c, cudaMemcpyAsync(c->pack_args.p, pargs.data(), sizeof(PackArgs) * n, cudaMemcpyHostToDevice,
                        c->stream));
  launch_pack_batch(c->pack_args.p, n, max_hw, max_nt, c->stream);
  CKL(c);
  std::vector<int> cnt(3 * n);
  CK(c, cudaMemcpyAsync(cnt.data(), c->counts.p, sizeof(int) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  if (trace_on()) {
    const auto t_end = std::chrono::steady_clock::now();
    fprintf(stderr, "sfb frames_upload: %d frames, scan %.2f ms (pointer checks), copy+pack %.2f ms\n", n,
            std::chrono::duration<double, std::milli>(t_scan - t_start).count(),
            std::chrono::duration<double, std::milli>(t_end - t_scan).count());
  }
  for (int k = 0; k < n; ++k)
    if (cnt[3 * k + 2] != 0) {
      c->free_blocks.emplace(block_bytes, block);
      c->cached_bytes += block_bytes;
      return fail(c, SFB_E_ARG, "cache planes contain non-finite values (frame " + std::to_string(k) + ")");
    }
  c->block_refs[block] = n;
  c->block_size[block] = block_bytes;
  int search = 0;
  for (int k = 0; k < n; ++k) {
    devs[k].n_valid_depth = cnt[3 * k];
    devs[k].n_valid_geo = cnt[3 * k + 1];
    while (search < (int)c->slots.size() && c->slots[search].alive) ++search;
    if (search == (int)c->slots.size()) c->slots.emplace_back();
    Slot& sl = c->slots[search];
    sl.dev = devs[k];
    sl.block = block;
    sl.alive = true;
    slots_out[k] = search;
  }
  return SFB_OK;
}

int sfb_frames_release(sfb_ctx* c, int32_t n, const int32_t* slots) {
  if (!c || (n > 0 && !slots)) return fail(c, SFB_E_ARG, "bad arguments");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  cudaSetDevice(c->device);
  for (int k = 0; k < n; ++k) {
    const int s = slots[k];
    if (s < 0 || s >= (int)c->slots.size() || !c->slots[s].alive) continue;
    Slot& sl = c->slots[s];
    sl.alive = false;
    if (sl.intensity) {
      cudaStreamSynchronize(c->stream);  // a dense_verify may still read it
      dev_cache().release(sl.intensity, sl.intensity_bytes);
      sl.intensity = nullptr;
      sl.intensity_bytes = 0;
      sl.dev.I = nullptr;
    }
    auto it = c->block_refs.find(sl.block);
    if (it != c->block_refs.end() && --it->second == 0) {
      // keep the block for reuse; problems still referencing it were
      // required to be destroyed first (frames are read-only while in use)
      const size_t bytes = c->block_size[it->first];
      c->free_blocks.emplace(bytes, it->first);
      c->cached_bytes += bytes;
      c->block_size.erase(it->first);
      c->block_refs.erase(it);
      while (c->cached_bytes > c->cache_limit && !c->free_blocks.empty()) {
        auto big = std::prev(c->free_blocks.end());
        cudaDeviceSynchronize();
        cudaFree(big->second);
        c->cached_bytes -= big->first;
        c->free_blocks.erase(big);
      }
    }
    sl.block = nullptr;
  }
  return SFB_OK;
}

int sfb_problem_attach_frames(sfb_problem* p, const int32_t* slots) {
  if (!p || !slots) return fail(p, SFB_E_ARG, "bad arguments");
  if (p->has_frames) return fail(p, SFB_E_ARG, "frames already attached");
  sfb_ctx* c = p->ctx;
  CK(p, cudaSetDevice(c->device));
  std::vector<FrameDev> fr(p->n);
  std::unique_lock<std::recursive_mutex> lk(c->mu);  // slots may grow on another thread
  for (int k = 0; k < p->n; ++k) {
    const int sl = slots[k];
    if (sl < 0 || sl >= (int)c->slots.size() || !c->slots[sl].alive)
      return fail(p, SFB_E_ARG, "frame slot not uploaded");
    fr[k] = c->slots[sl].dev;
  }
  lk.unlock();
  CK(p, upload_vec(p->frames, fr, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));  // fr dies here
  p->frames_h.swap(fr);
  p->slots.assign(slots, slots + p->n);
  p->has_frames = true;
  return SFB_OK;
}

int sfb_problem_create(sfb_ctx* c, int32_t n_frames, const int32_t* slots, int32_t n_sets,
                       const int32_t* set_fi, const int32_t* set_fj, const int64_t* set_off,
                       const double* pts_i, const double* pts_j, sfb_problem** out) {
  if (!c || !out || n_frames < 1 || n_sets < 0) return fail(c, SFB_E_ARG, "bad arguments");
  if (n_sets > 0 && (!set_fi || !set_fj || !set_off)) return fail(c, SFB_E_ARG, "null set arrays");
  CK(c, cudaSetDevice(c->device));
  sfb_problem* p = new sfb_problem();
  p->ctx = c;
  p->n = n_frames;
  p->n_blk = n_frames - 1;
  auto bail = [&](int code, const std::string& m) {
    sfb_problem_destroy(p);
    return fail(c, code, m);
  };
  if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(SFB_E_CUDA, "stream create failed");
  cudaStream_t s = p->stream;
  p->frames_h.assign(n_frames, FrameDev{});
  if (slots) {
    p->has_frames = true;
    p->slots.assign(slots, slots + n_frames);
    std::lock_guard<std::recursive_mutex> lk(c->mu);  // slots may grow on another thread
    for (int k = 0; k < n_frames; ++k) {
      const int sl = slots[k];
      if (sl < 0 || sl >= (int)c->slots.size() || !c->slots[sl].alive)
        return bail(SFB_E_ARG, "frame slot not uploaded");
      p->frames_h[k] = c->slots[sl].dev;
    }
  }
  if (upload_vec(p->frames, p->frames_h, s) != cudaSuccess) return bail(SFB_E_OOM, "frames");
  if (p->poses.ensure(n_frames) || p->best.ensure(n_frames)) return bail(SFB_E_OOM, "poses");
  // identity poses until set
  std::vector<PoseDev> idp(n_frames);
  for (auto& q : idp) {
    std::memset(&q, 0, sizeof(q));
    q.R[0] = q.R[4] = q.R[8] = 1.0;
  }
  if (upload_vec(p->poses, idp, s) || upload_vec(p->best, idp, s)) return bail(SFB_E_CUDA, "poses");
  // sparse term (build_sparse_term, solver.py:89-111)
  p->n_sets = n_sets;
  p->n_corr = n_sets > 0 ? set_off[n_sets] : 0;
  for (int k = 0; k < n_sets; ++k) {
    if (set_fi[k] < 0 || set_fi[k] >= n_frames || set_fj[k] < 0 || set_fj[k] >= n_frames ||
        set_off[k + 1] < set_off[k])
      return bail(SFB_E_ARG, "bad correspondence set");
  }
  p->set_fi_h.assign(set_fi, set_fi + n_sets);
  p->set_fj_h.assign(set_fj, set_fj + n_sets);
  p->set_beg_h.assign(set_off, set_off + n_sets);
  p->set_end_h.assign(n_sets > 0 ? set_off + 1 : set_off, n_sets > 0 ? set_off + 1 + n_sets : set_off);
  if (upload_vec(p->set_fi, p->set_fi_h, s) || upload_vec(p->set_fj, p->set_fj_h, s) ||
      upload_vec(p->set_off, p->set_beg_h, s) || upload_vec(p->set_end, p->set_end_h, s))
    return bail(SFB_E_OOM, "sets");
  const size_t nc = (size_t)std::max<int64_t>(p->n_corr, 1) * 3;
  if (p->pts_i.ensure(nc) || p->pts_j.ensure(nc) || p->world_i.ensure(nc) || p->world_j.ensure(nc) ||
      p->set_out.ensure((size_t)std::max(1, n_sets) * SFB_SET_STRIDE))
    return bail(SFB_E_OOM, "correspondences");
  if (p->n_corr > 0) {
    if (!pts_i || !pts_j) return bail(SFB_E_ARG, "null points");
    if (cudaMemcpyAsync(p->pts_i.p, pts_i, sizeof(double) * 3 * p->n_corr, cudaMemcpyHostToDevice, s) ||
        cudaMemcpyAsync(p->pts_j.p, pts_j, sizeof(double) * 3 * p->n_corr, cudaMemcpyHostToDevice, s))
      return bail(SFB_E_CUDA, "points upload");
  }
  const size_t nv = (size_t)std::max(1, 6 * p->n_blk);
  if (p->g.ensure(nv) || p->x.ensure(nv) || p->r.ensure(nv) || p->z.ensure(nv) || p->pv.ensure(nv) ||
      p->Ap.ensure(nv) || p->inv_diag.ensure(nv) || p->bvec.ensure(nv) || p->jdiag.ensure(nv) ||
      p->pv2.ensure(nv) || p->tmp.ensure(2 * nv) ||
      p->part.ensure(4 * 1024) || p->flags.ensure(64) || p->dscal.ensure(64) ||
      p->esum.ensure(SUM_ENERGY_SCRATCH))
    return bail(SFB_E_OOM, "vectors");
  if (pinned_scalars(&p->hscal) != cudaSuccess) return bail(SFB_E_OOM, "pinned");
  if (cudaMemsetAsync(p->esum.p, 0, sizeof(double) * SUM_ENERGY_SCRATCH, s) != cudaSuccess)
    return bail(SFB_E_CUDA, "energy-sum scratch");
  // host arrays are borrowed for the call only: the async copies above must
  // have landed before returning (they may come from reusable staging)
  if (p->n_corr > 0 && cudaStreamSynchronize(s) != cudaSuccess) return bail(SFB_E_CUDA, "points upload");
  int rc = rebuild_structure(p, 0);
  if (rc) {
    std::string m = p->err;
    sfb_problem_destroy(p);
    return fail(c, rc, m);
  }
  *out = p;
  return SFB_OK;
}

int sfb_problem_destroy(sfb_problem* p) {
  if (!p) return SFB_OK;
  cudaSetDevice(p->ctx->device);
  if (p->stream) cudaStreamSynchronize(p->stream);
  DBuf<int>* ib[] = {&p->set_fi, &p->set_fj, &p->edge_item_ptr, &p->d_ptr, &p->d_ent, &p->b_ptr,
                     &p->b_ent, &p->row_ptr, &p->row_ent, &p->row_col, &p->flags};
  for (auto* b : ib) b->release();
  DBuf<double>* db[] = {&p->pts_i, &p->pts_j, &p->world_i, &p->world_j, &p->set_out,
                        &p->item_out, &p->edge_out, &p->item_e2, &p->D, &p->B, &p->g, &p->x,
                        &p->r, &p->z, &p->pv, &p->Ap, &p->inv_diag, &p->bvec, &p->part, &p->tmp, &p->jdiag,
                        &p->pv2, &p->Brow, &p->bj_inv,
                        &p->dscal, &p->esum};
  for (auto* b : db) b->release();
  p->pair_key.release();
  p->edges_d.release();
  p->edge_rel.release();
  p->xsys.release();
  p->pcgs_state.release();
  for (int w = 0; w < 2; ++w) {
    for (void* q : p->p2p_open[w]) cudaIpcCloseMemHandle(q);
    p->p2p_open[w].clear();
  }
  p->p2p_flags.release();
  p->peer_edge_d.release();
  p->peer_flags_d.release();
  {
    auto& sc = p->sc;
    DBuf<int>* si[] = {&sc.icount, &sc.per, &sc.dcount, &sc.bcount, &sc.doff, &sc.boff, &sc.dval,
                       &sc.bval, &sc.runs, &sc.hval, &sc.hval2};
    for (auto* b : si) b->release();
    sc.pcount.release();
    sc.gcount.release();
    DBuf<unsigned>* su[] = {&sc.dkey, &sc.dkey2, &sc.bkey, &sc.bkey2, &sc.hkey, &sc.hkey2};
    for (auto* b : su) b->release();
    sc.scal.release();
    sc.temp.release();
  }
  p->frames.release();
  p->stride_counts.release();
  p->poses.release();
  p->best.release();
  p->set_off.release();
  p->set_end.release();
  p->dir_edges.release();
  p->items.release();
  p->photo_off.release();
  p->geo_off.release();
  for (int b = 0; b < 2; ++b) {
    p->photo_mask[b].release();
    p->geo_tgt[b].release();
    p->tile_any[b].release();
  }
  {
    p->edge_e2.release();
  }
  p->prof.destroy();
  p->f_all.release();
  p->f_cand.release();
  p->f_sel.release();
  p->f_fl.release();
  p->f_pass.release();
  p->f_temp.release();
  p->f_cnt.release();
  p->f_need.release();
  if (p->hscal) pinned_scalars_release(p->hscal);
  if (p->d2h_done) cudaEventDestroy(p->d2h_done);
  if (p->stream) cudaStreamDestroy(p->stream);
  delete p;
  return SFB_OK;
}

int sfb_problem_stream(sfb_problem* p, void** s) {
  if (!p || !s) return fail(p, SFB_E_ARG, "null argument");
  *s = (void*)p->stream;
  return SFB_OK;
}

int sfb_set_poses(sfb_problem* p, const double* R, const double* t, const uint8_t* fl) {
  if (!p || !R || !t) return fail(p, SFB_E_ARG, "null argument");
  CK(p, cudaSetDevice(p->ctx->device));
  std::vector<PoseDev> h(p->n);
  for (int k = 0; k < p->n; ++k) {
    std::memset(&h[k], 0, sizeof(PoseDev));
    std::memcpy(h[k].R, R + 9 * k, 9 * sizeof(double));
    std::memcpy(h[k].t, t + 3 * k, 3 * sizeof(double));
    h[k].f_layout = fl ? (fl[k] ? 1 : 0) : 0;
  }
  CK(p, cudaMemcpyAsync(p->poses.p, h.data(), sizeof(PoseDev) * p->n, cudaMemcpyHostToDevice, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  return SFB_OK;
}

int sfb_get_poses(sfb_problem* p, double* R, double* t) {
  if (!p || !R || !t) return fail(p, SFB_E_ARG, "null argument");
  CK(p, cudaSetDevice(p->ctx->device));
  std::vector<PoseDev> h(p->n);
  CK(p, cudaMemcpyAsync(h.data(), p->poses.p, sizeof(PoseDev) * p->n, cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  for (int k = 0; k < p->n; ++k) {
    std::memcpy(R + 9 * k, h[k].R, 9 * sizeof(double));
    std::memcpy(t + 3 * k, h[k].t, 3 * sizeof(double));
  }
  return SFB_OK;
}

int sfb_save_best(sfb_problem* p) {
  if (!p) return fail(p, SFB_E_ARG, "null problem");
  CK(p, cudaMemcpyAsync(p->best.p, p->poses.p, sizeof(PoseDev) * p->n, cudaMemcpyDeviceToDevice, p->stream));
  return SFB_OK;
}

int sfb_restore_best(sfb_problem* p) {
  if (!p) return fail(p, SFB_E_ARG, "null problem");
  CK(p, cudaMemcpyAsync(p->poses.p, p->best.p, sizeof(PoseDev) * p->n, cudaMemcpyDeviceToDevice, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  return SFB_OK;
}

// Filter phase 1: angle gate, candidate compaction, overlap test of this
// rank's candidates -> pass flags (f_pass, n_cand bytes; zero for candidates
// owned by other ranks).  Sharded callers sum the flags across ranks before
// sfb_build_dense_edges_end.
int sfb_build_dense_edges_begin(sfb_problem* p, double cos_min) {
  if (!p) return fail(p, SFB_E_ARG, "null argument");
  if (!p->has_frames) return fail(p, SFB_E_STATE, "problem has no frames (caches=None)");
  CK(p, cudaSetDevice(p->ctx->device));
  cudaStream_t s = p->stream;
  const int n = p->n;
  const int64_t P = (int64_t)n * (n - 1) / 2;
  p->edges.clear();
  p->n_cand = 0;
  if (P > 0) {
    if (P > INT32_MAX) return fail(p, SFB_E_ARG, "too many frames for the pair filter");
    DBuf<int2>& all = p->f_all;
    DBuf<int2>& cand = p->f_cand;
    DBuf<uint8_t>& fl = p->f_fl;
    DBuf<uint8_t>& pass = p->f_pass;
    DBuf<uint8_t>& temp = p->f_temp;
    DBuf<int>& cnt = p->f_cnt;
    CK(p, all.ensure(P));
    CK(p, cand.ensure(P));
    CK(p, fl.ensure(P));
    CK(p, cnt.ensure(2));
    dim3 grid((n + 255) / 256, n - 1);
    {
      ProfScope ps(p->prof, 3, s);
      sfb_count_launch();
      k_enumerate_pairs<<<grid, 256, 0, s>>>(n, all.p);
      CKL(p);
      launch_angle_gate(p->poses.p, n, p->ctx->rd, cos_min, fl.p, s);
      CKL(p);
      sfb_count_launch(2);
      CK(p, select_flagged(all.p, fl.p, cand.p, cnt.p, (int)P, temp, s));
    }
    int nc = 0;
    CK(p, cudaMemcpyAsync(&nc, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(p, cudaStreamSynchronize(s));
    p->n_cand = nc;
    if (nc > 0) {
      CK(p, pass.ensure(nc));
      CK(p, p->f_need.ensure((size_t)nc + 1, s));
      ProfScope ps(p->prof, 3, s);
      launch_overlap(p->frames.p, p->poses.p, cand.p, nc, p->ctx->rd, 0, pass.p, nullptr, s,
                     p->shard_rank, p->shard_world, p->f_need.p + 1, p->f_need.p, p->ctx->n_sm);
      CKL(p);
    }
  }
  return SFB_OK;
}

// Filter phase 2: compact the passing candidates (pair order = reference
// loop order) and rebuild the work structure.
int sfb_build_dense_edges_end(sfb_problem* p, int64_t* n_out) {
  if (!p || !n_out) return fail(p, SFB_E_ARG, "null argument");
  CK(p, cudaSetDevice(p->ctx->device));
  cudaStream_t s = p->stream;
  const int nc = p->n_cand;
  p->edges.clear();
  if (nc > 0) {
    CK(p, p->f_sel.ensure(nc));
    {
      ProfScope ps(p->prof, 3, s);
      sfb_count_launch(2);
      CK(p, select_flagged(p->f_cand.p, p->f_pass.p, p->f_sel.p, p->f_cnt.p + 1, nc, p->f_temp, s));
    }
    int ne = 0;
    CK(p, cudaMemcpyAsync(&ne, p->f_cnt.p + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(p, cudaStreamSynchronize(s));
    p->edges.resize(ne);
    if (ne > 0)
      CK(p, cudaMemcpyAsync(p->edges.data(), p->f_sel.p, sizeof(int2) * ne, cudaMemcpyDeviceToHost, s));
    CK(p, cudaStreamSynchronize(s));
  }
  *n_out = (int64_t)p->edges.size();
  return rebuild_structure(p, p->struct_bidir < 0 ? 0 : p->struct_bidir);
}

int sfb_build_dense_edges(sfb_problem* p, double cos_min, int64_t* n_out) {
  if (!p || !n_out) return fail(p, SFB_E_ARG, "null argument");
  if (p->shard_world > 1)
    return fail(p, SFB_E_STATE, "sharded problem: use sfb_build_dense_edges_begin/_end");
  const auto t0 = std::chrono::steady_clock::now();
  int rc = sfb_build_dense_edges_begin(p, cos_min);
  if (rc) return rc;
  rc = sfb_build_dense_edges_end(p, n_out);
  if (trace_on())
    fprintf(stderr, "sfb pair filter + rebuild: %.2f ms (%d frames, %lld edges)\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
            p->n, (long long)*n_out);
  return rc;
}


int sfb_get_dense_edges(sfb_problem* p, int32_t* out) {
  if (!p || (!out && !p->edges.empty())) return fail(p, SFB_E_ARG, "null argument");
  for (size_t k = 0; k < p->edges.size(); ++k) {
    out[2 * k] = p->edges[k].x;
    out[2 * k + 1] = p->edges[k].y;
  }
  return SFB_OK;
}

int sfb_set_dense_edges(sfb_problem* p, int64_t ne, const int32_t* pairs) {
  if (!p || ne < 0 || (ne > 0 && !pairs)) return fail(p, SFB_E_ARG, "bad arguments");
  std::vector<int2> e(ne);
  for (int64_t k = 0; k < ne; ++k) {
    const int a = pairs[2 * k], b = pairs[2 * k + 1];
    if (a < 0 || a >= p->n || b < 0 || b >= p->n) return fail(p, SFB_E_ARG, "edge frame out of range");
    e[k] = make_int2(a, b);
  }
  p->edges = e;
  return rebuild_structure(p, p->struct_bidir < 0 ? 0 : p->struct_bidir);
}

int sfb_frustum_overlap(sfb_problem* p, int64_t np_, const int32_t* pairs, double* out) {
  if (!p || np_ < 0 || (np_ > 0 && (!pairs || !out))) return fail(p, SFB_E_ARG, "bad arguments");
  if (!p->has_frames) return fail(p, SFB_E_STATE, "problem has no frames");
  if (np_ == 0) return SFB_OK;
  CK(p, cudaSetDevice(p->ctx->device));
  cudaStream_t s = p->stream;
  std::vector<int2> h(np_);
  for (int64_t k = 0; k < np_; ++k) {
    h[k] = make_int2(pairs[2 * k], pairs[2 * k + 1]);
    if (h[k].x < 0 || h[k].x >= p->n || h[k].y < 0 || h[k].y >= p->n)
      return fail(p, SFB_E_ARG, "pair frame out of range");
  }
  DBuf<int2> d;
  DBuf<int> cnt;
  CK(p, upload_vec(d, h, s));
  CK(p, cnt.ensure(2 * np_));
  launch_overlap(p->frames.p, p->poses.p, d.p, (int)np_, p->ctx->rd, 1, nullptr, cnt.p, s);
  CKL(p);
  std::vector<int> hc(2 * np_);
  CK(p, cudaMemcpyAsync(hc.data(), cnt.p, sizeof(int) * 2 * np_, cudaMemcpyDeviceToHost, s));
  CK(p, cudaStreamSynchronize(s));
  for (int64_t k = 0; k < np_; ++k) {
    const int total = p->frames_h[h[k].x].n_valid_depth;
    out[k] = total > 0 ? (double)hc[2 * k] / (double)total : 0.0;
  }
  d.release();
  cnt.release();
  return SFB_OK;
}

int sfb_linearize(sfb_problem* p, const sfb_weights* w, double w_dense, const sfb_config* cfg,
                  double e3[3]) {
  if (!p || !w || !cfg || !e3) return fail(p, SFB_E_ARG, "null argument");
  if (p->shard_world > 1) return fail(p, SFB_E_STATE, "sharded problem: use the _begin/_end form");
  CK(p, cudaSetDevice(p->ctx->device));
  int rc = enqueue_linearize(p, w, w_dense, cfg);
  if (rc) return rc;
  rc = enqueue_linearize_end(p);
  if (rc) return rc;
  CK(p, cudaMemcpyAsync(p->hscal, p->dscal.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  for (int k = 0; k < 3; ++k) e3[k] = p->hscal[k];
  return SFB_OK;
}

int sfb_pcg(sfb_problem* p, int32_t max_it, double tol, int32_t restart, int32_t* iters,
            double* rel, int32_t* status) {
  if (!p || !iters || !rel || !status) return fail(p, SFB_E_ARG, "null argument");
  if (!p->have_system) return fail(p, SFB_E_STATE, "pcg before linearize");
  if (restart < 1) return fail(p, SFB_E_ARG, "pcg_restart_interval must be >= 1");
  CK(p, cudaSetDevice(p->ctx->device));
  PcgArgs a = pcg_args(p);
  a.max_it = max_it;
  a.tol = tol;
  a.restart = restart;
  a.out_scalars = p->dscal.p + 8;
  a.skip = nullptr;
  p->spec_pcg = false;
  if (p->n_blk > 0) {
    ProfScope ps(p->prof, 2, p->stream);
    CK(p, launch_pcg(a, p->ctx->n_sm, p->stream));
  } else {
    double z3[3] = {0, 0, 0};
    CK(p, cudaMemcpyAsync(p->dscal.p + 8, z3, sizeof(z3), cudaMemcpyHostToDevice, p->stream));
  }
  CK(p, cudaMemcpyAsync(p->hscal + 8, p->dscal.p + 8, 3 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  *iters = (int32_t)p->hscal[8];
  *rel = p->hscal[9];
  *status = p->hscal[10] != 0.0 ? SFB_E_PCG_NONFINITE : SFB_OK;
  p->have_solution = true;
  return SFB_OK;
}

static int copy_out(sfb_problem* p, double* dst, const double* src, size_t n);

int sfb_get_solution(sfb_problem* p, double* x) {
  if (!p || (!x && p->n_blk > 0)) return fail(p, SFB_E_ARG, "null argument");
  if (!p->have_solution) return fail(p, SFB_E_STATE, "no PCG solution");
  CK(p, cudaSetDevice(p->ctx->device));
  return copy_out(p, x, p->x.p, 6 * (size_t)p->n_blk);
}

int sfb_pcg_dense(sfb_ctx* c, int32_t n, const double* A, const double* rhs, const double* diag,
                  int32_t max_it, double tol, int32_t restart, double* x_out, int32_t* iters,
                  double* rel, int32_t* status) {
  if (!c || n < 0 || (n > 0 && (!A || !rhs || !diag || !x_out)) || !iters || !rel || !status)
    return fail(c, SFB_E_ARG, "bad arguments");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  if (restart < 1) return fail(c, SFB_E_ARG, "restart_interval must be >= 1");
  if (n == 0) {
    *iters = 0;
    *rel = 0.0;
    *status = SFB_OK;
    return SFB_OK;
  }
  CK(c, cudaSetDevice(c->device));
  const int nb = (n + 5) / 6, n6 = 6 * nb;
  std::vector<double> hA((size_t)n6 * n6, 0.0), hg(n6, 0.0), hd(n6, 1.0);
  for (int r = 0; r < n; ++r) {
    std::memcpy(&hA[(size_t)r * n6], A + (size_t)r * n, sizeof(double) * n);
    hg[r] = -rhs[r];
    hd[r] = diag[r];
  }
  DBuf<double> dA, vec;
  CK(c, dA.ensure(hA.size()));
  CK(c, vec.ensure((size_t)n6 * 11 + 4 * 1024 + 8));
  cudaStream_t s = c->stream;
  CK(c, cudaMemcpyAsync(dA.p, hA.data(), sizeof(double) * hA.size(), cudaMemcpyHostToDevice, s));
  double* v = vec.p;
  PcgArgs a{};
  a.n_blk = nb;
  a.g = v;
  a.jdiag = v + n6;
  a.x = v + 2 * n6;
  a.r = v + 3 * n6;
  a.z = v + 4 * n6;
  a.p = v + 5 * n6;
  a.Ap = v + 6 * n6;
  a.inv_diag = v + 7 * n6;
  a.b = v + 8 * n6;
  a.out_scalars = v + 9 * n6;
  a.p2 = v + 10 * n6;
  a.part = v + 11 * n6;
  a.flags = reinterpret_cast<int*>(v + 11 * n6 + 4 * 1024);
  a.max_it = max_it;
  a.tol = tol;
  a.restart = restart;
  CK(c, cudaMemcpyAsync(const_cast<double*>(a.g), hg.data(), sizeof(double) * n6, cudaMemcpyHostToDevice, s));
  CK(c, cudaMemcpyAsync(const_cast<double*>(a.jdiag), hd.data(), sizeof(double) * n6, cudaMemcpyHostToDevice, s));
  CK(c, launch_pcg_dense(a, dA.p, c->n_sm, s));
  double sc[3];
  CK(c, cudaMemcpyAsync(x_out, a.x, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  CK(c, cudaMemcpyAsync(sc, a.out_scalars, sizeof(sc), cudaMemcpyDeviceToHost, s));
  CK(c, cudaStreamSynchronize(s));
  *iters = (int32_t)sc[0];
  *rel = sc[1];
  *status = sc[2] != 0.0 ? SFB_E_PCG_NONFINITE : SFB_OK;
  dA.release();
  vec.release();
  return SFB_OK;
}

int sfb_apply_step(sfb_problem* p, double* step_norm) {
  if (!p || !step_norm) return fail(p, SFB_E_ARG, "null argument");
  if (!p->have_solution) return fail(p, SFB_E_STATE, "apply_step before pcg");
  CK(p, cudaSetDevice(p->ctx->device));
  {
    ProfScope ps(p->prof, 6, p->stream);
    launch_pose_update(p->poses.p, p->n, p->x.p, p->dscal.p + 12, nullptr, p->stream);
  }
  CKL(p);
  CK(p, cudaMemcpyAsync(p->hscal + 12, p->dscal.p + 12, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  *step_norm = p->n_blk > 0 ? p->hscal[12] : 0.0;
  return SFB_OK;
}

int sfb_energy_frozen(sfb_problem* p, int32_t dense, double e3[3]) {
  if (!p || !e3) return fail(p, SFB_E_ARG, "null argument");
  if (p->shard_world > 1) return fail(p, SFB_E_STATE, "sharded problem: use the _begin/_end form");
  CK(p, cudaSetDevice(p->ctx->device));
  int rc = enqueue_energy_frozen(p, dense, p->dscal.p + 16);
  if (rc) return rc;
  CK(p, cudaMemcpyAsync(p->hscal + 16, p->dscal.p + 16, 3 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  for (int k = 0; k < 3; ++k) e3[k] = p->hscal[16 + k];
  return SFB_OK;
}

int sfb_gn_iteration(sfb_problem* p, const sfb_weights* w, double w_dense, const sfb_config* cfg,
                     int32_t max_it, double tol, int32_t restart, sfb_iter_result* out) {
  if (!p || !w || !cfg || !out) return fail(p, SFB_E_ARG, "null argument");
  if (restart < 1) return fail(p, SFB_E_ARG, "pcg_restart_interval must be >= 1");
  if (p->shard_world > 1) return fail(p, SFB_E_STATE, "sharded problem: use the _begin/_end form");
  CK(p, cudaSetDevice(p->ctx->device));
  int rc = enqueue_linearize(p, w, w_dense, cfg);
  if (rc) return rc;
  rc = enqueue_linearize_end(p);
  if (rc) return rc;
  cudaStream_t s = p->stream;
  if (p->n_blk > 0) {
    PcgArgs a = pcg_args(p);
    a.max_it = max_it;
    a.tol = tol;
    a.restart = restart;
    a.out_scalars = p->dscal.p + 8;
    a.skip = nullptr;
    {
      ProfScope ps(p->prof, 2, s);
      CK(p, launch_pcg(a, p->ctx->n_sm, s));
    }
    ProfScope ps(p->prof, 6, s);
    launch_pose_update(p->poses.p, p->n, p->x.p, p->dscal.p + 12, nullptr, s);
    CKL(p);
  }
  rc = enqueue_energy_frozen(p, w_dense > 0.0, p->dscal.p + 16);
  if (rc) return rc;
  CK(p, cudaMemcpyAsync(p->hscal, p->dscal.p, 20 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(p, cudaStreamSynchronize(s));
  const double* h = p->hscal;
  out->e_sparse = h[0];
  out->e_photo = h[1];
  out->e_geo = h[2];
  out->pcg_iterations = p->n_blk > 0 ? (int32_t)h[8] : 0;
  out->pcg_relative = p->n_blk > 0 ? h[9] : 0.0;
  out->pcg_status = (p->n_blk > 0 && h[10] != 0.0) ? SFB_E_PCG_NONFINITE : SFB_OK;
  out->step_norm = p->n_blk > 0 ? h[12] : 0.0;
  out->ea_sparse = h[16];
  out->ea_photo = h[17];
  out->ea_geo = h[18];
  p->have_solution = true;
  return SFB_OK;
}

int sfb_system_dims(sfb_problem* p, int32_t* n_vars, int64_t* n_pairs, int64_t* n_corr) {
  if (!p) return fail(p, SFB_E_ARG, "null problem");
  if (n_vars) *n_vars = 6 * p->n_blk;
  if (n_pairs) *n_pairs = p->n_pairs;
  if (n_corr) *n_corr = p->n_corr;
  return SFB_OK;
}

int sfb_matvec(sfb_problem* p, const double* x, double* y) {
  if (!p || !x || !y) return fail(p, SFB_E_ARG, "null argument");
  if (!p->have_system) return fail(p, SFB_E_STATE, "matvec before linearize");
  const int nv = 6 * p->n_blk;
  if (nv == 0) return SFB_OK;
  CK(p, cudaSetDevice(p->ctx->device));
  CK(p, cudaMemcpyAsync(p->tmp.p, x, sizeof(double) * nv, cudaMemcpyHostToDevice, p->stream));
  PcgArgs a = pcg_args(p);
  launch_matvec(a, p->tmp.p, p->tmp.p + nv, p->stream);
  CKL(p);
  CK(p, cudaMemcpyAsync(y, p->tmp.p + nv, sizeof(double) * nv, cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  return SFB_OK;
}

static int copy_out(sfb_problem* p, double* dst, const double* src, size_t n) {
  if (n == 0) return SFB_OK;
  CK(p, cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  return SFB_OK;
}

int sfb_get_gradient(sfb_problem* p, double* g) {
  if (!p || !g) return fail(p, SFB_E_ARG, "null argument");
  if (!p->have_system) return fail(p, SFB_E_STATE, "no system");
  return copy_out(p, g, p->g.p, 6 * (size_t)p->n_blk);
}

}  // extern "C"


extern "C" {

int sfb_get_diagonal(sfb_problem* p, double* d) {
  if (!p || !d) return fail(p, SFB_E_ARG, "null argument");
  if (!p->have_system) return fail(p, SFB_E_STATE, "no system");
  const int nv = 6 * p->n_blk;
  if (nv == 0) return SFB_OK;
  CK(p, cudaSetDevice(p->ctx->device));
  return copy_out(p, d, p->jdiag.p, nv);
}

int sfb_get_blocks(sfb_problem* p, double* diag_blocks, double* pair_blocks, int32_t* pair_vars) {
  if (!p) return fail(p, SFB_E_ARG, "null problem");
  if (!p->have_system) return fail(p, SFB_E_STATE, "no system");
  CK(p, cudaSetDevice(p->ctx->device));
  if (diag_blocks) {
    int rc = copy_out(p, diag_blocks, p->D.p, 36 * (size_t)p->n_blk);
    if (rc) return rc;
  }
  if (pair_blocks) {
    int rc = copy_out(p, pair_blocks, p->B.p, 36 * (size_t)p->n_pairs);
    if (rc) return rc;
  }
  if (pair_vars && p->n_pairs > 0) {
    std::vector<unsigned> keys(p->n_pairs);
    CK(p, cudaMemcpyAsync(keys.data(), p->pair_key.p, sizeof(unsigned) * p->n_pairs,
                          cudaMemcpyDeviceToHost, p->stream));
    CK(p, cudaStreamSynchronize(p->stream));
    for (int q = 0; q < p->n_pairs; ++q) {
      pair_vars[2 * q] = (int32_t)(keys[q] / (unsigned)p->n_blk);
      pair_vars[2 * q + 1] = (int32_t)(keys[q] % (unsigned)p->n_blk);
    }
  }
  return SFB_OK;
}

int sfb_get_sparse_world(sfb_problem* p, double* wi, double* wj) {
  if (!p || !wi || !wj) return fail(p, SFB_E_ARG, "null argument");
  if (!p->have_system) return fail(p, SFB_E_STATE, "no system");
  int rc = copy_out(p, wi, p->world_i.p, 3 * (size_t)p->n_corr);
  if (rc) return rc;
  return copy_out(p, wj, p->world_j.p, 3 * (size_t)p->n_corr);
}

int sfb_sparse_residuals(sfb_problem* p, double* res) {
  if (!p || (!res && p->n_corr > 0)) return fail(p, SFB_E_ARG, "null argument");
  if (p->n_corr == 0) return SFB_OK;
  CK(p, cudaSetDevice(p->ctx->device));
  DBuf<double> d;
  CK(p, d.ensure(3 * (size_t)p->n_corr));
  launch_sparse_residuals(sparse_args(p), d.p, nullptr, p->stream);
  CKL(p);
  int rc = copy_out(p, res, d.p, 3 * (size_t)p->n_corr);
  d.release();
  return rc;
}

int sfb_sparse_set_max(sfb_problem* p, double* out) {
  if (!p || (!out && p->n_sets > 0)) return fail(p, SFB_E_ARG, "null argument");
  if (p->n_sets == 0) return SFB_OK;
  CK(p, cudaSetDevice(p->ctx->device));
  DBuf<double> d;
  CK(p, d.ensure(p->n_sets));
  launch_sparse_residuals(sparse_args(p), nullptr, d.p, p->stream);
  CKL(p);
  int rc = copy_out(p, out, d.p, p->n_sets);
  d.release();
  return rc;
}

int sfb_associate(sfb_problem* p, int32_t fi, int32_t fj, int32_t kind, const sfb_config* cfg,
                  uint8_t* sel, int32_t* tgt) {
  if (!p || !cfg || !sel || !tgt) return fail(p, SFB_E_ARG, "null argument");
  if (!p->has_frames) return fail(p, SFB_E_STATE, "problem has no frames");
  if (fi < 0 || fi >= p->n || fj < 0 || fj >= p->n || kind < 0 || kind > 1)
    return fail(p, SFB_E_ARG, "bad edge");
  if (cfg->dense_pixel_stride < 1) return fail(p, SFB_E_ARG, "dense_pixel_stride must be >= 1");
  CK(p, cudaSetDevice(p->ctx->device));
  const FrameDev& F = p->frames_h[fi];
  const size_t hw = (size_t)F.w * F.h;
  DBuf<uint8_t> ds;
  DBuf<int> dt;
  CK(p, ds.ensure(hw));
  CK(p, dt.ensure(hw));
  DenseArgs a = dense_args(p);
  a.geo_dmax = cfg->geo_distance_max;
  a.geo_nmin = cfg->geo_normal_min;
  {
    int rc = ensure_stride_counts(p, cfg->dense_pixel_stride, &a);
    if (rc) return rc;
  }
  launch_associate(a, fi, fj, kind, ds.p, dt.p, p->stream);
  CKL(p);
  CK(p, cudaMemcpyAsync(sel, ds.p, hw, cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaMemcpyAsync(tgt, dt.p, hw * sizeof(int), cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  ds.release();
  dt.release();
  return SFB_OK;
}

int sfb_point_eval(sfb_problem* p, int32_t fi, int32_t fj, int32_t kind, int64_t m,
                   const double* pts, const double* aux, const double* tg, double* res, double* jac) {
  if (!p || m < 0 || (m > 0 && (!pts || !aux || !res || (kind == 1 && !tg))))
    return fail(p, SFB_E_ARG, "bad arguments");
  if (fi < 0 || fi >= p->n || fj < 0 || fj >= p->n || kind < 0 || kind > 1)
    return fail(p, SFB_E_ARG, "bad edge");
  if (kind == 0 && !p->has_frames) return fail(p, SFB_E_STATE, "photo terms need frames");
  if (m == 0) return SFB_OK;
  CK(p, cudaSetDevice(p->ctx->device));
  const int na = kind == 0 ? 2 : 3, nr = kind == 0 ? 2 : 1, nj = kind == 0 ? 12 : 6;
  DBuf<double> buf;
  const size_t tot = (size_t)m * (3 + na + 3 + nr + nj);
  CK(p, buf.ensure(tot));
  double* dp = buf.p;
  double* da = dp + 3 * m;
  double* dt = da + na * m;
  double* dr = dt + 3 * m;
  double* dj = dr + nr * m;
  cudaStream_t s = p->stream;
  CK(p, cudaMemcpyAsync(dp, pts, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, s));
  CK(p, cudaMemcpyAsync(da, aux, sizeof(double) * na * m, cudaMemcpyHostToDevice, s));
  if (kind == 1) CK(p, cudaMemcpyAsync(dt, tg, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, s));
  launch_point_eval(p->frames.p, p->poses.p, fi, fj, kind, m, dp, da, dt, dr, jac ? dj : nullptr, s);
  CKL(p);
  CK(p, cudaMemcpyAsync(res, dr, sizeof(double) * nr * m, cudaMemcpyDeviceToHost, s));
  if (jac) CK(p, cudaMemcpyAsync(jac, dj, sizeof(double) * nj * m, cudaMemcpyDeviceToHost, s));
  CK(p, cudaStreamSynchronize(s));
  buf.release();
  return SFB_OK;
}

}  // extern "C"

extern "C" {

int sfb_profile(sfb_problem* p, int32_t enable) {
  if (!p) return fail(p, SFB_E_ARG, "null problem");
  p->prof.on = enable != 0;
  return SFB_OK;
}

int sfb_profile_read(sfb_problem* p, double* ms, int64_t* launches, int32_t reset) {
  if (!p) return fail(p, SFB_E_ARG, "null problem");
  CK(p, cudaSetDevice(p->ctx->device));
  CK(p, cudaStreamSynchronize(p->stream));
  p->prof.drain();
  for (int k = 0; k < SFB_PROF_CLASSES; ++k) {
    if (ms) ms[k] = p->prof.ms[k];
    if (launches) launches[k] = p->prof.n[k];
    if (reset) {
      p->prof.ms[k] = 0.0;
      p->prof.n[k] = 0;
    }
  }
  return SFB_OK;
}

int sfb_launch_count(int64_t* out) {
  if (!out) return fail(nullptr, SFB_E_ARG, "null argument");
  *out = g_launches.load();
  return SFB_OK;
}

}  // extern "C"

extern "C" {

// E_after of the previous GN iteration and the next linearisation, at the
// same (current) poses, in one pass over the frame pairs (solver.py:662-672
// followed by :630-660).  out = {E_sparse, E_photo_frozen, E_geo_frozen,
// E_sparse, E_photo_new, E_geo_new} (raw sums).
// Sharded form: begin enqueues everything up to the per-edge sums and tells
// the caller which exchange buffers must be summed across ranks (bit 0:
// edge_out, bit 1: edge_e2); end assembles and returns the energies.
int sfb_energy_and_linearize_begin(sfb_problem* p, const sfb_weights* w, int32_t prev_dense,
                                   double w_dense_next, const sfb_config* cfg, int32_t* exchange) {
  if (!p || !w || !cfg || !exchange) return fail(p, SFB_E_ARG, "null argument");
  CK(p, cudaSetDevice(p->ctx->device));
  int mode = 0;
  int rc = enqueue_linearize(p, w, w_dense_next, cfg, prev_dense ? 1 : 0, &mode);
  if (rc) return rc;
  *exchange = (p->pending_dense_on && !p->p2p_on ? 1 : 0) | (mode == 2 ? 2 : 0);
  return SFB_OK;
}

int sfb_energy_and_linearize_end(sfb_problem* p, double out6[6]) {
  if (!p || !out6) return fail(p, SFB_E_ARG, "null argument");
  CK(p, cudaSetDevice(p->ctx->device));
  const int mode = p->pending_prev_mode;
  int rc = enqueue_linearize_end(p);
  if (rc) return rc;
  CK(p, cudaMemcpyAsync(p->hscal, p->dscal.p, 20 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  const double* h = p->hscal;
  out6[0] = h[0];
  out6[1] = mode == 1 ? h[3] : (mode == 2 ? h[17] : 0.0);
  out6[2] = mode == 1 ? h[4] : (mode == 2 ? h[18] : 0.0);
  out6[3] = h[0];
  out6[4] = h[1];
  out6[5] = h[2];
  return SFB_OK;
}

// One GN iteration after the linearisation, with a single host round trip:
// pcg_solve (solver.py:463-508) -> _apply_step (:674-677, skipped on the
// device when the PCG diverged) -> the frozen energy of this linearisation at
// the new poses (:662-672), fused with the next linearisation when
// `relinearize` (the GN loop evaluates both at identical poses).  Sharded
// problems exchange the buffers flagged by *exchange between _begin and _end
// (enqueued on the problem's stream; no host sync in between).
// out[0] PCG iterations, [1] relative residual, [2] 1 if non-finite,
// [3] step norm, [4..6] energy after (sparse, photo, geo), [7..9] the next
// linearisation's energies (relinearize only).
int sfb_gn_step_begin(sfb_problem* p, int32_t max_it, double tol, int32_t restart,
                      const sfb_weights* w, int32_t prev_dense, int32_t relinearize,
                      double w_dense_next, const sfb_config* cfg, int32_t* exchange) {
  if (!p || !w || !cfg || !exchange) return fail(p, SFB_E_ARG, "null argument");
  if (!p->have_system) return fail(p, SFB_E_STATE, "gn_step before linearize");
  if (restart < 1) return fail(p, SFB_E_ARG, "pcg_restart_interval must be >= 1");
  CK(p, cudaSetDevice(p->ctx->device));
  cudaStream_t s = p->stream;
  p->spec_max_it = max_it;  // the PCG parameters a speculative PCG will reuse
  p->spec_tol = tol;
  p->spec_restart = restart;
  if (p->n_blk > 0) {
    // the previous _end may already have enqueued this PCG (same system,
    // same parameters) to run while the host decided to continue
    const bool have = p->spec_pcg && p->spec_pcg_args[0] == max_it &&
                      p->spec_pcg_tol == tol && p->spec_pcg_args[1] == restart;
    p->spec_pcg = false;
    if (!have) {
      PcgArgs a = pcg_args(p);
      a.max_it = max_it;
      a.tol = tol;
      a.restart = restart;
      a.out_scalars = p->dscal.p + 8;
      a.skip = nullptr;
      ProfScope ps(p->prof, 2, s);
      CK(p, launch_pcg(a, p->ctx->n_sm, s));
    }
    ProfScope ps(p->prof, 6, s);
    launch_pose_update(p->poses.p, p->n, p->x.p, p->dscal.p + 12, p->dscal.p + 10, s);
    CKL(p);
  } else {
    double z[5] = {0, 0, 0, 0, 0};
    CK(p, cudaMemcpyAsync(p->dscal.p + 8, z, sizeof(z), cudaMemcpyHostToDevice, s));
  }
  p->have_solution = true;
  p->pending_gn_relin = relinearize != 0;
  if (relinearize) {
    int mode = 0;
    int rc = enqueue_linearize(p, w, w_dense_next, cfg, prev_dense ? 1 : 0, &mode);
    if (rc) return rc;
    *exchange = (p->pending_dense_on && !p->p2p_on ? 1 : 0) | (mode == 2 ? 2 : 0);
  } else {
    int rc = enqueue_energy_frozen_begin(p, prev_dense);
    if (rc) return rc;
    *exchange = p->pending_energy_dense ? 2 : 0;
  }
  return SFB_OK;
}

int sfb_gn_step_end(sfb_problem* p, double out[10]) {
  if (!p || !out) return fail(p, SFB_E_ARG, "null argument");
  CK(p, cudaSetDevice(p->ctx->device));
  cudaStream_t s = p->stream;
  const bool relin = p->pending_gn_relin;
  const int mode = p->pending_prev_mode;
  int rc = relin ? enqueue_linearize_end(p) : enqueue_energy_frozen_end(p, p->dscal.p + 16);
  if (rc) return rc;
  CK(p, cudaMemcpyAsync(p->hscal, p->dscal.p, 20 * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (!p->d2h_done) CK(p, cudaEventCreateWithFlags(&p->d2h_done, cudaEventDisableTiming));
  CK(p, cudaEventRecord(p->d2h_done, s));
  if (relin && p->n_blk > 0) {
    // Speculative next PCG on the system just assembled: it runs while the
    // host reads these scalars and decides; a stop (converged / aborted /
    // energy <= 1e-18) simply never consumes it - it only writes the PCG
    // vectors and status words, which nothing else reads.
    PcgArgs a = pcg_args(p);
    a.max_it = p->spec_max_it;
    a.tol = p->spec_tol;
    a.restart = p->spec_restart;
    a.out_scalars = p->dscal.p + 8;
    a.skip = nullptr;
    ProfScope ps(p->prof, 2, s);
    CK(p, launch_pcg(a, p->ctx->n_sm, s));
    p->spec_pcg = true;
    p->spec_pcg_args[0] = a.max_it;
    p->spec_pcg_args[1] = a.restart;
    p->spec_pcg_tol = a.tol;
  }
  CK(p, cudaEventSynchronize(p->d2h_done));
  const double* h = p->hscal;
  out[0] = p->n_blk > 0 ? h[8] : 0.0;
  out[1] = p->n_blk > 0 ? h[9] : 0.0;
  out[2] = (p->n_blk > 0 && h[10] != 0.0) ? 1.0 : 0.0;
  out[3] = p->n_blk > 0 ? h[12] : 0.0;
  if (relin) {
    out[4] = h[0];
    out[5] = mode == 1 ? h[3] : (mode == 2 ? h[17] : 0.0);
    out[6] = mode == 1 ? h[4] : (mode == 2 ? h[18] : 0.0);
    out[7] = h[0];
    out[8] = h[1];
    out[9] = h[2];
  } else {
    out[4] = h[16];
    out[5] = h[17];
    out[6] = h[18];
    out[7] = out[8] = out[9] = 0.0;
  }
  return SFB_OK;
}

int sfb_gn_step(sfb_problem* p, int32_t max_it, double tol, int32_t restart, const sfb_weights* w,
                int32_t prev_dense, int32_t relinearize, double w_dense_next,
                const sfb_config* cfg, double out[10]) {
  if (p && p->shard_world > 1) return fail(p, SFB_E_STATE, "sharded problem: use the _begin/_end forms");
  int32_t ex = 0;
  int rc = sfb_gn_step_begin(p, max_it, tol, restart, w, prev_dense, relinearize, w_dense_next, cfg, &ex);
  if (rc) return rc;
  return sfb_gn_step_end(p, out);
}

int sfb_energy_and_linearize(sfb_problem* p, const sfb_weights* w, int32_t prev_dense,
                             double w_dense_next, const sfb_config* cfg, double out6[6]) {
  if (p && p->shard_world > 1) return fail(p, SFB_E_STATE, "sharded problem: use the _begin/_end form");
  int32_t ex = 0;
  int rc = sfb_energy_and_linearize_begin(p, w, prev_dense, w_dense_next, cfg, &ex);
  if (rc) return rc;
  return sfb_energy_and_linearize_end(p, out6);
}

int sfb_linearize_begin(sfb_problem* p, const sfb_weights* w, double w_dense, const sfb_config* cfg,
                        int32_t* exchange) {
  if (!p || !w || !cfg || !exchange) return fail(p, SFB_E_ARG, "null argument");
  CK(p, cudaSetDevice(p->ctx->device));
  int rc = enqueue_linearize(p, w, w_dense, cfg);
  if (rc) return rc;
  *exchange = (p->pending_dense_on && p->shard_mode == 0 && !p->p2p_on) ? 1 : 0;
  return SFB_OK;
}

// Sharded-PCG mode: assemble this rank's partial system and pack
// [g | jdiag | e_photo e_geo | D (block Jacobi)] into exchange buffer 3.
int sfb_linearize_end_system(sfb_problem* p) {
  if (!p) return fail(p, SFB_E_ARG, "null problem");
  if (p->shard_mode != 1) return fail(p, SFB_E_STATE, "not in sharded-PCG mode");
  CK(p, cudaSetDevice(p->ctx->device));
  const int saved = p->precond;
  p->precond = 0;  // the block inverses need the reduced D (sfb_linearize_finish)
  int rc = enqueue_linearize_end(p);
  p->precond = saved;
  if (rc) return rc;
  const int n6 = 6 * p->n_blk;
  CK(p, p->xsys.ensure((size_t)sys_pack_len(n6, 1), p->stream));
  launch_sys_pack(p->g.p, p->jdiag.p, p->dscal.p, p->D.p, n6, p->precond, p->xsys.p, 0, p->stream);
  CKL(p);
  return SFB_OK;
}

// ... after the all-reduce of buffer 3: unpack, block inverses, energies.
int sfb_linearize_finish(sfb_problem* p, double e3[3]) {
  if (!p || !e3) return fail(p, SFB_E_ARG, "null argument");
  if (p->shard_mode != 1) return fail(p, SFB_E_STATE, "not in sharded-PCG mode");
  CK(p, cudaSetDevice(p->ctx->device));
  const int n6 = 6 * p->n_blk;
  launch_sys_pack(p->g.p, p->jdiag.p, p->dscal.p, p->D.p, n6, p->precond, p->xsys.p, 1, p->stream);
  CKL(p);
  if (p->precond && p->n_blk > 0) {
    CK(p, p->bj_inv.ensure((size_t)p->n_blk * 36, p->stream));
    launch_block_jacobi_inv(p->D.p, p->jdiag.p, p->n_blk, p->bj_inv.p, p->stream);
    CKL(p);
  }
  CK(p, cudaMemcpyAsync(p->hscal, p->dscal.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  for (int k = 0; k < 3; ++k) e3[k] = p->hscal[k];
  return SFB_OK;
}

// PCG over the partial systems (sfb_pcg_sharded.cu): per iteration the
// caller's fn all-reduces (sums) the n_vars partial A.p in place on `stream`.
int sfb_pcg_sharded(sfb_problem* p, int32_t max_it, double tol, int32_t restart,
                    sfb_allreduce_fn fn, void* user, int32_t* iters, double* rel, int32_t* status) {
  if (!p || !fn || !iters || !rel || !status) return fail(p, SFB_E_ARG, "null argument");
  if (!p->have_system) return fail(p, SFB_E_STATE, "pcg before linearize");
  if (restart < 1) return fail(p, SFB_E_ARG, "pcg_restart_interval must be >= 1");
  CK(p, cudaSetDevice(p->ctx->device));
  cudaStream_t s = p->stream;
  PcgArgs a = pcg_args(p);
  a.max_it = max_it;
  a.tol = tol;
  a.restart = restart;
  const int n6 = 6 * p->n_blk;
  CK(p, p->pcgs_state.ensure(8, s));
  double* st = p->pcgs_state.p;
  p->spec_pcg = false;
  if (p->n_blk > 0) {
    ProfScope ps(p->prof, 2, s);
    launch_pcgs_init(a, st, s);
    CKL(p);
    for (int k = 1; k <= max_it; ++k) {
      const int rs = (k % restart) == 0 ? 1 : 0;
      launch_matvec(a, a.p, a.Ap, s);
      CKL(p);
      if (fn(user, a.Ap, n6, (void*)s) != 0) return fail(p, SFB_E_CUDA, "all-reduce callback failed");
      launch_pcgs_step(a, st, k, rs, s);
      CKL(p);
      if (rs) {
        launch_matvec(a, a.x, a.Ap, s);
        CKL(p);
        if (fn(user, a.Ap, n6, (void*)s) != 0) return fail(p, SFB_E_CUDA, "all-reduce callback failed");
        launch_pcgs_restart(a, st, s);
        CKL(p);
      }
      if ((k & 7) == 0 || k == max_it) {  // stop early once every rank is done
        CK(p, cudaMemcpyAsync(p->hscal + 24, st, 8 * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(p, cudaStreamSynchronize(s));
        if (p->hscal[24 + 6] != 0.0) break;
      }
    }
    CK(p, cudaMemcpyAsync(p->hscal + 24, st, 8 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(p, cudaStreamSynchronize(s));
    *iters = (int32_t)p->hscal[24 + 4];
    *rel = p->hscal[24 + 3];
    *status = p->hscal[24 + 5] != 0.0 ? SFB_E_PCG_NONFINITE : SFB_OK;
  } else {
    *iters = 0;
    *rel = 0.0;
    *status = SFB_OK;
  }
  p->have_solution = true;
  return SFB_OK;
}

int sfb_linearize_end(sfb_problem* p, double e3[3]) {
  if (!p || !e3) return fail(p, SFB_E_ARG, "null argument");
  CK(p, cudaSetDevice(p->ctx->device));
  int rc = enqueue_linearize_end(p);
  if (rc) return rc;
  CK(p, cudaMemcpyAsync(p->hscal, p->dscal.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  for (int k = 0; k < 3; ++k) e3[k] = p->hscal[k];
  return SFB_OK;
}

int sfb_energy_frozen_begin(sfb_problem* p, int32_t dense, int32_t* exchange) {
  if (!p || !exchange) return fail(p, SFB_E_ARG, "null argument");
  CK(p, cudaSetDevice(p->ctx->device));
  int rc = enqueue_energy_frozen_begin(p, dense);
  if (rc) return rc;
  *exchange = p->pending_energy_dense ? 2 : 0;
  return SFB_OK;
}

int sfb_energy_frozen_end(sfb_problem* p, double e3[3]) {
  if (!p || !e3) return fail(p, SFB_E_ARG, "null argument");
  CK(p, cudaSetDevice(p->ctx->device));
  int rc = enqueue_energy_frozen_end(p, p->dscal.p + 16);
  if (rc) return rc;
  CK(p, cudaMemcpyAsync(p->hscal + 16, p->dscal.p + 16, 3 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CK(p, cudaStreamSynchronize(p->stream));
  for (int k = 0; k < 3; ++k) e3[k] = p->hscal[16 + k];
  return SFB_OK;
}

int sfb_set_shard(sfb_problem* p, int32_t rank, int32_t world) {
  if (!p || world < 1 || rank < 0 || rank >= world) return fail(p, SFB_E_ARG, "bad shard");
  CK(p, cudaSetDevice(p->ctx->device));
  p->shard_rank = rank;
  p->shard_world = world;
  return rebuild_structure(p, p->struct_bidir < 0 ? 0 : p->struct_bidir);
}

int sfb_problem_drop_sets(sfb_problem* p, int64_t n, const int32_t* set_ids) {
  if (!p || n < 0 || (n > 0 && !set_ids)) return fail(p, SFB_E_ARG, "bad arguments");
  CK(p, cudaSetDevice(p->ctx->device));
  std::vector<char> drop(p->n_sets, 0);
  for (int64_t k = 0; k < n; ++k) {
    if (set_ids[k] < 0 || set_ids[k] >= p->n_sets) return fail(p, SFB_E_ARG, "set id out of range");
    drop[set_ids[k]] = 1;
  }
  // compact the per-set arrays (the survivors keep their order and their
  // resident correspondence ranges): the problem is then exactly one built
  // from the surviving sets
  std::vector<int> fi, fj;
  std::vector<int64_t> beg, end;
  for (int k = 0; k < p->n_sets; ++k) {
    if (drop[k]) continue;
    fi.push_back(p->set_fi_h[k]);
    fj.push_back(p->set_fj_h[k]);
    beg.push_back(p->set_beg_h[k]);
    end.push_back(p->set_end_h[k]);
  }
  CK(p, cudaStreamSynchronize(p->stream));  // no kernel may still read the old arrays
  p->set_fi_h.swap(fi);
  p->set_fj_h.swap(fj);
  p->set_beg_h.swap(beg);
  p->set_end_h.swap(end);
  p->n_sets = (int)p->set_fi_h.size();
  if (p->n_sets > 0) {
    CK(p, upload_vec(p->set_fi, p->set_fi_h, p->stream));
    CK(p, upload_vec(p->set_fj, p->set_fj_h, p->stream));
    CK(p, upload_vec(p->set_off, p->set_beg_h, p->stream));
    CK(p, upload_vec(p->set_end, p->set_end_h, p->stream));
  }
  p->spec_pcg = false;
  p->have_solution = false;
  return rebuild_structure(p, p->struct_bidir < 0 ? 0 : p->struct_bidir);
}

int sfb_set_preconditioner(sfb_problem* p, int32_t kind) {
  if (!p || kind < 0 || kind > 1) return fail(p, SFB_E_ARG, "preconditioner must be 0 or 1");
  CK(p, cudaSetDevice(p->ctx->device));
  if (kind == p->precond) return SFB_OK;
  CK(p, cudaStreamSynchronize(p->stream));  // a speculative PCG used the previous one
  p->precond = kind;
  p->spec_pcg = false;
  p->have_solution = false;
  if (kind && p->have_system && p->n_blk > 0) {
    CK(p, p->bj_inv.ensure((size_t)p->n_blk * 36, p->stream));
    launch_block_jacobi_inv(p->D.p, p->jdiag.p, p->n_blk, p->bj_inv.p, p->stream);
    CKL(p);
  }
  return SFB_OK;
}

// ---- peer-memory exchange (one process per GPU on one node) -----------------
int sfb_ipc_export(sfb_problem* p, int32_t which, void* handle64, int64_t* bytes) {
  if (!p || !handle64 || !bytes || which < 0 || which > 1) return fail(p, SFB_E_ARG, "bad arguments");
  CK(p, cudaSetDevice(p->ctx->device));
  void* ptr = nullptr;
  if (which == 0) {
    ptr = p->edge_out.p;
    *bytes = (int64_t)p->edge_out.n * (int64_t)sizeof(double);
  } else {
    if (!p->p2p_flags.p) {
      CK(p, p->p2p_flags.ensure(64, p->stream));
      CK(p, cudaMemsetAsync(p->p2p_flags.p, 0, 64 * sizeof(unsigned), p->stream));
      CK(p, cudaStreamSynchronize(p->stream));
    }
    ptr = p->p2p_flags.p;
    *bytes = 64 * (int64_t)sizeof(unsigned);
  }
  if (!ptr) return fail(p, SFB_E_STATE, "buffer not allocated");
  cudaIpcMemHandle_t h;
  CK(p, cudaIpcGetMemHandle(&h, ptr));
  std::memcpy(handle64, &h, sizeof(h));
  return SFB_OK;
}

int sfb_ipc_attach(sfb_problem* p, int32_t which, int32_t world, const void* handles) {
  if (!p || !handles || which < 0 || which > 1 || world != p->shard_world || world > 64)
    return fail(p, SFB_E_ARG, "bad arguments");
  CK(p, cudaSetDevice(p->ctx->device));
  CK(p, cudaStreamSynchronize(p->stream));  // no kernel may still use the old mappings
  for (void* q : p->p2p_open[which]) cudaIpcCloseMemHandle(q);
  p->p2p_open[which].clear();
  p->p2p_ready[which] = false;
  std::vector<void*> ptrs(world, nullptr);
  for (int r = 0; r < world; ++r) {
    if (r == p->shard_rank) {
      ptrs[r] = which == 0 ? (void*)p->edge_out.p : (void*)p->p2p_flags.p;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, (const char*)handles + 64 * r, sizeof(h));
    void* q = nullptr;
    CK(p, cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
    p->p2p_open[which].push_back(q);
    ptrs[r] = q;
  }
  if (which == 0) {
    CK(p, p->peer_edge_d.ensure(world, p->stream));
    CK(p, cudaMemcpyAsync(p->peer_edge_d.p, ptrs.data(), sizeof(void*) * world, cudaMemcpyHostToDevice, p->stream));
  } else {
    CK(p, p->peer_flags_d.ensure(world, p->stream));
    CK(p, cudaMemcpyAsync(p->peer_flags_d.p, ptrs.data(), sizeof(void*) * world, cudaMemcpyHostToDevice, p->stream));
  }
  CK(p, cudaStreamSynchronize(p->stream));
  p->p2p_ready[which] = true;
  return SFB_OK;
}

int sfb_set_p2p(sfb_problem* p, int32_t on) {
  if (!p) return fail(p, SFB_E_ARG, "null problem");
  p->p2p_on = on != 0;
  return SFB_OK;
}

int sfb_set_shard_mode(sfb_problem* p, int32_t mode) {
  if (!p || mode < 0 || mode > 1) return fail(p, SFB_E_ARG, "shard mode must be 0 or 1");
  CK(p, cudaSetDevice(p->ctx->device));
  if (mode == p->shard_mode) return SFB_OK;
  p->shard_mode = mode;
  return rebuild_structure(p, p->struct_bidir < 0 ? 0 : p->struct_bidir);
}

int sfb_exchange_buffer(sfb_problem* p, int32_t which, void** dev_ptr, int64_t* bytes) {
  if (!p || !dev_ptr || !bytes) return fail(p, SFB_E_ARG, "null argument");
  switch (which) {
    case 0:
      *dev_ptr = p->edge_out.p;
      *bytes = (int64_t)p->n_dir * SFB_ITEM_STRIDE * (int64_t)sizeof(double);
      return SFB_OK;
    case 1:
      *dev_ptr = p->edge_e2.p;
      *bytes = (int64_t)p->n_dir * 2 * (int64_t)sizeof(double);
      return SFB_OK;
    case 2:
      *dev_ptr = p->f_pass.p;
      *bytes = p->n_cand;
      return SFB_OK;
    case 3:
      *dev_ptr = p->xsys.p;
      *bytes = (int64_t)sys_pack_len(6 * p->n_blk, p->precond) * (int64_t)sizeof(double);
      return SFB_OK;
    default:
      return fail(p, SFB_E_ARG, "unknown exchange buffer");
  }
}

}  // extern "C"
