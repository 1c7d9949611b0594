// Block-system structure on the device (rebuilt after every frame-pair
// filter): which frames couple, the dense work decomposition and the CSR
// contribution lists that k_assemble and the PCG walk.
//
//   directed edges (solver.py:151-155) -> (edge, 16x16 source-tile range)
//   work items and the tile-major frozen-association offsets;
//   D/g contributions per variable: every correspondence set (set order,
//   solver.py:89-111) then every directed edge (edge order) - the order the
//   sums are assembled in, so the system is built deterministically;
//   coupled pairs (a < b) with their B contributions (same order), pair ids
//   in key order a * nb + b;
//   matvec rows: the diagonal block first, then the coupled columns in
//   increasing order, with each pair's slot in row a and (transposed) in
//   row b.
// Stable radix sorts (CUB) group the lists; everything stays on the device
// (the host loop this replaces cost 1.1 ms at 500 frames and 4-5 ms at 2000).
#include "sfb_kernels.cuh"

__global__ void k_struct_edges(const int2* edges, int n_e, int bidir, const FrameDev* frames,
                               int shard_rank, int shard_world, int target, int2* dir,
                               int* icount, int64_t* pcount, int64_t* gcount, int* per_out) {
  const int n_dir = n_e * (bidir ? 2 : 1);
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d > n_dir) return;
  if (d == n_dir) {  // trailing zero: the exclusive scans yield the totals
    icount[d] = 0;
    pcount[d] = 0;
    gcount[d] = 0;
    return;
  }
  int2 e = edges[d < n_e ? d : d - n_e];
  if (d >= n_e) e = make_int2(e.y, e.x);
  dir[d] = e;
  const FrameDev& F = frames[e.x];
  const int nt = F.tiles_x * F.tiles_y;
  int parts = max(1, (target + n_dir - 1) / max(1, n_dir));
  parts = max(parts, (nt + 1023) / 1024);
  parts = min(parts, nt);
  const int per = max(1, (nt + parts - 1) / max(1, parts));
  const bool owned = shard_world <= 1 || d % shard_world == shard_rank;
  icount[d] = owned ? (nt + per - 1) / per : 0;
  pcount[d] = (int64_t)nt * 8;
  gcount[d] = (int64_t)nt * 256;
  per_out[d] = per;
}

__global__ void k_struct_items(const int2* dir, int n_dir, const FrameDev* frames, const int* eptr,
                               const int* per_in, int4* items) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n_dir) return;
  const FrameDev& F = frames[dir[d].x];
  const int nt = F.tiles_x * F.tiles_y;
  const int per = per_in[d];
  int k = eptr[d];
  const int end = eptr[d + 1];
  for (int b = 0; b < nt && k < end; b += per, ++k) items[k] = make_int4(d, b, min(nt, b + per), 0);
}

// Contribution counts of unit u: sets [0, n_sets), then directed edges.
// An empty set (no correspondences, or dropped by sfb_problem_drop_sets)
// contributes nothing and couples nothing.
__device__ __forceinline__ void contrib_vars(const int* set_fi, const int* set_fj,
                                             const int64_t* set_off, const int64_t* set_end,
                                             int n_sets, const int2* dir, int u, int& vi, int& vj,
                                             bool& is_set) {
  is_set = u < n_sets;
  if (is_set) {
    const bool empty = set_end[u] <= set_off[u];
    vi = empty ? -1 : set_fi[u] - 1;
    vj = empty ? -1 : set_fj[u] - 1;
  } else {
    const int2 e = dir[u - n_sets];
    vi = e.x - 1;
    vj = e.y - 1;
  }
}

__global__ void k_struct_count(const int* set_fi, const int* set_fj, const int64_t* set_off,
                               const int64_t* set_end, int n_sets, const int2* dir, int n_dir,
                               int* dcount, int* bcount) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = n_sets + n_dir;
  if (u > n) return;
  if (u == n) {
    dcount[u] = 0;
    bcount[u] = 0;
    return;
  }
  int vi, vj;
  bool is_set;
  contrib_vars(set_fi, set_fj, set_off, set_end, n_sets, dir, u, vi, vj, is_set);
  if (is_set && vi == vj) {
    dcount[u] = vi >= 0 ? 3 : 0;
    bcount[u] = 0;
    return;
  }
  dcount[u] = (vi >= 0) + (vj >= 0);
  bcount[u] = (vi >= 0 && vj >= 0) ? 1 : 0;
}

// D entries (id << 3 | kind): kind 0/1 set side i/j, 2 self-set, 4/5 edge
// source/destination; B entries keyed by the pair a * nb + b (a < b), kind
// 0/1 = which side of the set is the pair's first variable, 4 for edges.
__global__ void k_struct_fill(const int* set_fi, const int* set_fj, const int64_t* set_off,
                              const int64_t* set_end, int n_sets, const int2* dir, int n_dir, int nb,
                              const int* doff, const int* boff, unsigned* dkey, int* dval,
                              unsigned* bkey, int* bval) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n_sets + n_dir) return;
  int vi, vj;
  bool is_set;
  contrib_vars(set_fi, set_fj, set_off, set_end, n_sets, dir, u, vi, vj, is_set);
  int k = doff[u];
  const int id = is_set ? u : u - n_sets;
  if (is_set) {
    if (vi == vj) {
      if (vi >= 0) {
        dkey[k] = vi; dval[k] = id << 3 | 0; ++k;
        dkey[k] = vi; dval[k] = id << 3 | 1; ++k;
        dkey[k] = vi; dval[k] = id << 3 | 2;
      }
      return;
    }
    if (vi >= 0) { dkey[k] = vi; dval[k] = id << 3 | 0; ++k; }
    if (vj >= 0) { dkey[k] = vj; dval[k] = id << 3 | 1; }
  } else {
    if (vi >= 0) { dkey[k] = vi; dval[k] = id << 3 | 4; ++k; }
    if (vj >= 0) { dkey[k] = vj; dval[k] = id << 3 | 5; }
  }
  if (vi >= 0 && vj >= 0) {
    const int a = min(vi, vj), b = max(vi, vj);
    const int kb = boff[u];
    bkey[kb] = (unsigned)a * (unsigned)nb + (unsigned)b;
    bval[kb] = is_set ? (id << 3 | (vi == a ? 0 : 1)) : (id << 3 | 4);
  }
}

// ptr[v] = first index of key v in sorted keys[0, n) (v in [0, rows])
__global__ void k_struct_ptr(const unsigned* keys, int n, int rows, int* ptr) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v > rows) return;
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (keys[mid] < (unsigned)v) lo = mid + 1;
    else hi = mid;
  }
  ptr[v] = lo;
}

// half-edge list of the matvec rows: the diagonal of row v (column rank 0)
// and, per pair q = (a, b), (row a, col b) -> slot 2q and (row b, col a) -> 2q+1
__global__ void k_rows_keys(const unsigned* pair_key, const int* n_pairs_d, int nb,
                            unsigned* hkey, int* hval) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int np = *n_pairs_d;
  if (i < nb) {
    hkey[i] = (unsigned)i * (unsigned)(nb + 1);
    hval[i] = -1;
    return;
  }
  const int h = i - nb;
  if (h >= 2 * np) return;
  const int q = h >> 1;
  const unsigned a = pair_key[q] / (unsigned)nb, b = pair_key[q] % (unsigned)nb;
  if ((h & 1) == 0) hkey[i] = a * (unsigned)(nb + 1) + b + 1;
  else hkey[i] = b * (unsigned)(nb + 1) + a + 1;
  hval[i] = h;
}

__global__ void k_rows_out(const unsigned* hkey, const int* hval, const int* n_pairs_d, int nb,
                           int* row_ptr, int* row_col, int* pair_slot) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = nb + 2 * *n_pairs_d;
  if (i == 0) row_ptr[nb] = n;
  if (i >= n) return;
  const unsigned row = hkey[i] / (unsigned)(nb + 1), c = hkey[i] % (unsigned)(nb + 1);
  row_col[i] = c == 0 ? (int)row : (int)c - 1;
  if (c == 0) row_ptr[row] = i;
  if (hval[i] >= 0) pair_slot[hval[i]] = i;
}

// pairs = runs of the sorted B keys minus the trailing sentinel run
__global__ void k_struct_pairs_count(const unsigned* unique_keys, const int* n_runs, int* n_pairs) {
  const int r = *n_runs;
  *n_pairs = (r > 0 && unique_keys[r - 1] == 0xFFFFFFFFu) ? r - 1 : r;
}

void launch_struct_pairs_count(const unsigned* unique_keys, const int* n_runs, int* n_pairs,
                               cudaStream_t s) {
  sfb_count_launch();
  k_struct_pairs_count<<<1, 1, 0, s>>>(unique_keys, n_runs, n_pairs);
}

void launch_struct_edges(const int2* edges, int n_e, int bidir, const FrameDev* frames,
                         int shard_rank, int shard_world, int target, int2* dir, int* icount,
                         int64_t* pcount, int64_t* gcount, int* per, cudaStream_t s) {
  const int n = n_e * (bidir ? 2 : 1) + 1;
  sfb_count_launch();
  k_struct_edges<<<(n + 255) / 256, 256, 0, s>>>(edges, n_e, bidir, frames, shard_rank, shard_world,
                                                 target, dir, icount, pcount, gcount, per);
}

void launch_struct_items(const int2* dir, int n_dir, const FrameDev* frames, const int* eptr,
                         const int* per, int4* items, cudaStream_t s) {
  if (n_dir <= 0) return;
  sfb_count_launch();
  k_struct_items<<<(n_dir + 255) / 256, 256, 0, s>>>(dir, n_dir, frames, eptr, per, items);
}

void launch_struct_count(const int* set_fi, const int* set_fj, const int64_t* set_off,
                         const int64_t* set_end, int n_sets, const int2* dir, int n_dir,
                         int* dcount, int* bcount, cudaStream_t s) {
  const int n = n_sets + n_dir + 1;
  sfb_count_launch();
  k_struct_count<<<(n + 255) / 256, 256, 0, s>>>(set_fi, set_fj, set_off, set_end, n_sets, dir,
                                                 n_dir, dcount, bcount);
}

void launch_struct_fill(const int* set_fi, const int* set_fj, const int64_t* set_off,
                        const int64_t* set_end, int n_sets, const int2* dir, int n_dir, int nb,
                        const int* doff, const int* boff, unsigned* dkey, int* dval, unsigned* bkey,
                        int* bval, cudaStream_t s) {
  const int n = n_sets + n_dir;
  if (n <= 0) return;
  sfb_count_launch();
  k_struct_fill<<<(n + 255) / 256, 256, 0, s>>>(set_fi, set_fj, set_off, set_end, n_sets, dir, n_dir,
                                                nb, doff, boff, dkey, dval, bkey, bval);
}

void launch_struct_ptr(const unsigned* keys, int n, int rows, int* ptr, cudaStream_t s) {
  sfb_count_launch();
  k_struct_ptr<<<(rows + 1 + 255) / 256, 256, 0, s>>>(keys, n, rows, ptr);
}

void launch_rows_keys(const unsigned* pair_key, const int* n_pairs_d, int nb, int n_max,
                      unsigned* hkey, int* hval, cudaStream_t s) {
  if (n_max <= 0) return;
  sfb_count_launch();
  k_rows_keys<<<(n_max + 255) / 256, 256, 0, s>>>(pair_key, n_pairs_d, nb, hkey, hval);
}

void launch_rows_out(const unsigned* hkey, const int* hval, const int* n_pairs_d, int nb, int n_max,
                     int* row_ptr, int* row_col, int* pair_slot, cudaStream_t s) {
  sfb_count_launch();
  k_rows_out<<<((n_max > 0 ? n_max : 1) + 255) / 256, 256, 0, s>>>(hkey, hval, n_pairs_d, nb, row_ptr,
                                                              row_col, pair_slot);
}
