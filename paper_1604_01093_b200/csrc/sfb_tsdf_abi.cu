// sfb_tsdf_abi.cu — the hashed TSDF volume handle (tsdf.py:55-267): block
// dictionary (key -> device pool slot, insertion order) on the host, voxel
// accumulators in a device pool; kernels in sfb_tsdf.cu (see include/sfb.h).
#include "sfb_host.cuh"


struct sfb_tsdf : Handle {
  sfb_ctx* ctx = nullptr;
  double vs = 0.004, trunc = 0.02, extent = 0.032;
  int dw = 0;
  // block dictionary: key -> pool slot, insertion order with tombstones
  std::unordered_map<long long, int> map;
  std::vector<long long> order;
  std::unordered_map<long long, size_t> pos;
  size_t dead = 0;
  std::vector<int> free_slots;
  int cap = 0, used = 0;
  float *weight = nullptr, *wdist = nullptr, *wcolor = nullptr;
  DBuf<long long> keys, tmp;
  DBuf<uint8_t> temp, color;
  DBuf<int> cnt, slots, aux;
  DBuf<unsigned char> hit, flags;
  DBuf<double> tvals;
  DBuf<float> depth, pack;
};

namespace {

long long tsdf_decode(long long key, int k) {
  const long long m = (1LL << 21) - 1, S = 1LL << 20;
  return (k == 0 ? ((key >> 42) & m) : k == 1 ? ((key >> 21) & m) : (key & m)) - S;
}

long long tsdf_encode(const int64_t* c) {
  const long long S = 1LL << 20;
  return (long long)((((unsigned long long)(c[0] + S)) << 42) |
                     (((unsigned long long)(c[1] + S)) << 21) | ((unsigned long long)(c[2] + S)));
}

int tsdf_grow(sfb_tsdf* t, int need) {
  if (need <= t->cap) return SFB_OK;
  int nc = std::max(need, std::max(1024, 2 * t->cap));
  float *w = nullptr, *d = nullptr, *c = nullptr;
  if (cudaMalloc(&w, sizeof(float) * 512 * (size_t)nc) != cudaSuccess ||
      cudaMalloc(&d, sizeof(float) * 512 * (size_t)nc) != cudaSuccess ||
      cudaMalloc(&c, sizeof(float) * 1536 * (size_t)nc) != cudaSuccess) {
    cudaFree(w);
    cudaFree(d);
    cudaFree(c);
    return fail(t, SFB_E_OOM, "TSDF block pool");
  }
  cudaStream_t s = t->ctx->stream;
  CK(t, cudaMemsetAsync(w, 0, sizeof(float) * 512 * (size_t)nc, s));
  CK(t, cudaMemsetAsync(d, 0, sizeof(float) * 512 * (size_t)nc, s));
  CK(t, cudaMemsetAsync(c, 0, sizeof(float) * 1536 * (size_t)nc, s));
  if (t->cap > 0) {
    CK(t, cudaMemcpyAsync(w, t->weight, sizeof(float) * 512 * (size_t)t->cap, cudaMemcpyDeviceToDevice, s));
    CK(t, cudaMemcpyAsync(d, t->wdist, sizeof(float) * 512 * (size_t)t->cap, cudaMemcpyDeviceToDevice, s));
    CK(t, cudaMemcpyAsync(c, t->wcolor, sizeof(float) * 1536 * (size_t)t->cap, cudaMemcpyDeviceToDevice, s));
    CK(t, cudaStreamSynchronize(s));
    cudaFree(t->weight);
    cudaFree(t->wdist);
    cudaFree(t->wcolor);
  }
  t->weight = w;
  t->wdist = d;
  t->wcolor = c;
  t->cap = nc;
  return SFB_OK;
}

int tsdf_new_slot(sfb_tsdf* t, long long key) {
  int sl;
  if (!t->free_slots.empty()) {
    sl = t->free_slots.back();
    t->free_slots.pop_back();
  } else {
    sl = t->used++;
  }
  t->map[key] = sl;
  t->pos[key] = t->order.size();
  t->order.push_back(key);
  return sl;
}

void tsdf_drop(sfb_tsdf* t, long long key, std::vector<int>& freed) {
  auto it = t->map.find(key);
  if (it == t->map.end()) return;
  freed.push_back(it->second);
  t->free_slots.push_back(it->second);
  t->map.erase(it);
  auto p = t->pos.find(key);
  t->order[p->second] = LLONG_MIN;  // tombstone
  t->pos.erase(p);
  if (++t->dead > 1024 && t->dead * 2 > t->order.size()) {  // compact
    std::vector<long long> o;
    o.reserve(t->map.size());
    for (long long k : t->order)
      if (k != LLONG_MIN) {
        t->pos[k] = o.size();
        o.push_back(k);
      }
    t->order.swap(o);
    t->dead = 0;
  }
}

int tsdf_zero_slots(sfb_tsdf* t, const std::vector<int>& sl) {
  if (sl.empty()) return SFB_OK;
  cudaStream_t s = t->ctx->stream;
  CK(t, t->aux.ensure(sl.size(), s));
  CK(t, cudaMemcpyAsync(t->aux.p, sl.data(), sizeof(int) * sl.size(), cudaMemcpyHostToDevice, s));
  CK(t, launch_tsdf_zero(t->aux.p, (int)sl.size(), t->weight, t->wdist, t->wcolor, s));
  CK(t, cudaStreamSynchronize(s));
  return SFB_OK;
}

}  // namespace

extern "C" {

int sfb_tsdf_create(sfb_ctx* c, double voxel_size, double truncation, int32_t depth_weighting,
                    sfb_tsdf** out) {
  if (!c || !out || !(voxel_size > 0.0) || !(truncation > 0.0))
    return fail(c, SFB_E_ARG, "bad arguments");
  sfb_tsdf* t = new sfb_tsdf();
  t->ctx = c;
  t->vs = voxel_size;
  t->trunc = truncation;
  t->extent = voxel_size * 8;  // TsdfVolume.block_extent (tsdf.py:83-85)
  t->dw = depth_weighting ? 1 : 0;
  *out = t;
  return SFB_OK;
}

int sfb_tsdf_destroy(sfb_tsdf* t) {
  if (!t) return SFB_OK;
  cudaSetDevice(t->ctx->device);
  cudaStreamSynchronize(t->ctx->stream);
  cudaFree(t->weight);
  cudaFree(t->wdist);
  cudaFree(t->wcolor);
  DBuf<long long>* kb[] = {&t->keys, &t->tmp};
  for (auto* b : kb) b->release();
  t->temp.release();
  t->color.release();
  t->cnt.release();
  t->slots.release();
  t->aux.release();
  t->hit.release();
  t->flags.release();
  t->tvals.release();
  t->depth.release();
  t->pack.release();
  delete t;
  return SFB_OK;
}

int sfb_tsdf_apply(sfb_tsdf* t, int32_t sign, int32_t width, int32_t height, const uint8_t* color,
                   const float* depth, const double* k4, const double* pose_R, const double* pose_t,
                   int32_t pose_ord, const double* inv_R, const double* inv_t, int32_t inv_ord,
                   const double* tvals, int32_t n_samples, int32_t* status, int64_t* err_coord) {
  if (!t || !color || !depth || !k4 || !pose_R || !pose_t || !inv_R || !inv_t || !tvals || !status ||
      !err_coord || width < 1 || height < 1 || n_samples < 1 || (sign != 1 && sign != -1))
    return fail(t, SFB_E_ARG, "bad arguments");
  if (pose_ord < 0 || pose_ord > 5 || inv_ord < 0 || inv_ord > 5)
    return fail(t, SFB_E_ARG, "rounding code out of range");
  *status = 0;
  CK(t, cudaSetDevice(t->ctx->device));
  cudaStream_t s = t->ctx->stream;
  const size_t hw = (size_t)width * height;
  CK(t, t->depth.ensure(hw, s));
  CK(t, t->color.ensure(hw * 3, s));
  CK(t, t->tvals.ensure(n_samples, s));
  CK(t, cudaMemcpyAsync(t->depth.p, depth, sizeof(float) * hw, cudaMemcpyHostToDevice, s));
  CK(t, cudaMemcpyAsync(t->color.p, color, hw * 3, cudaMemcpyHostToDevice, s));
  CK(t, cudaMemcpyAsync(t->tvals.p, tvals, sizeof(double) * n_samples, cudaMemcpyHostToDevice, s));
  // touched blocks: ray samples -> keys -> sorted unique (np.unique)
  const size_t nk = hw * n_samples;
  if (nk > (size_t)INT32_MAX) return fail(t, SFB_E_ARG, "frame too large");
  CK(t, t->keys.ensure(nk, s));
  CK(t, t->tmp.ensure(nk, s));
  CK(t, t->cnt.ensure(1, s));
  TsdfTouchArgs ta{};
  ta.depth = t->depth.p;
  ta.W = width;
  ta.H = height;
  ta.fx = k4[0]; ta.fy = k4[1]; ta.cx = k4[2]; ta.cy = k4[3];
  for (int q = 0; q < 9; ++q) ta.pose.R[q] = pose_R[q];
  for (int q = 0; q < 3; ++q) ta.pose.t[q] = pose_t[q];
  ta.ord = pose_ord;
  ta.trunc = t->trunc;
  ta.extent = t->extent;
  ta.t = t->tvals.p;
  ta.n_samples = n_samples;
  ta.keys = t->keys.p;
  CK(t, launch_tsdf_touch(ta, s));
  size_t tb = 0;
  CK(t, tsdf_sort_unique(t->keys.p, t->tmp.p, (int)nk, nullptr, &tb, t->cnt.p, s));
  CK(t, t->temp.ensure(std::max<size_t>(tb, 1), s));
  CK(t, tsdf_sort_unique(t->keys.p, t->tmp.p, (int)nk, t->temp.p, &tb, t->cnt.p, s));
  int nu = 0;
  CK(t, cudaMemcpyAsync(&nu, t->cnt.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(t, cudaStreamSynchronize(s));
  std::vector<long long> keys(nu);
  if (nu > 0)
    CK(t, cudaMemcpyAsync(keys.data(), t->keys.p, sizeof(long long) * nu, cudaMemcpyDeviceToHost, s));
  CK(t, cudaStreamSynchronize(s));
  int n = nu;
  if (n > 0 && keys[n - 1] == LLONG_MAX) --n;  // invalid pixels' sentinel
  if (n == 0) {
    if (sign < 0) *status = 1;  // "frame has no integrated content"
    return SFB_OK;
  }
  // EVAL: which touched blocks receive a hit
  TsdfVoxelArgs va{};
  va.keys = t->keys.p;
  va.extent = t->extent;
  va.vs = t->vs;
  va.trunc = t->trunc;
  for (int q = 0; q < 9; ++q) va.inv_pose.R[q] = inv_R[q];
  for (int q = 0; q < 3; ++q) va.inv_pose.t[q] = inv_t[q];
  va.ord = inv_ord;
  va.fx = k4[0]; va.fy = k4[1]; va.cx = k4[2]; va.cy = k4[3];
  va.W = width;
  va.H = height;
  va.depth = t->depth.p;
  va.color = t->color.p;
  va.depth_weighting = t->dw;
  va.sign = (float)sign;
  va.snap_end = n;
  CK(t, t->hit.ensure(n, s));
  CK(t, t->flags.ensure(n, s));
  CK(t, t->slots.ensure(n, s));
  va.flags = t->hit.p;
  va.slots = nullptr;
  CK(t, launch_tsdf_voxels(va, 0, n, s));
  std::vector<unsigned char> hit(n);
  CK(t, cudaMemcpyAsync(hit.data(), t->hit.p, n, cudaMemcpyDeviceToHost, s));
  CK(t, cudaStreamSynchronize(s));
  // the reference's block loop, in touched (sorted key) order (tsdf.py:130-156)
  std::vector<int> slot(n, -1);
  int limit = n;
  if (sign > 0) {
    int need = t->used;
    for (int b = 0; b < n; ++b)
      if (hit[b] && !t->map.count(keys[b])) ++need;
    int rc = tsdf_grow(t, need);
    if (rc) return rc;
    for (int b = 0; b < n; ++b) {
      if (!hit[b]) continue;
      auto it = t->map.find(keys[b]);
      slot[b] = it != t->map.end() ? it->second : tsdf_new_slot(t, keys[b]);
    }
  } else {
    for (int b = 0; b < n; ++b) {
      auto it = t->map.find(keys[b]);
      if (hit[b] && it == t->map.end()) {  // "block ... missing during de-integration"
        limit = b;
        *status = 2;
        for (int k = 0; k < 3; ++k) err_coord[k] = tsdf_decode(keys[b], k);
        break;
      }
      slot[b] = it != t->map.end() ? it->second : -1;
    }
  }
  CK(t, cudaMemcpyAsync(t->slots.p, slot.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
  va.slots = t->slots.p;
  va.hit = t->hit.p;
  va.weight = t->weight;  // (the pool may have grown above)
  va.wdist = t->wdist;
  va.wcolor = t->wcolor;
  int k2 = -1;
  if (sign < 0 && limit > 0) {  // CHECK: the first block whose weight would go negative
    va.flags = t->flags.p;
    CK(t, launch_tsdf_voxels(va, 1, limit, s));
    std::vector<unsigned char> neg(limit);
    CK(t, cudaMemcpyAsync(neg.data(), t->flags.p, limit, cudaMemcpyDeviceToHost, s));
    CK(t, cudaStreamSynchronize(s));
    for (int b = 0; b < limit; ++b)
      if (slot[b] >= 0 && hit[b] && neg[b]) {
        k2 = b;
        break;
      }
    if (k2 >= 0) {
      limit = k2 + 1;     // that block's update lands, then the error (tsdf.py:146-150)
      va.snap_end = k2;   // ... before its snap / clear / drop
      *status = 3;
      for (int k = 0; k < 3; ++k) err_coord[k] = tsdf_decode(keys[k2], k);
    }
  }
  if (limit > 0) {  // COMMIT
    va.flags = t->flags.p;
    CK(t, launch_tsdf_voxels(va, 2, limit, s));
  }
  if (sign < 0 && limit > 0) {  // drop blocks left empty (tsdf.py:156-160)
    std::vector<unsigned char> empty(limit);
    CK(t, cudaMemcpyAsync(empty.data(), t->flags.p, limit, cudaMemcpyDeviceToHost, s));
    CK(t, cudaStreamSynchronize(s));
    std::vector<int> freed;
    for (int b = 0; b < limit; ++b)
      if (slot[b] >= 0 && empty[b] && b != k2) tsdf_drop(t, keys[b], freed);
    int rc = tsdf_zero_slots(t, freed);
    if (rc) return rc;
  }
  CK(t, cudaStreamSynchronize(s));
  return SFB_OK;
}

int sfb_tsdf_count(sfb_tsdf* t, int64_t* n_blocks) {
  if (!t || !n_blocks) return fail(t, SFB_E_ARG, "null argument");
  *n_blocks = (int64_t)t->map.size();
  return SFB_OK;
}

// Blocks in insertion order (the reference's dict order): coords (n, 3) and
// weight (n, 512), wdist (n, 512), wcolor (n, 512, 3); any output may be NULL.
int sfb_tsdf_export(sfb_tsdf* t, int64_t n, int64_t* coords, float* weight, float* wdist,
                    float* wcolor) {
  if (!t || n != (int64_t)t->map.size()) return fail(t, SFB_E_ARG, "n must equal the block count");
  CK(t, cudaSetDevice(t->ctx->device));
  cudaStream_t s = t->ctx->stream;
  std::vector<int> sl;
  sl.reserve(n);
  int64_t k = 0;
  for (long long key : t->order) {
    if (key == LLONG_MIN) continue;
    if (coords)
      for (int q = 0; q < 3; ++q) coords[3 * k + q] = tsdf_decode(key, q);
    sl.push_back(t->map[key]);
    ++k;
  }
  if (n == 0 || (!weight && !wdist && !wcolor)) return SFB_OK;
  CK(t, t->aux.ensure(n, s));
  CK(t, t->pack.ensure((size_t)n * 2560, s));
  CK(t, cudaMemcpyAsync(t->aux.p, sl.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
  float* pw = t->pack.p;
  float* pd = pw + (size_t)n * 512;
  float* pc = pd + (size_t)n * 512;
  CK(t, launch_tsdf_copy(t->aux.p, (int)n, 0, t->weight, t->wdist, t->wcolor, pw, pd, pc, s));
  if (weight) CK(t, cudaMemcpyAsync(weight, pw, sizeof(float) * 512 * n, cudaMemcpyDeviceToHost, s));
  if (wdist) CK(t, cudaMemcpyAsync(wdist, pd, sizeof(float) * 512 * n, cudaMemcpyDeviceToHost, s));
  if (wcolor) CK(t, cudaMemcpyAsync(wcolor, pc, sizeof(float) * 1536 * n, cudaMemcpyDeviceToHost, s));
  CK(t, cudaStreamSynchronize(s));
  return SFB_OK;
}

// Insert (or overwrite) blocks with the given accumulators; new keys append
// to the insertion order (TsdfVolume.allocate / load_volume, tsdf.py:75-81,260-267).
int sfb_tsdf_import(sfb_tsdf* t, int64_t n, const int64_t* coords, const float* weight,
                    const float* wdist, const float* wcolor) {
  if (!t || n < 0 || (n > 0 && (!coords || !weight || !wdist || !wcolor)))
    return fail(t, SFB_E_ARG, "bad arguments");
  if (n == 0) return SFB_OK;
  CK(t, cudaSetDevice(t->ctx->device));
  cudaStream_t s = t->ctx->stream;
  int need = t->used;
  for (int64_t b = 0; b < n; ++b)
    if (!t->map.count(tsdf_encode(coords + 3 * b))) ++need;
  int rc = tsdf_grow(t, need);
  if (rc) return rc;
  std::vector<int> sl(n);
  for (int64_t b = 0; b < n; ++b) {
    const long long key = tsdf_encode(coords + 3 * b);
    auto it = t->map.find(key);
    sl[b] = it != t->map.end() ? it->second : tsdf_new_slot(t, key);
  }
  CK(t, t->aux.ensure(n, s));
  CK(t, t->pack.ensure((size_t)n * 2560, s));
  float* pw = t->pack.p;
  float* pd = pw + (size_t)n * 512;
  float* pc = pd + (size_t)n * 512;
  CK(t, cudaMemcpyAsync(t->aux.p, sl.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
  CK(t, cudaMemcpyAsync(pw, weight, sizeof(float) * 512 * n, cudaMemcpyHostToDevice, s));
  CK(t, cudaMemcpyAsync(pd, wdist, sizeof(float) * 512 * n, cudaMemcpyHostToDevice, s));
  CK(t, cudaMemcpyAsync(pc, wcolor, sizeof(float) * 1536 * n, cudaMemcpyHostToDevice, s));
  CK(t, launch_tsdf_copy(t->aux.p, (int)n, 1, t->weight, t->wdist, t->wcolor, pw, pd, pc, s));
  CK(t, cudaStreamSynchronize(s));
  return SFB_OK;
}

// One block's accumulators (found = 0 when absent): TsdfVolume.block / voxel_state.
int sfb_tsdf_get_block(sfb_tsdf* t, const int64_t* coord, int32_t* found, float* weight,
                       float* wdist, float* wcolor) {
  if (!t || !coord || !found) return fail(t, SFB_E_ARG, "null argument");
  auto it = t->map.find(tsdf_encode(coord));
  *found = it != t->map.end() ? 1 : 0;
  if (!*found) return SFB_OK;
  CK(t, cudaSetDevice(t->ctx->device));
  cudaStream_t s = t->ctx->stream;
  const size_t sl = it->second;
  if (weight) CK(t, cudaMemcpyAsync(weight, t->weight + sl * 512, 2048, cudaMemcpyDeviceToHost, s));
  if (wdist) CK(t, cudaMemcpyAsync(wdist, t->wdist + sl * 512, 2048, cudaMemcpyDeviceToHost, s));
  if (wcolor) CK(t, cudaMemcpyAsync(wcolor, t->wcolor + sl * 1536, 6144, cudaMemcpyDeviceToHost, s));
  CK(t, cudaStreamSynchronize(s));
  return SFB_OK;
}

}  // extern "C"
