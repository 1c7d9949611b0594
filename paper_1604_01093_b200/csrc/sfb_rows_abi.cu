// sfb_rows_abi.cu — extern "C" entry points of the rows beside the solver:
// page-locked staging, dense_verify (filters.py:216-277) and build_cache
// (frames.py:75-151) on the context's frame store (see include/sfb.h).
#include "sfb_host.cuh"

extern "C" {

// Page-locked host staging (reused by the host runtime across calls).
int sfb_host_alloc(int64_t bytes, void** ptr) {
  if (!ptr || bytes < 0) return fail(nullptr, SFB_E_ARG, "bad arguments");
  cudaError_t e = cudaMallocHost(ptr, (size_t)std::max<int64_t>(bytes, 1));
  if (e != cudaSuccess) return fail(nullptr, SFB_E_OOM, cudaGetErrorString(e));
  return SFB_OK;
}
int sfb_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
  return SFB_OK;
}

int sfb_frames_set_intensity(sfb_ctx* c, int32_t n, const int32_t* slots,
                             const float* const* intensity) {
  if (!c || n < 0 || (n > 0 && (!slots || !intensity))) return fail(c, SFB_E_ARG, "bad arguments");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  CK(c, cudaSetDevice(c->device));
  for (int k = 0; k < n; ++k) {
    const int s = slots[k];
    if (s < 0 || s >= (int)c->slots.size() || !c->slots[s].alive)
      return fail(c, SFB_E_ARG, "slot " + std::to_string(s) + " is not resident");
    if (!intensity[k]) return fail(c, SFB_E_ARG, "null intensity plane");
    Slot& sl = c->slots[s];
    const size_t bytes = (size_t)sl.dev.w * sl.dev.h * sizeof(float);
    if (!sl.intensity) {
      void* p = nullptr;
      CK(c, dev_cache().alloc(&p, bytes));
      sl.intensity = static_cast<float*>(p);
      sl.intensity_bytes = bytes;
    }
    CK(c, cudaMemcpyAsync(sl.intensity, intensity[k], bytes, cudaMemcpyHostToDevice, c->stream));
    sl.dev.I = sl.intensity;
  }
  CK(c, cudaStreamSynchronize(c->stream));  // host planes are borrowed for the call only
  return SFB_OK;
}

int sfb_dense_verify(sfb_ctx* c, int32_t n_items, const int32_t* src_slots,
                     const int32_t* dst_slots, const double* R9, const double* t3,
                     const uint8_t* flags, const sfb_verify_config* cfg,
                     double* err_out, int64_t* count_out) {
  if (!c || n_items < 0 || !cfg) return fail(c, SFB_E_ARG, "bad arguments");
  if (n_items == 0) return SFB_OK;
  if (!src_slots || !dst_slots || !R9 || !t3 || !flags || !err_out || !count_out)
    return fail(c, SFB_E_ARG, "null argument");
  for (int32_t o : {cfg->apply_n, cfg->apply_1, cfg->apply_nf, cfg->apply_1f})
    if (o < 0 || o > 5) return fail(c, SFB_E_ARG, "rounding code out of range");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  CK(c, cudaSetDevice(c->device));
  std::vector<VerifyItem> items(n_items);
  int max_hw = 1;
  for (int k = 0; k < n_items; ++k) {
    const int ss = src_slots[k], ds = dst_slots[k];
    for (int s : {ss, ds}) {
      if (s < 0 || s >= (int)c->slots.size() || !c->slots[s].alive)
        return fail(c, SFB_E_ARG, "slot " + std::to_string(s) + " is not resident");
      if (!c->slots[s].intensity)
        return fail(c, SFB_E_ARG, "slot " + std::to_string(s) + " has no intensity plane");
    }
    VerifyItem& it = items[k];
    it.src = c->slots[ss].dev;
    it.dst = c->slots[ds].dev;
    const bool inv = flags[k] & 1, f_ord = flags[k] & 2;
    const double* R = R9 + 9 * (size_t)k;
    const double* t = t3 + 3 * (size_t)k;
    if (inv) {
      // RigidTransform.inverse (geometry.py:135-137): R.T.copy() (C-ordered)
      // and -(R.T) @ t with NumPy's gemv order for R.T's memory layout
      const int mv = f_ord ? c->rd.mv_c : c->rd.mv_f;
      for (int r = 0; r < 3; ++r)
        for (int q = 0; q < 3; ++q) it.R[r * 3 + q] = R[q * 3 + r];
      for (int r = 0; r < 3; ++r)
        it.t[r] = -host_dot3o(it.R[r * 3 + 0], it.R[r * 3 + 1], it.R[r * 3 + 2], t[0], t[1], t[2], mv);
      it.ord_n = cfg->apply_n;
      it.ord_1 = cfg->apply_1;
    } else {
      for (int q = 0; q < 9; ++q) it.R[q] = R[q];
      for (int q = 0; q < 3; ++q) it.t[q] = t[q];
      it.ord_n = f_ord ? cfg->apply_nf : cfg->apply_n;
      it.ord_1 = f_ord ? cfg->apply_1f : cfg->apply_1;
    }
    max_hw = std::max(max_hw, it.src.w * it.src.h);
  }
  if (max_hw > verify_max_pixels())
    return fail(c, SFB_E_ARG, "dense_verify supports frames of at most " +
                                  std::to_string(verify_max_pixels()) + " pixels");
  CK(c, c->verify_items.ensure(n_items));
  CK(c, c->verify_err.ensure(n_items));
  CK(c, c->verify_cnt.ensure(n_items));
  CK(c, cudaMemcpyAsync(c->verify_items.p, items.data(), sizeof(VerifyItem) * n_items,
                        cudaMemcpyHostToDevice, c->stream));
  const VerifyCfg vc{cfg->depth_max, cfg->normal_min, cfg->color_max};
  CK(c, launch_dense_verify(c->verify_items.p, n_items, max_hw, vc, c->verify_err.p,
                            c->verify_cnt.p, c->stream));
  CK(c, cudaMemcpyAsync(err_out, c->verify_err.p, sizeof(double) * n_items, cudaMemcpyDeviceToHost,
                        c->stream));
  std::vector<long long> cnt(n_items);
  CK(c, cudaMemcpyAsync(cnt.data(), c->verify_cnt.p, sizeof(long long) * n_items,
                        cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  for (int k = 0; k < n_items; ++k) count_out[k] = cnt[k];
  return SFB_OK;
}

int sfb_build_cache(sfb_ctx* c, int32_t n, int32_t width, int32_t height, int32_t low_width,
                    int32_t low_height, const uint8_t* const* colors, const float* const* depths,
                    const double* k_low, int32_t luma_order, void* host_out, int32_t* slots_out) {
  if (!c || n < 0 || (n > 0 && (!colors || !depths || !k_low || !host_out || !slots_out)))
    return fail(c, SFB_E_ARG, "bad arguments");
  if (n == 0) return SFB_OK;
  if (low_width < 2 || low_height < 2 || width % low_width || height % low_height)
    return fail(c, SFB_E_ARG, "frame does not divide into low_width x low_height blocks");
  if (luma_order < 0 || luma_order > 5) return fail(c, SFB_E_ARG, "rounding code out of range");
  const int bw = width / low_width, bh = height / low_height;
  if (bw * bh > 64) return fail(c, SFB_E_ARG, "blocks of more than 64 samples are not supported");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  CK(c, cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  const size_t HW = (size_t)width * height, hw = (size_t)low_width * low_height;
  const size_t raw_b = align256(HW * 3) + align256(HW * 4), out_b = 42 * hw;
  CK(c, c->cache_raw.ensure(raw_b * n, s));
  CK(c, c->cache_out.ensure(align256(out_b) * n, s));
  CK(c, c->cache_frames.ensure(n, s));
  std::vector<CacheFrame> fr(n);
  for (int k = 0; k < n; ++k) {
    uint8_t* raw = c->cache_raw.p + raw_b * k;
    const void* src[2] = {colors[k], depths[k]};
    void* dst[2] = {raw, raw + align256(HW * 3)};
    const size_t sz[2] = {HW * 3, HW * 4};
    const void* use[2];
    for (int q = 0; q < 2; ++q) {
      if (!src[q]) return fail(c, SFB_E_ARG, "null frame plane");
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, src[q]) == cudaSuccess &&
          ((at.type == cudaMemoryTypeHost && at.devicePointer != nullptr) ||
           (at.type == cudaMemoryTypeDevice && at.device == c->device))) {
        use[q] = at.devicePointer;  // pinned (zero-copy) or device-resident input
        continue;
      }
      cudaGetLastError();
      CK(c, cudaMemcpyAsync(dst[q], src[q], sz[q], cudaMemcpyHostToDevice, s));
      use[q] = dst[q];
    }
    uint8_t* o = c->cache_out.p + align256(out_b) * k;
    CacheFrame& f = fr[k];
    f.color = static_cast<const uint8_t*>(use[0]);
    f.depth_in = static_cast<const float*>(use[1]);
    f.intensity = reinterpret_cast<float*>(o);
    f.depth = reinterpret_cast<float*>(o + 4 * hw);
    f.points = reinterpret_cast<float*>(o + 8 * hw);
    f.normals = reinterpret_cast<float*>(o + 20 * hw);
    f.grad = reinterpret_cast<float*>(o + 32 * hw);
    f.valid = o + 40 * hw;
    f.valid_n = o + 41 * hw;
  }
  CK(c, cudaMemcpyAsync(c->cache_frames.p, fr.data(), sizeof(CacheFrame) * n, cudaMemcpyHostToDevice, s));
  CacheArgs ca{c->cache_frames.p, width, height, low_width, low_height, bw, bh,
               k_low[0], k_low[1], k_low[2], k_low[3], luma_order};
  CK(c, launch_build_cache(ca, n, s));
  // the planes become resident frame slots (read in place by the pack kernel)
  std::vector<sfb_frame_desc> d(n);
  for (int k = 0; k < n; ++k) {
    d[k].width = low_width;
    d[k].height = low_height;
    d[k].fx = k_low[0];
    d[k].fy = k_low[1];
    d[k].cx = k_low[2];
    d[k].cy = k_low[3];
    d[k].valid_depth = fr[k].valid;
    d[k].valid_normal = fr[k].valid_n;
    d[k].points = fr[k].points;
    d[k].normals = fr[k].normals;
    d[k].grad = fr[k].grad;
  }
  int rc = sfb_frames_upload(c, n, d.data(), slots_out);
  if (rc) return rc;
  // intensity_low for dense_verify, then the host image of every plane
  for (int k = 0; k < n; ++k) {
    Slot& sl = c->slots[slots_out[k]];
    if (!sl.intensity) {
      void* p = nullptr;
      CK(c, dev_cache().alloc(&p, hw * sizeof(float)));
      sl.intensity = static_cast<float*>(p);
      sl.intensity_bytes = hw * sizeof(float);
    }
    CK(c, cudaMemcpyAsync(sl.intensity, fr[k].intensity, hw * sizeof(float), cudaMemcpyDeviceToDevice, s));
    sl.dev.I = sl.intensity;
    CK(c, cudaMemcpyAsync(static_cast<uint8_t*>(host_out) + out_b * k, fr[k].intensity, out_b,
                          cudaMemcpyDeviceToHost, s));
  }
  CK(c, cudaStreamSynchronize(s));
  return SFB_OK;
}

}  // extern "C"
