// sfb_host.cuh — host-side internals shared by the ABI translation units
// (sfb_abi.cu, sfb_rows_abi.cu, sfb_tsdf_abi.cu): error handling, the
// device allocation cache, device buffers, the frame store of a context.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/sfb.h"
#include "sfb_kernels.cuh"

namespace sfbh {

inline thread_local std::string g_tls_err;

// CUDA-event timing of kernel classes on one stream (enabled per problem).
struct Prof {
  bool on = false;
  double ms[SFB_PROF_CLASSES] = {0};
  int64_t n[SFB_PROF_CLASSES] = {0};
  struct Pending {
    int cls;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  void begin(int cls, cudaStream_t s, Pending* slot) {
    slot->cls = cls;
    slot->a = get();
    slot->b = get();
    cudaEventRecord(slot->a, s);
  }
  void end(const Pending& pd, cudaStream_t s) {
    cudaEventRecord(pd.b, s);
    pending.push_back(pd);
  }
  // call after a stream sync
  void drain() {
    for (auto& pd : pending) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, pd.a, pd.b) == cudaSuccess) {
        ms[pd.cls] += t;
        n[pd.cls] += 1;
      }
      pool.push_back(pd.a);
      pool.push_back(pd.b);
    }
    pending.clear();
  }
  void destroy() {
    drain();
    for (auto e : pool) cudaEventDestroy(e);
    pool.clear();
  }
};

// RAII scope: times the kernels enqueued inside it as one class.
struct ProfScope {
  Prof* pr;
  cudaStream_t s;
  Prof::Pending pd{};
  ProfScope(Prof& p, int cls, cudaStream_t st) : pr(p.on ? &p : nullptr), s(st) {
    if (pr) pr->begin(cls, s, &pd);
  }
  ~ProfScope() {
    if (pr) pr->end(pd, s);
  }
};

struct Handle {
  std::string err;
};

inline bool trace_on() {
  static const bool on = getenv("SFB_TRACE") != nullptr;
  return on;
}

// Process-wide cache of idle device allocations (per device, keyed by size).
// Blocks enter it only from DBuf::release(), which callers invoke after the
// owning stream has been synchronised, so a cached block is never in flight.
struct DevCache {
  std::mutex mu;
  std::map<std::pair<int, size_t>, std::vector<void*>> free;
  size_t bytes = 0;
  static constexpr size_t kLimit = (size_t)8 << 30;
  static size_t round(size_t b) {
    if (b <= 4096) return 4096;
    size_t r = 4096;
    while (r < b && r < ((size_t)1 << 26)) r <<= 1;  // powers of two up to 64 MiB
    return r < b ? ((b + ((size_t)2 << 20) - 1) & ~(((size_t)2 << 20) - 1)) : r;
  }
  cudaError_t alloc(void** p, size_t b) {
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t rb = round(b);
    {
      std::lock_guard<std::mutex> g(mu);
      auto it = free.find({dev, rb});
      if (it != free.end() && !it->second.empty()) {
        *p = it->second.back();
        it->second.pop_back();
        bytes -= rb;
        return cudaSuccess;
      }
    }
    return cudaMalloc(p, rb);
  }
  void release(void* p, size_t b) {
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t rb = round(b);
    std::lock_guard<std::mutex> g(mu);
    if (bytes + rb > kLimit) {
      cudaFree(p);
      return;
    }
    free[{dev, rb}].push_back(p);
    bytes += rb;
  }
};
inline DevCache& dev_cache() {
  static DevCache* c = new DevCache();  // leaked on purpose: outlives static teardown
  return *c;
}

// Pinned 64-double scalar mirrors for problem handles, recycled (a fresh
// cudaMallocHost costs milliseconds).
inline std::mutex g_pin_mu;
inline std::vector<double*> g_pin_free;
inline cudaError_t pinned_scalars(double** out) {
  {
    std::lock_guard<std::mutex> g(g_pin_mu);
    if (!g_pin_free.empty()) {
      *out = g_pin_free.back();
      g_pin_free.pop_back();
      return cudaSuccess;
    }
  }
  return cudaMallocHost(reinterpret_cast<void**>(out), 64 * sizeof(double));
}
inline void pinned_scalars_release(double* p) {
  std::lock_guard<std::mutex> g(g_pin_mu);
  g_pin_free.push_back(p);
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  // Grow to at least `want` elements.  The old block may still be read by
  // work in flight: with the owning stream given it is synchronised and the
  // block recycled through the cache (cudaFree costs milliseconds on this
  // driver); without one it is freed.
  cudaError_t ensure(size_t want, cudaStream_t owner = nullptr) {
    if (want <= n && p) return cudaSuccess;
    const auto t0 = std::chrono::steady_clock::now();
    const bool had = p != nullptr;
    if (p) {
      if (owner != nullptr && cudaStreamSynchronize(owner) == cudaSuccess)
        dev_cache().release(p, n * sizeof(T));
      else
        cudaFree(p);
    }
    p = nullptr;
    n = 0;
    const size_t cnt = std::max<size_t>(want, 1);
    cudaError_t e = dev_cache().alloc(reinterpret_cast<void**>(&p), cnt * sizeof(T));
    if (e == cudaSuccess) n = cnt;
    if (trace_on()) {
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (ms > 0.5) fprintf(stderr, "sfb ensure %zu B (%s): %.2f ms\n", cnt * sizeof(T), had ? "grow" : "new", ms);
    }
    return e;
  }
  void release() {  // caller has synchronised the stream that used the buffer
    if (p) dev_cache().release(p, n * sizeof(T));
    p = nullptr;
    n = 0;
  }
};

// Host twin of dot3o (sfb_internal.cuh): NumPy/OpenBLAS 3-term FMA chain
// fma(a_k b_k, fma(a_j b_j, a_i * b_i)) for permutation code o.
inline double host_dot3o(double a0, double a1, double a2, double b0, double b1, double b2, int o) {
  static const int P[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  const double a[3] = {a0, a1, a2}, b[3] = {b0, b1, b2};
  const int i = P[o][0], j = P[o][1], k = P[o][2];
  volatile double p = a[i] * b[i];  // rounded product, kept out of the fma
  return std::fma(a[k], b[k], std::fma(a[j], b[j], (double)p));
}

struct Slot {
  FrameDev dev;
  void* block = nullptr;
  bool alive = false;
  float* intensity = nullptr;  // owned (dev_cache), dense_verify only
  size_t intensity_bytes = 0;
};


inline int fail(Handle* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  g_tls_err = msg;
  return code;
}

#define CK(h, expr)                                                                    \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) {                                                           \
      return fail(h, _e == cudaErrorMemoryAllocation ? SFB_E_OOM : SFB_E_CUDA,         \
                  std::string(#expr) + ": " + cudaGetErrorString(_e));                 \
    }                                                                                  \
  } while (0)

#define CKL(h)                                                                         \
  do {                                                                                 \
    cudaError_t _e = cudaGetLastError();                                               \
    if (_e != cudaSuccess) return fail(h, SFB_E_CUDA, std::string("launch: ") + cudaGetErrorString(_e)); \
  } while (0)

inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

}  // namespace sfbh

using namespace sfbh;

struct sfb_ctx : Handle {
  // Serialises every call that touches the frame-store slots or the shared
  // per-context buffers / stream below (frames upload / release, problem
  // creation from slots, dense_verify, build_cache, the dense PCG): distinct
  // problems may be solved concurrently (reference solver.py:551-552), and
  // they share this context.
  std::recursive_mutex mu;
  int device = 0;
  int n_sm = 148;
  cudaStream_t stream = nullptr;
  Rounding rd{2, 0, 0, 0, 2, 0};
  std::vector<Slot> slots;
  std::map<void*, int> block_refs;
  DBuf<uint8_t> staging;
  DBuf<int> counts;
  DBuf<PackArgs> pack_args;
  DBuf<VerifyItem> verify_items;
  DBuf<CopyJob> copy_jobs;
  DBuf<uint8_t> cache_raw, cache_out;
  DBuf<CacheFrame> cache_frames;
  DBuf<double> verify_err;
  DBuf<long long> verify_cnt;
  std::map<void*, size_t> block_size;
  std::multimap<size_t, void*> free_blocks;  // released frame blocks kept for reuse
  size_t cached_bytes = 0;
  size_t cache_limit = (size_t)16 << 30;
};
