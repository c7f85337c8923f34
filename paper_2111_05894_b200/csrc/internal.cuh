// Internal plumbing shared by the tiergraph B200 kernels: error model, the
// per-device context (stream + scratch), host|device pointer staging, and the
// launch counter the bench reports as gpu_launches.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "tg_capi.h"

namespace tgb {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void domain_error(const std::string& m) { throw Error(TG_ERR_DOMAIN, m); }
[[noreturn]] inline void format_error(const std::string& m) { throw Error(TG_ERR_FORMAT, m); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(TG_ERR_INTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
}
#define TGB_CUDA(x) ::tgb::cuda_check((x), #x)

// Device allocations that survive the memory pool's cache: the library
// keeps freed stream-ordered temporaries mapped in the device's default pool
// (capi.cu, TIERGRAPH_POOL_KEEP_MB), which plain cudaMalloc and the next large
// cudaMallocAsync cannot use. On an out-of-memory error the pool is trimmed
// to zero (after a device synchronise, so pending frees have landed) and the
// allocation is retried once.
inline void trim_default_pool() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceSynchronize();
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  cudaGetLastError();
}
template <typename T>
inline cudaError_t dev_malloc(T** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    trim_default_pool();
    e = cudaMalloc(p, bytes);
  }
  return e;
}
template <typename T>
inline cudaError_t dev_malloc_async(T** p, size_t bytes, cudaStream_t s) {
  cudaError_t e = cudaMallocAsync(p, bytes, s);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    trim_default_pool();
    e = cudaMallocAsync(p, bytes, s);
  }
  return e;
}

extern std::atomic<uint64_t> g_launches;
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
// Check the launch itself (configuration errors); execution errors surface at
// the next synchronising call.
#define TGB_LAUNCHED()                                                 \
  do {                                                                 \
    ::tgb::count_launch();                                             \
    ::tgb::cuda_check(cudaGetLastError(), "kernel launch");            \
  } while (0)

// --------------------------------------------------------------- context
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) TGB_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

enum Slot : int {
  kScratchA = 0, kScratchB, kScratchC, kScratchD, kScratchE, kScratchF,
  kStageIn0, kStageIn1, kStageIn2, kStageOut0, kStageOut1, kSmall, kNumSlots
};

}  // namespace tgb

struct tg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  void* slot_ptr[tgb::kNumSlots] = {};
  size_t slot_size[tgb::kNumSlots] = {};
  void* pinned_small = nullptr;  // 4 KB mapped host scratch for small results
  void* pipe_buf[2] = {};        // pinned staging of copy_h2d / copy_d2h (allocated on first use)
  cudaEvent_t pipe_ev[2] = {};
  // Fork-join side stream (concurrent kernels inside one stream-ordered call).
  cudaStream_t aux = nullptr, aux2 = nullptr, aux3 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr, ev_join3 = nullptr;

  // Work enqueued on `aux` between fork() and join() runs concurrently with
  // `stream` and is ordered after everything before fork() and before
  // everything after join() (event edges; also valid under graph capture).
  void fork() {
    if (!aux) {
      // highest priority: the side stream carries the critical-path work
      // (e.g. K3's longest rows), so its CTAs are scheduled first
      int lo = 0, hi = 0;
      tgb::cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
      tgb::cuda_check(cudaStreamCreateWithPriority(&aux, cudaStreamNonBlocking, hi), "aux stream");
      tgb::cuda_check(cudaStreamCreateWithPriority(&aux2, cudaStreamNonBlocking, hi), "aux stream");
      tgb::cuda_check(cudaStreamCreateWithPriority(&aux3, cudaStreamNonBlocking, lo), "aux stream");
      tgb::cuda_check(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "event");
      tgb::cuda_check(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming), "event");
      tgb::cuda_check(cudaEventCreateWithFlags(&ev_join2, cudaEventDisableTiming), "event");
      tgb::cuda_check(cudaEventCreateWithFlags(&ev_join3, cudaEventDisableTiming), "event");
    }
    tgb::cuda_check(cudaEventRecord(ev_fork, stream), "fork record");
    tgb::cuda_check(cudaStreamWaitEvent(aux, ev_fork, 0), "fork wait");
    tgb::cuda_check(cudaStreamWaitEvent(aux2, ev_fork, 0), "fork wait");
    tgb::cuda_check(cudaStreamWaitEvent(aux3, ev_fork, 0), "fork wait");
  }
  void join() {
    tgb::cuda_check(cudaEventRecord(ev_join, aux), "join record");
    tgb::cuda_check(cudaStreamWaitEvent(stream, ev_join, 0), "join wait");
    tgb::cuda_check(cudaEventRecord(ev_join2, aux2), "join record");
    tgb::cuda_check(cudaStreamWaitEvent(stream, ev_join2, 0), "join wait");
    tgb::cuda_check(cudaEventRecord(ev_join3, aux3), "join record");
    tgb::cuda_check(cudaStreamWaitEvent(stream, ev_join3, 0), "join wait");
  }

  // Grow-only scratch buffer bound to a slot. Stream-ordered reuse is safe
  // because every user of the context enqueues on `stream`.
  void* scratch(int slot, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (slot_size[slot] < bytes) {
      if (slot_ptr[slot]) {
        tgb::cuda_check(cudaStreamSynchronize(stream), "scratch sync");
        tgb::cuda_check(cudaFree(slot_ptr[slot]), "scratch free");
        slot_ptr[slot] = nullptr;
        slot_size[slot] = 0;
      }
      size_t sz = bytes + bytes / 8;
      tgb::cuda_check(tgb::dev_malloc(&slot_ptr[slot], sz), "scratch alloc");
      slot_size[slot] = sz;
    }
    return slot_ptr[slot];
  }
  template <typename T>
  T* scratch_t(int slot, size_t count) {
    return static_cast<T*>(scratch(slot, count * sizeof(T)));
  }
  void sync() { tgb::cuda_check(cudaStreamSynchronize(stream), "stream sync"); }
};

namespace tgb {

inline bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Device pointer to mapped pinned host memory, or nullptr if `p` is not
// registered/pinned.
inline void* mapped_device_ptr(const void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type == cudaMemoryTypeHost) return a.devicePointer;
  return nullptr;
}

// Large pageable host <-> device copies, pipelined through two pinned staging
// buffers of the context (DMA of one chunk while the host cores move the
// other): several times the rate of a cudaMemcpy from pageable memory, which
// the driver stages through one thread. Synchronous on return. Small copies
// (< kPipeMin) use cudaMemcpyAsync on the stream as before.
void parallel_memcpy(void* dst, const void* src, size_t bytes);  // host_memcpy.cpp (OpenMP)
constexpr size_t kPipeMin = 32ull << 20;
void copy_h2d(tg_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes, bool sync_end = true);
// u64 host values -> u32 device array through the same pinned pipeline,
// narrowed by the host cores; returns the first index whose value is >= limit
// (~0 when none is). Asynchronous like copy_h2d(sync_end = false).
uint64_t copy_h2d_narrow(tg_ctx* ctx, uint32_t* dst_dev, const uint64_t* src_host, size_t count,
                         uint64_t limit);
uint64_t parallel_narrow_u64(uint32_t* dst, const uint64_t* src, size_t count, uint64_t limit);
void copy_d2h(tg_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes);
inline bool is_pinned_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Read-only input that may live on the host: returns a device pointer,
// copying into a scratch slot when needed.
template <typename T>
const T* dev_in(tg_ctx* ctx, const T* p, size_t count, int slot) {
  if (count == 0) return ctx->scratch_t<T>(slot, 1);
  if (is_device_ptr(p)) return p;
  T* d = ctx->scratch_t<T>(slot, count);
  if (count * sizeof(T) >= kPipeMin && !is_pinned_host(p))
    copy_h2d(ctx, d, p, count * sizeof(T));
  else
    TGB_CUDA(cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return d;
}

// Output that may live on the host: write into dev(), then finish() copies
// back (and synchronises) when the destination is host memory.
template <typename T>
struct DevOut {
  tg_ctx* ctx;
  T* user;
  size_t count;
  T* d;
  bool host;
  DevOut(tg_ctx* c, T* u, size_t n, int slot) : ctx(c), user(u), count(n) {
    host = !is_device_ptr(u);
    d = host ? c->scratch_t<T>(slot, n ? n : 1) : u;
  }
  T* dev() { return d; }
  void finish() {
    if (host && count) {
      if (count * sizeof(T) >= kPipeMin && !is_pinned_host(user)) {
        copy_d2h(ctx, user, d, count * sizeof(T));
        return;
      }
      TGB_CUDA(cudaMemcpyAsync(user, d, count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
    }
    ctx->sync();
  }
};

inline unsigned grid_for(uint64_t work, unsigned per_block, unsigned cap = 148u * 64u) {
  uint64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

}  // namespace tgb

namespace tgb {
// Thread-local message + exception → error-code translation for the C-ABI.
void set_last_error(const std::string& m);
template <typename F>
int guard(F&& f) {
  try {
    f();
    return TG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of memory");
    return TG_ERR_INTERNAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return TG_ERR_INTERNAL;
  }
}

__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) {
  return __reduce_min_sync(0xffffffffu, v);
}
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
  return __reduce_max_sync(0xffffffffu, v);
}

// Validates a permutation (reorder.cpp:10-21); optionally writes its inverse (u32).
void check_permutation(tg_ctx* ctx, const uint64_t* perm_dev, uint64_t n, uint32_t* inv_dev);
// Rows [rb, re) of a u32 CSR ordered by length descending, ties by id (K3's
// schedule). Stream-ordered; uses private temporaries, not scratch slots.
void sort_rows_by_length(tg_ctx* ctx, const uint32_t* off, uint64_t rb, uint64_t re,
                         uint32_t* order_dev);
// Ids [0, n) ordered by val[id] descending, ties by id (stable radix sort).
void sort_ids_by_value_desc(tg_ctx* ctx, const uint32_t* val, uint64_t n, uint32_t* order_dev);
// In-place exclusive prefix sum of n u64 values (device).
void exclusive_scan_u64(tg_ctx* ctx, uint64_t* data, uint64_t n);
// Mean us to read `rows` random rows of [0, region_rows) (R bytes at
// `stride`) from device-visible memory, L2 flushed before each launch.
double measure_rows_us(tg_ctx* ctx, const uint8_t* src_dev, uint64_t region_rows, uint64_t stride,
                       uint64_t R, uint64_t rows, int reps);

}  // namespace tgb
