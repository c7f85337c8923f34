// C-ABI plumbing: error reporting, contexts, device selection, the launch
// counter, the graph reorder (K9, Algorithm 2) and the link microbenchmarks
// used for the roofline denominators.
#include <map>
#include <mutex>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "internal.cuh"

namespace tgb {

std::atomic<uint64_t> g_launches{0};
thread_local std::string t_err;
void set_last_error(const std::string& m) { t_err = m; }

// ---------------------------------------------------------------- scan
// Exclusive scan of u64 values in place, three phases (tile sums, scan of the
// sums in one CTA, add-back). Used by reorder_graph's offset rebuild.
constexpr int kScanTile = 2048;

__global__ void __launch_bounds__(1024) tile_sum_kernel(const uint64_t* __restrict__ in, uint64_t n,
                                                        uint64_t* __restrict__ sums) {
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  uint64_t s = 0;
  for (uint64_t i = base + threadIdx.x; i < base + kScanTile && i < n; i += blockDim.x) s += in[i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ uint64_t ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += ws[w];
    sums[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) sums_scan_kernel(uint64_t* __restrict__ sums, uint64_t m) {
  __shared__ uint64_t part[1024];
  const uint64_t per = (m + blockDim.x - 1) / blockDim.x;
  const uint64_t b = threadIdx.x * per, e = b + per < m ? b + per : m;
  uint64_t local = 0;
  for (uint64_t i = b; i < e; ++i) local += sums[i];
  part[threadIdx.x] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const uint64_t v = part[i];
      part[i] = run;
      run += v;
    }
  }
  __syncthreads();
  uint64_t run = part[threadIdx.x];
  for (uint64_t i = b; i < e; ++i) {
    const uint64_t v = sums[i];
    sums[i] = run;
    run += v;
  }
}

__global__ void __launch_bounds__(1024) tile_scan_kernel(uint64_t* __restrict__ data, uint64_t n,
                                                         const uint64_t* __restrict__ sums) {
  // each thread handles 2 consecutive elements of the tile
  __shared__ uint64_t ws[32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + 2 * threadIdx.x;
  const uint64_t a = base < n ? data[base] : 0;
  const uint64_t b = base + 1 < n ? data[base + 1] : 0;
  uint64_t incl = a + b;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) ws[w] = incl;
  __syncthreads();
  if (w == 0) {
    const uint64_t t = ws[lane];
    uint64_t ti = t;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    ws[lane] = ti - t;
  }
  __syncthreads();
  const uint64_t excl = sums[blockIdx.x] + ws[w] + incl - (a + b);
  if (base < n) data[base] = excl;
  if (base + 1 < n) data[base + 1] = excl + a;
}

void exclusive_scan_u64(tg_ctx* ctx, uint64_t* data, uint64_t n) {
  if (n == 0) return;
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  uint64_t* sums = ctx->scratch_t<uint64_t>(kScratchE, tiles);
  tile_sum_kernel<<<static_cast<unsigned>(tiles), 1024, 0, ctx->stream>>>(data, n, sums);
  TGB_LAUNCHED();
  sums_scan_kernel<<<1, 1024, 0, ctx->stream>>>(sums, tiles);
  TGB_LAUNCHED();
  tile_scan_kernel<<<static_cast<unsigned>(tiles), 1024, 0, ctx->stream>>>(data, n, sums);
  TGB_LAUNCHED();
}

// ------------------------------------------------------- K9 reorder_graph
// reorder.cpp:39-66: scatter row lengths to their new ids, prefix-sum them,
// then copy every old row into its new block with targets relabelled. Rows
// keep their old internal order (they are NOT re-sorted).
__global__ void scatter_lengths_kernel(const uint64_t* __restrict__ off, const uint64_t* __restrict__ perm,
                                       uint64_t n, uint64_t* __restrict__ lens) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x)
    lens[perm[u]] = off[u + 1] - off[u];
}

__global__ void relabel_rows_kernel(const uint64_t* __restrict__ off, const uint64_t* __restrict__ tgt,
                                    const uint64_t* __restrict__ perm, uint64_t n,
                                    const uint64_t* __restrict__ new_off, uint64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t u = warp; u < n; u += nw) {
    const uint64_t b = off[u], e = off[u + 1];
    uint64_t* dst = out + new_off[perm[u]];
    for (uint64_t i = b + lane; i < e; i += 32) dst[i - b] = perm[tgt[i]];
  }
}

}  // namespace tgb

struct tg_ctx;
using namespace tgb;

namespace tgb {
constexpr size_t kPipeChunk = 64ull << 20;

static void pipe_init(tg_ctx* c) {
  if (c->pipe_buf[0]) return;
  for (int i = 0; i < 2; ++i) {
    TGB_CUDA(cudaHostAlloc(&c->pipe_buf[i], kPipeChunk, cudaHostAllocDefault));
    TGB_CUDA(cudaEventCreateWithFlags(&c->pipe_ev[i], cudaEventDisableTiming));
  }
}

// chunk k: host memcpy into pinned buffer k%2 (all cores), then its DMA on
// the stream; buffer k%2 is refilled only after chunk k-2's DMA completed
void copy_h2d(tg_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes, bool sync_end) {
  pipe_init(ctx);
  const size_t nch = (bytes + kPipeChunk - 1) / kPipeChunk;
  for (size_t k = 0; k < nch; ++k) {
    const size_t off = k * kPipeChunk, len = std::min(kPipeChunk, bytes - off);
    const int b = static_cast<int>(k & 1);
    TGB_CUDA(cudaEventSynchronize(ctx->pipe_ev[b]));  // its previous DMA (this call or an earlier one)
    parallel_memcpy(ctx->pipe_buf[b], static_cast<const char*>(src_host) + off, len);
    TGB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst_dev) + off, ctx->pipe_buf[b], len,
                             cudaMemcpyHostToDevice, ctx->stream));
    TGB_CUDA(cudaEventRecord(ctx->pipe_ev[b], ctx->stream));
  }
  if (sync_end) ctx->sync();
}

uint64_t copy_h2d_narrow(tg_ctx* ctx, uint32_t* dst_dev, const uint64_t* src_host, size_t count,
                         uint64_t limit) {
  pipe_init(ctx);
  constexpr size_t per = kPipeChunk / sizeof(uint32_t);
  uint64_t first = ~0ull;
  for (size_t off = 0, k = 0; off < count; off += per, ++k) {
    const size_t len = std::min(per, count - off);
    const int b = static_cast<int>(k & 1);
    TGB_CUDA(cudaEventSynchronize(ctx->pipe_ev[b]));
    const uint64_t f = parallel_narrow_u64(static_cast<uint32_t*>(ctx->pipe_buf[b]), src_host + off,
                                           len, limit);
    if (first == ~0ull && f != ~0ull) first = off + f;
    TGB_CUDA(cudaMemcpyAsync(dst_dev + off, ctx->pipe_buf[b], len * sizeof(uint32_t),
                             cudaMemcpyHostToDevice, ctx->stream));
    TGB_CUDA(cudaEventRecord(ctx->pipe_ev[b], ctx->stream));
  }
  return first;
}

// chunk k's DMA into pinned buffer k%2 is issued before chunk k-1 is moved
// out of buffer (k-1)%2 by the host cores
void copy_d2h(tg_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes) {
  pipe_init(ctx);
  const size_t nch = (bytes + kPipeChunk - 1) / kPipeChunk;
  auto issue = [&](size_t k) {
    const size_t off = k * kPipeChunk, len = std::min(kPipeChunk, bytes - off);
    const int b = static_cast<int>(k & 1);
    TGB_CUDA(cudaMemcpyAsync(ctx->pipe_buf[b], static_cast<const char*>(src_dev) + off, len,
                             cudaMemcpyDeviceToHost, ctx->stream));
    TGB_CUDA(cudaEventRecord(ctx->pipe_ev[b], ctx->stream));
  };
  issue(0);
  for (size_t k = 0; k < nch; ++k) {
    const size_t off = k * kPipeChunk, len = std::min(kPipeChunk, bytes - off);
    const int b = static_cast<int>(k & 1);
    TGB_CUDA(cudaEventSynchronize(ctx->pipe_ev[b]));
    if (k + 1 < nch) issue(k + 1);  // into the other buffer, drained at step k-1
    parallel_memcpy(static_cast<char*>(dst_host) + off, ctx->pipe_buf[b], len);
  }
  ctx->sync();
}
}  // namespace tgb

extern "C" {

const char* tg_last_error(void) { return t_err.c_str(); }
const char* tg_version(void) { return "tiergraph_b200 0.1 sm_100a"; }
uint64_t tg_kernel_launches(void) { return g_launches.load(); }

int tg_default_device(void) {
  if (const char* s = std::getenv("TIERGRAPH_DEVICES")) {
    const int d = std::atoi(s);
    if (d >= 0) return d;
  }
  return 0;
}

int tg_device_list(int* out, int cap) {
  std::vector<int> v;
  if (const char* s = std::getenv("TIERGRAPH_DEVICES")) {
    const char* p = s;
    while (*p) {
      char* end = nullptr;
      const long d = std::strtol(p, &end, 10);
      if (end == p) break;
      if (d >= 0) v.push_back(static_cast<int>(d));
      p = end;
      while (*p == ',' || *p == ' ') ++p;
    }
  }
  if (v.empty()) v.push_back(0);
  for (int i = 0; i < cap && i < static_cast<int>(v.size()); ++i) out[i] = v[i];
  return static_cast<int>(v.size());
}

int tg_device_count(void) {
  if (const char* s = std::getenv("TIERGRAPH_DEVICES")) {
    int n = 1;
    for (const char* p = s; *p; ++p) n += *p == ',';
    return n;
  }
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

static int ctx_create(int device, void* stream, bool given, tg_ctx** out) {
  return guard([&] {
    int count = 0;
    TGB_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
      domain_error("device " + std::to_string(device) + " out of range for " +
                   std::to_string(count) + " visible devices");
    DeviceGuard dg(device);
    int major = 0, minor = 0;
    TGB_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    TGB_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10 || minor != 0)
      throw Error(TG_ERR_INTERNAL, "tiergraph_b200 is built for sm_100a (B200); device " +
                                       std::to_string(device) + " is sm_" + std::to_string(major) +
                                       std::to_string(minor));
    // Keep freed stream-ordered temporaries (radix-sort status words, the
    // binned K1's partition buffer) mapped in the device's default pool
    // across calls, up to TIERGRAPH_POOL_KEEP_MB (default 8 GB): with the
    // pool's default threshold of 0 every call re-maps them (C2 selection
    // 0.43 ms of kernels took 1.46 ms per call).
    static bool pool_set[TG_MAX_DEVICES] = {};
    if (!pool_set[device % TG_MAX_DEVICES]) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = 8ull << 30;
        if (const char* e = std::getenv("TIERGRAPH_POOL_KEEP_MB")) keep = std::strtoull(e, nullptr, 10) << 20;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      cudaGetLastError();
      pool_set[device % TG_MAX_DEVICES] = true;
    }
    auto* c = new tg_ctx;
    c->device = device;
    TGB_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    if (given) {  // 0 = the legacy default stream, used as is
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      TGB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    *out = c;
  });
}

int tg_ctx_create(int device, tg_ctx** out) { return ctx_create(device, nullptr, false, out); }
int tg_ctx_create_on_stream(int device, void* stream, tg_ctx** out) {
  return ctx_create(device, stream, true, out);
}

int tg_ctx_destroy(tg_ctx* c) {
  if (!c) return TG_OK;
  DeviceGuard dg(c->device);
  cudaStreamSynchronize(c->stream);
  for (int i = 0; i < kNumSlots; ++i)
    if (c->slot_ptr[i]) cudaFree(c->slot_ptr[i]);
  for (int i = 0; i < 2; ++i) {
    if (c->pipe_buf[i]) cudaFreeHost(c->pipe_buf[i]);
    if (c->pipe_ev[i]) cudaEventDestroy(c->pipe_ev[i]);
  }
  if (c->aux) {
    cudaStreamSynchronize(c->aux);
    cudaStreamSynchronize(c->aux2);
    cudaStreamSynchronize(c->aux3);
    cudaStreamDestroy(c->aux);
    cudaStreamDestroy(c->aux2);
    cudaStreamDestroy(c->aux3);
    cudaEventDestroy(c->ev_fork);
    cudaEventDestroy(c->ev_join);
    cudaEventDestroy(c->ev_join2);
    cudaEventDestroy(c->ev_join3);
  }
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return TG_OK;
}

int tg_ctx_trim(tg_ctx* c) {
  return guard([&] {
    DeviceGuard dg(c->device);
    c->sync();
    for (int i = 0; i < kNumSlots; ++i) {
      if (c->slot_ptr[i]) TGB_CUDA(cudaFree(c->slot_ptr[i]));
      c->slot_ptr[i] = nullptr;
      c->slot_size[i] = 0;
    }
    trim_default_pool();
  });
}

int tg_memcpy_async(tg_ctx* c, void* dst, const void* src, uint64_t bytes) {
  return guard([&] {
    if (!bytes) return;
    DeviceGuard dg(c->device);
    TGB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
  });
}

int tg_ctx_sync(tg_ctx* c) {
  return guard([&] { c->sync(); });
}
void* tg_ctx_stream(tg_ctx* c) { return c ? c->stream : nullptr; }
int tg_ctx_device(tg_ctx* c) { return c ? c->device : -1; }

int tg_reorder_graph(tg_ctx* ctx, const uint64_t* offsets, const uint64_t* targets, uint64_t n,
                     uint64_t e, const uint64_t* perm, uint64_t perm_len, uint64_t* out_offsets,
                     uint64_t* out_targets) {
  return guard([&] {
    if (perm_len != n)
      domain_error("permutation length " + std::to_string(perm_len) + " != num_nodes " +
                   std::to_string(n));  // reorder.cpp:41-43
    DeviceGuard dg(ctx->device);
    const uint64_t* p = dev_in(ctx, perm, n, kStageIn0);
    check_permutation(ctx, p, n, nullptr);
    const uint64_t* off = dev_in(ctx, offsets, n + 1, kStageIn1);
    const uint64_t* tgt = dev_in(ctx, targets, e, kStageIn2);
    DevOut<uint64_t> oo(ctx, out_offsets, n + 1, kStageOut0);
    DevOut<uint64_t> ot(ctx, out_targets, e, kStageOut1);
    TGB_CUDA(cudaMemsetAsync(oo.dev(), 0, 8 * (n + 1), ctx->stream));
    if (n) {
      scatter_lengths_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(off, p, n, oo.dev());
      TGB_LAUNCHED();
    }
    exclusive_scan_u64(ctx, oo.dev(), n + 1);  // lens[v] -> offsets[v]; offsets[n] = e
    if (n && e) {
      relabel_rows_kernel<<<grid_for(n * 32, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
          off, tgt, p, n, oo.dev(), ot.dev());
      TGB_LAUNCHED();
    }
    if (oo.host && n + 1)
      TGB_CUDA(cudaMemcpyAsync(out_offsets, oo.dev(), 8 * (n + 1), cudaMemcpyDeviceToHost,
                               ctx->stream));
    ot.finish();
  });
}

}  // extern "C"

// ------------------------------------------------------------ measurement
namespace tgb {

__global__ void host_read_kernel(const uint8_t* __restrict__ src, uint64_t rows, uint64_t R,
                                 uint8_t* __restrict__ dst, uint64_t seed, uint64_t region = 0,
                                 uint64_t stride = 0) {
  // `rows` random rows of [0, region) (default: all of them), 16 B vectors,
  // one warp per row
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  if (!region) region = rows;
  if (!stride) stride = R;
  for (uint64_t i = warp; i < rows; i += nw) {
    uint64_t x = (i + seed * 0x632BE59BD9B4E019ull) * 0x9E3779B97F4A7C15ull;
    x ^= x >> 31;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 29;
    const uint64_t r = x % region;
    const uint4* s = reinterpret_cast<const uint4*>(src + r * stride);
    uint4* d = reinterpret_cast<uint4*>(dst + i * R);
    for (uint64_t c = lane; c < R / 16; c += 32) d[c] = s[c];
  }
}

double measure_rows_us(tg_ctx* ctx, const uint8_t* src_dev, uint64_t region_rows, uint64_t stride,
                       uint64_t R, uint64_t rows, int reps) {
  if (R % 16 || R == 0 || stride % 16) domain_error("row_bytes and stride must be multiples of 16");
  if (!rows || !region_rows) domain_error("empty measurement");
  uint8_t* d = ctx->scratch_t<uint8_t>(kScratchF, rows * R);
  uint8_t* fl = ctx->scratch_t<uint8_t>(kScratchE, 256ull << 20);
  cudaEvent_t a, b;
  TGB_CUDA(cudaEventCreate(&a));
  TGB_CUDA(cudaEventCreate(&b));
  const unsigned grid = ctx->num_sms * 8;
  double tot = 0;
  for (int i = 0; i <= reps; ++i) {
    TGB_CUDA(cudaMemsetAsync(fl, i, 256ull << 20, ctx->stream));  // L2 flush, as the bench
    TGB_CUDA(cudaEventRecord(a, ctx->stream));
    host_read_kernel<<<grid, 256, 0, ctx->stream>>>(src_dev, rows, R, d, 1000 + i, region_rows,
                                                    stride);
    TGB_LAUNCHED();
    TGB_CUDA(cudaEventRecord(b, ctx->stream));
    TGB_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    TGB_CUDA(cudaEventElapsedTime(&ms, a, b));
    if (i) tot += ms;  // the first launch warms
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return tot / std::max(reps, 1) * 1e3;
}

}  // namespace tgb

extern "C" {

int tg_measure_host_read_gbps(tg_ctx* ctx, uint64_t bytes, uint64_t R, int reps, double* gbps) {
  return guard([&] {
    if (R % 16 || R == 0) domain_error("row_bytes must be a positive multiple of 16");
    DeviceGuard dg(ctx->device);
    const uint64_t rows = bytes / R;
    void* h = nullptr;
    TGB_CUDA(cudaHostAlloc(&h, rows * R, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(h, 1, rows * R);
    void* hd = nullptr;
    TGB_CUDA(cudaHostGetDevicePointer(&hd, h, 0));
    uint8_t* d = ctx->scratch_t<uint8_t>(kScratchF, rows * R);
    cudaEvent_t a, b;
    TGB_CUDA(cudaEventCreate(&a));
    TGB_CUDA(cudaEventCreate(&b));
    const unsigned grid = ctx->num_sms * 8;
    host_read_kernel<<<grid, 256, 0, ctx->stream>>>(static_cast<uint8_t*>(hd), rows, R, d, 1);
    TGB_LAUNCHED();
    float best = 1e30f;
    for (int i = 0; i < reps; ++i) {
      TGB_CUDA(cudaEventRecord(a, ctx->stream));
      host_read_kernel<<<grid, 256, 0, ctx->stream>>>(static_cast<uint8_t*>(hd), rows, R, d, i + 7);
      TGB_LAUNCHED();
      TGB_CUDA(cudaEventRecord(b, ctx->stream));
      TGB_CUDA(cudaEventSynchronize(b));
      float ms = 0;
      TGB_CUDA(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFreeHost(h);
    *gbps = static_cast<double>(rows * R) / (best * 1e-3) / 1e9;
  });
}

int tg_measure_host_rows_us(tg_ctx* ctx, const void* host, uint64_t region_rows, uint64_t stride,
                            uint64_t R, uint64_t rows, int reps, double* us) {
  return guard([&] {
    DeviceGuard dg(ctx->device);
    const void* hd = is_device_ptr(host) ? host : mapped_device_ptr(host);
    if (!hd) domain_error("tg_measure_host_rows_us: the region is not device-visible");
    *us = measure_rows_us(ctx, static_cast<const uint8_t*>(hd), region_rows, stride, R, rows, reps);
  });
}

int tg_measure_hbm_copy_gbps(tg_ctx* ctx, uint64_t bytes, int reps, double* gbps) {
  return guard([&] {
    DeviceGuard dg(ctx->device);
    uint8_t* s = ctx->scratch_t<uint8_t>(kScratchE, bytes);
    uint8_t* d = ctx->scratch_t<uint8_t>(kScratchF, bytes);
    TGB_CUDA(cudaMemsetAsync(s, 1, bytes, ctx->stream));
    cudaEvent_t a, b;
    TGB_CUDA(cudaEventCreate(&a));
    TGB_CUDA(cudaEventCreate(&b));
    float best = 1e30f;
    for (int i = 0; i < reps + 1; ++i) {
      TGB_CUDA(cudaEventRecord(a, ctx->stream));
      TGB_CUDA(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
      TGB_CUDA(cudaEventRecord(b, ctx->stream));
      TGB_CUDA(cudaEventSynchronize(b));
      float ms = 0;
      TGB_CUDA(cudaEventElapsedTime(&ms, a, b));
      if (i) best = std::min(best, ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *gbps = 2.0 * static_cast<double>(bytes) / (best * 1e-3) / 1e9;  // read + write
  });
}

}  // extern "C"
