// the reference's binary containers loaded straight into
// the device tiers, without materialising the N x R matrix or the u64 CSR in
// host memory first.
//
// Formats (reference proj/include/tiergraph/io.hpp:14-22, little-endian):
//   CSRG v1: "CSRG", u32 version, u64 n, u64 e, (n+1) x u64 offsets, e x u64 targets
//   FEAT v1: "FEAT", u32 version, u64 rows, u64 dim, u32 elem_bytes, rows*dim*eb bytes
// Header errors keep the reference's messages (io.cpp:65-75, 95-110, 163-180):
// bad magic / unsupported version / truncated ... -> FormatError; a file that
// cannot be opened -> IoError.
//
// Both loaders stream the payload through two pinned staging buffers: the
// host reads chunk k+1 from the file while the GPU consumes chunk k
// (narrowing the CSR to the u32 device layout; placing feature rows into
// this device's HBM slots and the pinned cold tier by the permutation).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "internal.cuh"
#include "store_internal.cuh"

namespace tgb {
namespace {

[[noreturn]] void io_error(const std::string& m) { throw Error(TG_ERR_IO, m); }

struct File {
  int fd = -1;
  uint64_t size = 0, pos = 0;
  std::string path;
  explicit File(const char* p) : path(p ? p : "") {
    fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) io_error("cannot open for reading: " + path);  // io.cpp:27-31
    struct stat st;
    if (::fstat(fd, &st) == 0) size = static_cast<uint64_t>(st.st_size);
  }
  ~File() {
    if (fd >= 0) ::close(fd);
  }
  // reads exactly n bytes at the current position (io.cpp:40-46 message)
  void read_exact(void* p, uint64_t n, const char* what) {
    uint64_t got = 0;
    while (got < n) {
      const ssize_t r = ::pread(fd, static_cast<char*>(p) + got, n - got, pos + got);
      if (r <= 0) break;
      got += static_cast<uint64_t>(r);
    }
    pos += got;
    if (got != n)
      format_error(path + ": truncated while reading " + what + " (wanted " + std::to_string(n) +
                   " bytes, got " + std::to_string(got) + ")");
  }
  template <typename T>
  T get(const char* what) {
    T v;
    read_exact(&v, sizeof(T), what);
    return v;
  }
  void expect(const char magic[4]) {  // io.cpp:65-75
    char got[4];
    read_exact(got, 4, "magic");
    if (std::memcmp(got, magic, 4) != 0)
      format_error(path + ": bad magic \"" + std::string(got, 4) + "\", expected \"" +
                   std::string(magic, 4) + "\"");
    const uint32_t version = get<uint32_t>("version");
    if (version != 1) format_error(path + ": unsupported version " + std::to_string(version));
  }
  // the payload must be there before any device work starts
  void need(uint64_t bytes, const char* what) {
    const uint64_t have = size > pos ? size - pos : 0;
    if (have < bytes)
      format_error(path + ": truncated while reading " + what + " (wanted " +
                   std::to_string(bytes) + " bytes, got " + std::to_string(have) + ")");
  }
};

// Double-buffered pinned staging: fill(k) reads chunk k on the host while
// the stream still consumes chunk k-1 from the other buffer.
struct Staging {
  tg_ctx* ctx;
  uint8_t* buf[2] = {nullptr, nullptr};
  uint8_t* dev[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  uint64_t cap;
  Staging(tg_ctx* c, uint64_t bytes) : ctx(c), cap(bytes) {
    for (int i = 0; i < 2; ++i) {
      TGB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&buf[i]), cap, cudaHostAllocMapped));
      void* d = nullptr;
      TGB_CUDA(cudaHostGetDevicePointer(&d, buf[i], 0));
      dev[i] = static_cast<uint8_t*>(d);
      TGB_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
  }
  ~Staging() {
    for (int i = 0; i < 2; ++i) {
      if (done[i]) {
        cudaEventSynchronize(done[i]);
        cudaEventDestroy(done[i]);
      }
      if (buf[i]) cudaFreeHost(buf[i]);
    }
  }
  // wait until the GPU is done with buffer b, then it may be refilled
  void acquire(int b) { TGB_CUDA(cudaEventSynchronize(done[b])); }
  void release(int b) { TGB_CUDA(cudaEventRecord(done[b], ctx->stream)); }
};

constexpr uint64_t kStageBytes = 64ull << 20;

__global__ void narrow_chunk_kernel(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                                    uint64_t count, uint64_t base, uint64_t n,
                                    unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = in[i];
    if (v >= n) atomicMin(bad, (unsigned long long)(base + i));
    out[i] = static_cast<uint32_t>(v);
  }
}

// Rows [r0, r0 + cnt) of the ORIGINAL matrix (staged, mapped) to their tier
// slots: new id p = new_id_of[r]; p < lb -> HBM slot p; lb <= p < mb and
// (p - lb) mod D == dev -> HBM slot lb + (p - lb) / D; p >= mb -> cold slot
// p - mb (pinned, stride cs); rows owned by other devices are skipped.
// One warp per row, 16 B vectors when R allows.
template <typename V>
__global__ void __launch_bounds__(256) place_chunk_kernel(const uint8_t* __restrict__ src,
                                                          uint64_t r0, uint64_t cnt, uint64_t R,
                                                          const uint64_t* __restrict__ new_id_of,
                                                          uint8_t* local, uint8_t* cold, uint64_t cs,
                                                          uint64_t lb, uint64_t mb, uint32_t D,
                                                          uint32_t dev, uint8_t* tail, uint64_t H) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t C = R / sizeof(V);
  for (uint64_t i = warp; i < cnt; i += nw) {
    const uint64_t p = new_id_of[r0 + i];
    uint8_t* d;
    const V* s = reinterpret_cast<const V*>(src + i * R);
    if (p >= mb && H) {  // TG_COLD_SPLIT_TAIL: whole lines to the host row, the rest to HBM
      V* dh = reinterpret_cast<V*>(cold + (p - mb) * cs);
      V* dt = reinterpret_cast<V*>(tail + (p - mb) * (R - H));
      const uint64_t Hc = H / sizeof(V);
      for (uint64_t c = lane; c < C; c += 32) {
        if (c < Hc) dh[c] = s[c];
        else dt[c - Hc] = s[c];
      }
      continue;
    }
    if (p < lb) {
      d = local + p * R;
    } else if (p < mb) {
      const uint64_t o = p - lb;
      if (o % D != dev) continue;
      d = local + (lb + o / D) * R;
    } else {
      d = cold + (p - mb) * cs;
    }
    V* dv = reinterpret_cast<V*>(d);
    for (uint64_t c = lane; c < C; c += 32) dv[c] = s[c];
  }
}

}  // namespace
}  // namespace tgb

using namespace tgb;

extern "C" {

int tg_graph_load_csrg(tg_ctx* ctx, const char* path, tg_graph** out) {
  return guard([&] {
    if (!ctx || !out) domain_error("tg_graph_load_csrg: null argument");
    File f(path);
    f.expect("CSRG");
    const uint64_t n = f.get<uint64_t>("num_nodes");
    const uint64_t e = f.get<uint64_t>("num_edges");
    if (n >= 0xffffffffull || e >= 0xffffffffull)
      domain_error("tg_graph_load_csrg: n and e must be < 2^32 for the u32 device layout");
    f.need((n + 1) * 8, "offsets");
    DeviceGuard dg(ctx->device);
    // offsets: whole array to the device (u64), narrowed + validated there
    uint64_t* off64 = nullptr;
    uint32_t* tgt32 = nullptr;
    TGB_CUDA(tgb::dev_malloc_async(&off64, 8 * (n + 1), ctx->stream));
    TGB_CUDA(tgb::dev_malloc(&tgt32, 4 * std::max<uint64_t>(e, 1) + 16));  // +16: K3 reads 16 B target groups
    auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 1);
    TGB_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
    {
      Staging st(ctx, kStageBytes);
      const uint64_t per = kStageBytes / 8;
      int b = 0;
      for (uint64_t i0 = 0; i0 < n + 1; i0 += per, b ^= 1) {
        const uint64_t cnt = std::min(per, n + 1 - i0);
        st.acquire(b);
        f.read_exact(st.buf[b], cnt * 8, "offsets");
        TGB_CUDA(cudaMemcpyAsync(off64 + i0, st.buf[b], cnt * 8, cudaMemcpyHostToDevice, ctx->stream));
        st.release(b);
      }
      f.need(e * 8, "targets");
      for (uint64_t i0 = 0; i0 < e; i0 += per, b ^= 1) {
        const uint64_t cnt = std::min(per, e - i0);
        st.acquire(b);
        f.read_exact(st.buf[b], cnt * 8, "targets");
        narrow_chunk_kernel<<<grid_for(cnt, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
            reinterpret_cast<const uint64_t*>(st.dev[b]), tgt32 + i0, cnt, i0, n, bad);
        TGB_LAUNCHED();
        st.release(b);
      }
      ctx->sync();
    }
    unsigned long long hb;
    TGB_CUDA(cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost));
    tg_graph* g = nullptr;
    try {
      // offsets validated + narrowed by the regular constructor path
      if (hb != ~0ull) {
        cudaFree(tgt32);
        tgt32 = nullptr;
        format_error("csr: target out of range at edge " + std::to_string(hb));
      }
      graph_from_device(ctx, off64, tgt32, n, e, &g);  // takes ownership of tgt32
      tgt32 = nullptr;
    } catch (...) {
      cudaFreeAsync(off64, ctx->stream);
      if (tgt32) cudaFree(tgt32);
      throw;
    }
    TGB_CUDA(cudaFreeAsync(off64, ctx->stream));
    ctx->sync();
    *out = g;
  });
}

int tg_store_place_feat(tg_store* s, const char* path, const uint64_t* new_id_of) {
  return guard([&] {
    tg_ctx* ctx = s->ctx;
    if (s->flags & TG_COLD_INDIRECT)
      domain_error("tg_store_place_feat: TG_COLD_INDIRECT reads a matrix in memory; place from a "
                   "file into the reordered cold tier instead");
    File f(path);
    f.expect("FEAT");
    const uint64_t rows = f.get<uint64_t>("num_rows");
    const uint64_t dim = f.get<uint64_t>("dim");
    const uint32_t eb = f.get<uint32_t>("elem_bytes");
    const uint64_t N = s->L.num_rows, R = s->R;
    if (rows != N || dim * eb != R)
      format_error(f.path + ": holds " + std::to_string(rows) + " rows of " +
                   std::to_string(dim * eb) + " bytes, the layout has " + std::to_string(N) +
                   " rows of " + std::to_string(R) + " bytes");
    f.need(rows * R, "feature data");
    DeviceGuard dg(ctx->device);
    if (N == 0) {
      s->placed = true;
      return;
    }
    const uint64_t* perm = dev_in(ctx, new_id_of, N, kStageIn0);
    check_permutation(ctx, perm, N, nullptr);
    const uint8_t* cold_dev = ensure_cold_tier(s);
    const int w = vec_width(R, {});
    const uint64_t per = std::max<uint64_t>(1, kStageBytes / R);
    {
      Staging st(ctx, per * R);
      int b = 0;
      for (uint64_t r0 = 0; r0 < N; r0 += per, b ^= 1) {
        const uint64_t cnt = std::min(per, N - r0);
        st.acquire(b);
        f.read_exact(st.buf[b], cnt * R, "feature data");
        const unsigned grid = grid_for(cnt * 32, 256, ctx->num_sms * 8);
        const uint64_t lb = s->L.local_boundary, mb = s->L.multi_boundary;
        uint8_t* cold = const_cast<uint8_t*>(cold_dev);
        if (w == 16)
          place_chunk_kernel<uint4><<<grid, 256, 0, ctx->stream>>>(st.dev[b], r0, cnt, R, perm,
                                                                   s->local, cold, s->cold_stride,
                                                                   lb, mb, s->L.num_devices, s->dev,
                                                                   s->cold_tail, s->cold_head);
        else
          place_chunk_kernel<uint8_t><<<grid, 256, 0, ctx->stream>>>(st.dev[b], r0, cnt, R, perm,
                                                                     s->local, cold, s->cold_stride,
                                                                     lb, mb, s->L.num_devices,
                                                                     s->dev, s->cold_tail,
                                                                     s->cold_head);
        TGB_LAUNCHED();
        st.release(b);
      }
      ctx->sync();
    }
    s->placed = true;
  });
}

}  // extern "C"
