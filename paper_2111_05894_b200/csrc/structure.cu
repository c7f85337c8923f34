// Graph-structure tiering — SURVEY §8(f) row 2 (the
// reference's estimate is tools/tiergraph_cli.cpp:389-406, --structure-of).
// Placement of the transposed, score-reordered graph's neighbour lists into
// the tiers of a TierLayout (structure_internal.cuh): replicated rows and
// this device's interleaved slice in HBM, cold rows in pinned mapped host
// memory. The sampler (sampling.cu) reads row v through resolve(v).
//
// Placement runs on the device: the u64 CSR is narrowed to u32 into a
// transient device copy (chunked from the host, range-checked as
// tg_graph_create does), the interleaved rows' slice starts come from one
// exclusive scan over (device, slot)-ordered row lengths, and each tier is a
// copy out of the transient: rows [0, lb) and the cold edge suffix are
// contiguous edge ranges (one D2D / one D2H copy), the slice is a
// warp-per-row copy of the rows (v - lb) % D == self.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "internal.cuh"
#include "structure_internal.cuh"

namespace tgb {
void validate_layout(const tg_layout& l);  // tiering.cu (tiering.cpp:10-18)

namespace {

__global__ void sg_narrow_offsets(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                                  uint64_t n, uint64_t e, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = in[i];
    bool ok = v <= e;
    if (i == 0) ok = ok && v == 0;
    if (i == n) ok = ok && v == e;
    if (i > 0) ok = ok && in[i - 1] <= v;
    if (!ok) atomicMin(bad, (unsigned long long)i);
    out[i] = static_cast<uint32_t>(v);
  }
}

__global__ void sg_narrow_targets(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                                  uint64_t count, uint64_t base, uint64_t n,
                                  unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = in[i];
    if (v >= n) atomicMin(bad, (unsigned long long)(base + i));
    out[i] = static_cast<uint32_t>(v);
  }
}

// Row lengths of [lb, mb) in (device, slot) order: entry d*S + slot is row
// lb + slot*D + d (0 past mb). One extra trailing 0 for the scan's total.
__global__ void sg_class_lengths(const uint32_t* __restrict__ off, uint64_t lb, uint64_t mb,
                                 uint32_t D, uint64_t S, uint64_t* __restrict__ len) {
  const uint64_t total = static_cast<uint64_t>(D) * S + 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t v = 0;
    if (i < total - 1) {
      const uint64_t d = i / S, slot = i % S, r = lb + slot * D + d;
      if (r < mb) v = off[r + 1] - off[r];
    }
    len[i] = v;
  }
}

// start[r - lb] = scan[d*S + slot] - scan[d*S] (the row's place in device d's slice)
__global__ void sg_starts(const uint64_t* __restrict__ scan, uint64_t lb, uint64_t mb, uint32_t D,
                          uint64_t S, uint32_t* __restrict__ start) {
  for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < mb - lb;
       o += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = o % D, slot = o / D;
    start[o] = static_cast<uint32_t>(scan[d * S + slot] - scan[d * S]);
  }
}

// One warp per row of this device's class: copy its neighbour ids into the slice.
__global__ void sg_fill_slice(const uint32_t* __restrict__ off, const uint32_t* __restrict__ tgt,
                              uint64_t lb, uint64_t mb, uint32_t D, uint32_t self,
                              const uint32_t* __restrict__ start, uint32_t* __restrict__ slice) {
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t rows = mb > lb + self ? (mb - lb - self + D - 1) / D : 0;
  for (uint64_t k = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; k < rows; k += warps) {
    const uint64_t r = lb + self + k * D;
    const uint32_t b = off[r], len = off[r + 1] - b;
    uint32_t* dst = slice + start[r - lb];
    for (uint32_t j = lane; j < len; j += 32) dst[j] = tgt[b + j];
  }
}

}  // namespace
}  // namespace tgb

tgb::SGraphView tg_sgraph::view() const {
  tgb::SGraphView v;
  v.off = off;
  v.rep = rep;
  for (uint32_t d = 0; d < TG_MAX_DEVICES; ++d) v.ilv[d] = d == dev ? slice : peer[d];
  v.ilv_start = ilv_start;
  v.cold = cold_dev;
  v.cold_base = e - cold_len;
  v.lb = static_cast<uint32_t>(L.local_boundary);
  v.mb = static_cast<uint32_t>(L.multi_boundary);
  v.n = static_cast<uint32_t>(n);
  v.D = L.num_devices;
  v.self = dev;
  return v;
}

using namespace tgb;

extern "C" {

uint64_t tg_sgraph_cold_bytes(const uint64_t* offsets, uint64_t n, const tg_layout* layout) {
  if (!offsets || !layout || layout->multi_boundary > n) return 0;
  uint64_t a = 0, b = 0;
  if (is_device_ptr(offsets)) {
    if (cudaMemcpy(&a, offsets + layout->multi_boundary, 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(&b, offsets + n, 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
  } else {
    a = offsets[layout->multi_boundary];
    b = offsets[n];
  }
  return std::max<uint64_t>(4 * (b - a), 16);
}

int tg_sgraph_destroy(tg_sgraph* s);

int tg_sgraph_create(tg_ctx* ctx, const tg_layout* layout, uint32_t device_index,
                     const uint64_t* offsets, const uint64_t* targets, uint64_t n, uint64_t e,
                     void* cold_host, uint64_t cold_bytes, int cold_fill, tg_sgraph** out) {
  return guard([&] {
    if (!ctx || !layout || !out || (!offsets && n)) domain_error("tg_sgraph_create: null argument");
    validate_layout(*layout);
    if (layout->num_rows != n)
      domain_error("tg_sgraph_create: layout covers " + std::to_string(layout->num_rows) +
                   " rows but the graph has " + std::to_string(n) + " nodes");
    if (device_index >= layout->num_devices)
      domain_error("requesting device " + std::to_string(device_index) + " out of range for " +
                   std::to_string(layout->num_devices) + " devices");
    if (layout->num_devices > TG_MAX_DEVICES)
      domain_error("tg_sgraph_create: at most " + std::to_string(TG_MAX_DEVICES) + " devices");
    if (n >= 0xffffffffull || e >= 0xffffffffull)
      domain_error("tg_sgraph_create: n and e must be < 2^32 for the u32 device layout");
    DeviceGuard dg(ctx->device);
    auto* s = new tg_sgraph;
    s->ctx = ctx;
    s->L = *layout;
    s->dev = device_index;
    s->n = n;
    s->e = e;
    uint32_t* tmp = nullptr;
    uint64_t* lens = nullptr;
    try {
      const uint64_t lb = layout->local_boundary, mb = layout->multi_boundary;
      const uint32_t D = layout->num_devices;
      auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 2);
      TGB_CUDA(cudaMemsetAsync(bad, 0xff, 2 * sizeof(unsigned long long), ctx->stream));
      // offsets -> u32 on this device (every device holds them)
      TGB_CUDA(tgb::dev_malloc(&s->off, 4 * (n + 1)));
      const uint64_t* doff = dev_in(ctx, offsets, n + 1, kStageIn0);
      sg_narrow_offsets<<<grid_for(n + 1, 256), 256, 0, ctx->stream>>>(doff, s->off, n, e, bad);
      TGB_LAUNCHED();
      // the transient u32 copy of every neighbour id (range-checked)
      TGB_CUDA(tgb::dev_malloc(&tmp, 4 * std::max<uint64_t>(e, 1)));
      const bool tdev = is_device_ptr(targets);
      const uint64_t chunk = tdev ? std::max<uint64_t>(e, 1) : (32ull << 20);
      for (uint64_t base = 0; base < e; base += chunk) {
        const uint64_t cnt = std::min(chunk, e - base);
        const uint64_t* src = targets + base;
        if (!tdev) {
          auto* st = ctx->scratch_t<uint64_t>(kStageIn1, cnt);
          TGB_CUDA(cudaMemcpyAsync(st, src, cnt * 8, cudaMemcpyHostToDevice, ctx->stream));
          src = st;
        }
        sg_narrow_targets<<<grid_for(cnt, 256), 256, 0, ctx->stream>>>(src, tmp + base, cnt, base,
                                                                       n, bad + 1);
        TGB_LAUNCHED();
      }
      unsigned long long hb[2];
      TGB_CUDA(cudaMemcpyAsync(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      if (hb[0] != ~0ull)
        format_error("csr: offsets invalid at index " + std::to_string(hb[0]) +
                     " (need offsets[0]==0, monotone, offsets[num_nodes]==num_edges)");
      if (hb[1] != ~0ull) format_error("csr: target out of range at edge " + std::to_string(hb[1]));
      uint32_t off_lb = 0, off_mb = 0;
      TGB_CUDA(cudaMemcpy(&off_lb, s->off + lb, 4, cudaMemcpyDeviceToHost));
      TGB_CUDA(cudaMemcpy(&off_mb, s->off + mb, 4, cudaMemcpyDeviceToHost));
      // [0, lb): replicated
      TGB_CUDA(tgb::dev_malloc(&s->rep, 4 * std::max<uint64_t>(off_lb, 1)));
      if (off_lb)
        TGB_CUDA(cudaMemcpyAsync(s->rep, tmp, 4ull * off_lb, cudaMemcpyDeviceToDevice, ctx->stream));
      // [lb, mb): slice starts from one scan over (device, slot)-ordered lengths
      const uint64_t inter = mb - lb, S = (inter + D - 1) / D;
      TGB_CUDA(tgb::dev_malloc(&s->ilv_start, 4 * std::max<uint64_t>(inter, 1)));
      if (inter) {
        const uint64_t m = static_cast<uint64_t>(D) * S + 1;
        TGB_CUDA(tgb::dev_malloc(&lens, 8 * m));
        sg_class_lengths<<<grid_for(m, 256), 256, 0, ctx->stream>>>(s->off, lb, mb, D, S, lens);
        TGB_LAUNCHED();
        exclusive_scan_u64(ctx, lens, m);
        sg_starts<<<grid_for(inter, 256), 256, 0, ctx->stream>>>(lens, lb, mb, D, S, s->ilv_start);
        TGB_LAUNCHED();
        uint64_t se[2];
        TGB_CUDA(cudaMemcpyAsync(&se[0], lens + device_index * S, 8, cudaMemcpyDeviceToHost, ctx->stream));
        TGB_CUDA(cudaMemcpyAsync(&se[1], lens + (device_index + 1) * S, 8, cudaMemcpyDeviceToHost,
                                 ctx->stream));
        ctx->sync();
        s->slice_len = se[1] - se[0];
      }
      TGB_CUDA(tgb::dev_malloc(&s->slice, 4 * std::max<uint64_t>(s->slice_len, 1)));
      if (s->slice_len) {
        sg_fill_slice<<<grid_for((S + 7) / 8, 1, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
            s->off, tmp, lb, mb, D, device_index, s->ilv_start, s->slice);
        TGB_LAUNCHED();
      }
      // [mb, N): the contiguous edge suffix in pinned mapped host memory
      s->cold_len = e - off_mb;
      const uint64_t need = std::max<uint64_t>(4 * s->cold_len, 16);
      if (cold_host) {
        if (cold_bytes < need)
          domain_error("tg_sgraph_create: cold tier needs " + std::to_string(need) +
                       " bytes, got " + std::to_string(cold_bytes));
        void* dv = mapped_device_ptr(cold_host);
        if (!dv) domain_error("tg_sgraph_create: cold memory is not mapped for the device (register it)");
        s->cold_host = static_cast<uint32_t*>(cold_host);
        s->cold_dev = static_cast<const uint32_t*>(dv);
        s->cold_attached = true;
        s->cold_fill = cold_fill != 0;
      } else {
        TGB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->cold_host), need,
                               cudaHostAllocMapped | cudaHostAllocPortable));
        s->own_cold = true;
        void* dv = nullptr;
        TGB_CUDA(cudaHostGetDevicePointer(&dv, s->cold_host, 0));
        s->cold_dev = static_cast<const uint32_t*>(dv);
      }
      if (s->cold_len && s->cold_fill)
        TGB_CUDA(cudaMemcpyAsync(s->cold_host, tmp + off_mb, 4 * s->cold_len,
                                 cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      cudaFree(tmp);
      tmp = nullptr;
      cudaFree(lens);
      lens = nullptr;
      s->placed = true;
    } catch (...) {
      cudaFree(tmp);
      cudaFree(lens);
      tg_sgraph_destroy(s);
      throw;
    }
    *out = s;
  });
}

int tg_sgraph_destroy(tg_sgraph* s) {
  if (!s) return TG_OK;
  DeviceGuard dg(s->ctx->device);
  cudaStreamSynchronize(s->ctx->stream);
  cudaFree(s->off);
  cudaFree(s->rep);
  cudaFree(s->slice);
  cudaFree(s->ilv_start);
  if (s->own_cold) cudaFreeHost(s->cold_host);
  delete s;
  return TG_OK;
}

void* tg_sgraph_local_base(const tg_sgraph* s) { return s ? s->slice : nullptr; }

int tg_sgraph_set_peer(tg_sgraph* s, uint32_t d, const void* peer_slice_base) {
  return guard([&] {
    if (!s) domain_error("tg_sgraph_set_peer: null argument");
    if (d >= s->L.num_devices)
      domain_error("requesting device " + std::to_string(d) + " out of range for " +
                   std::to_string(s->L.num_devices) + " devices");
    s->peer[d] = static_cast<const uint32_t*>(peer_slice_base);
  });
}

void* tg_sgraph_cold_host(const tg_sgraph* s) { return s ? s->cold_host : nullptr; }

int tg_sgraph_info(const tg_sgraph* s, uint64_t* out) {
  return guard([&] {
    if (!s || !out) domain_error("tg_sgraph_info: null argument");
    uint32_t off_lb = 0;
    DeviceGuard dg(s->ctx->device);
    TGB_CUDA(cudaMemcpy(&off_lb, s->off + s->L.local_boundary, 4, cudaMemcpyDeviceToHost));
    out[0] = 4ull * off_lb;          // replicated rows' neighbour ids (HBM)
    out[1] = 4ull * s->slice_len;    // this device's interleaved slice (HBM)
    out[2] = 4ull * s->cold_len;     // cold rows (pinned host)
    out[3] = 4ull * (s->n + 1) + 4ull * (s->L.multi_boundary - s->L.local_boundary);  // offsets + starts
  });
}

}  // extern "C"
