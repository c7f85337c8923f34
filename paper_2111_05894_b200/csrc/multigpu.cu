// Partitioned reverse PageRank over several devices of one process
// (the reference's "bit-identical for any worker
// count" contract, parallel.hpp:5-7, read as "for any device count").
//
//   * Rows are split into contiguous EDGE-balanced blocks (tg_row_blocks):
//     on R-MAT, equal-row blocks put 3.4x the mean edge count on the first
//     rank, so the split follows `offsets`.
//   * Each device holds only its block of the CSR (tg_graph_create_rows):
//     1/G of the targets, not the whole graph.
//   * K1 is sharded: every device counts the in-degrees of its own edges, and
//     the partial counts are summed over the devices (peer copies into device
//     0, one add per device, peer copies back): the all-reduce of §8e, once
//     per graph.
//   * K3 step s on device r writes rows [rb_r, re_r) of norm_out; the block is
//     then pushed to every other device as ONE contiguous peer copy (copy
//     engines over NVLink/NVSwitch; a same-device copy for virtual devices),
//     and every device's next step waits on the events of all pushes. The
//     scattered 8 B remote stores of round 1's fused epilogue became G-1
//     contiguous bulk transfers per device per step.
// A row's sum is computed by exactly one device with the single-device
// kernels, so the scores are bit-identical to one device and to the
// reference for any G (scoring.cpp:50-74).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"
#include "pagerank_internal.cuh"

struct tg_mgraph {
  uint32_t G = 0;
  uint64_t n = 0, e = 0;
  tg_ctx* ctx[TG_MAX_DEVICES] = {};
  tg_graph* g[TG_MAX_DEVICES] = {};
  uint32_t* indeg[TG_MAX_DEVICES] = {};   // the SUMMED in-degrees, on every device
  cudaEvent_t ev[TG_MAX_DEVICES] = {};    // "device r's block of this step has been pushed"
  uint64_t bounds[TG_MAX_DEVICES + 1] = {};
  float indeg_ms = 0.0f;                  // sharded K1 + the reduction (device 0 clock)
};

namespace tgb {

__global__ void add_u32_kernel(uint32_t* __restrict__ acc, const uint32_t* __restrict__ x,
                               uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc[i] += x[i];
}

__global__ void widen_kernel(const uint32_t* __restrict__ in, uint64_t* __restrict__ out,
                             uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

// Edge-balanced contiguous blocks: bounds[r] = the first row whose offset
// reaches ceil(r * E / parts); with no edges, equal row counts.
void edge_balanced(const uint64_t* off, uint64_t n, uint32_t parts, uint64_t* bounds) {
  const uint64_t e = n ? off[n] : 0;
  bounds[0] = 0;
  for (uint32_t r = 1; r < parts; ++r) {
    if (e == 0) {
      bounds[r] = n * r / parts;
      continue;
    }
    const uint64_t want = (e * r + parts - 1) / parts;
    bounds[r] = static_cast<uint64_t>(std::lower_bound(off, off + n + 1, want) - off);
    bounds[r] = std::min(std::max(bounds[r], bounds[r - 1]), n);
  }
  bounds[parts] = n;
}

void push_block(tg_mgraph* m, uint32_t r, const double* src_r, double* const* dst, uint64_t rb,
                uint64_t re) {
  if (re <= rb) return;
  for (uint32_t q = 0; q < m->G; ++q) {
    if (q == r) continue;
    TGB_CUDA(cudaMemcpyPeerAsync(dst[q] + rb, m->ctx[q]->device, src_r + rb, m->ctx[r]->device,
                                 8 * (re - rb), m->ctx[r]->stream));
  }
}

// every device waits for every other device's pushes of this step
void exchange_barrier(tg_mgraph* m) {
  for (uint32_t r = 0; r < m->G; ++r) {
    DeviceGuard dg(m->ctx[r]->device);
    TGB_CUDA(cudaEventRecord(m->ev[r], m->ctx[r]->stream));
  }
  for (uint32_t q = 0; q < m->G; ++q)
    for (uint32_t r = 0; r < m->G; ++r)
      if (r != q) TGB_CUDA(cudaStreamWaitEvent(m->ctx[q]->stream, m->ev[r], 0));
}

}  // namespace tgb

using namespace tgb;

extern "C" {

int tg_row_blocks(const uint64_t* offsets, uint64_t n, uint32_t parts, uint64_t* bounds) {
  return guard([&] {
    if (parts < 1) domain_error("tg_row_blocks: parts must be >= 1");
    edge_balanced(offsets, n, parts, bounds);
  });
}

int tg_mgraph_destroy(tg_mgraph* m) {
  if (!m) return TG_OK;
  for (uint32_t r = 0; r < m->G; ++r) {
    if (!m->ctx[r]) continue;
    DeviceGuard dg(m->ctx[r]->device);
    cudaStreamSynchronize(m->ctx[r]->stream);
    tg_graph_destroy(m->g[r]);
    cudaFree(m->indeg[r]);
    if (m->ev[r]) cudaEventDestroy(m->ev[r]);
  }
  delete m;
  return TG_OK;
}

int tg_mgraph_create(tg_ctx* const* ctxs, uint32_t ndev, const uint64_t* offsets,
                     const uint64_t* targets, uint64_t n, uint64_t e, tg_mgraph** out) {
  return guard([&] {
    if (!ctxs || !out || !offsets) domain_error("tg_mgraph_create: null argument");
    if (ndev < 1 || ndev > TG_MAX_DEVICES)
      domain_error("tg_mgraph_create: 1.." + std::to_string(TG_MAX_DEVICES) + " devices");
    std::vector<uint64_t> hoff;
    const uint64_t* off = offsets;
    if (is_device_ptr(offsets)) {
      hoff.resize(n + 1);
      TGB_CUDA(cudaMemcpy(hoff.data(), offsets, 8 * (n + 1), cudaMemcpyDeviceToHost));
      off = hoff.data();
    }
    for (uint32_t a = 0; a < ndev; ++a)
      for (uint32_t b = a + 1; b < ndev; ++b)
        if (ctxs[a] == ctxs[b])
          domain_error("tg_mgraph_create: every device needs its own context (scratch)");
    auto* m = new tg_mgraph;
    m->G = ndev;
    m->n = n;
    m->e = e;
    try {
      edge_balanced(off, n, ndev, m->bounds);
      for (uint32_t r = 0; r < ndev; ++r) m->ctx[r] = ctxs[r];
      // peer access between distinct devices (copy engines over NVLink)
      for (uint32_t a = 0; a < ndev; ++a)
        for (uint32_t b = 0; b < ndev; ++b)
          if (ctxs[a]->device != ctxs[b]->device) {
            const int rc = tg_enable_peer_access(ctxs[a]->device, ctxs[b]->device);
            if (rc != TG_OK) throw Error(rc, tg_last_error());
          }
      for (uint32_t r = 0; r < ndev; ++r) {
        DeviceGuard dg(ctxs[r]->device);
        const int rc = tg_graph_create_rows(ctxs[r], offsets, targets, n, e, m->bounds[r],
                                            m->bounds[r + 1], &m->g[r]);
        if (rc != TG_OK) throw Error(rc, tg_last_error());
        TGB_CUDA(tgb::dev_malloc(&m->indeg[r], 4 * std::max<uint64_t>(n, 1)));
        TGB_CUDA(cudaEventCreateWithFlags(&m->ev[r], cudaEventDisableTiming));
      }
      // K1 all-reduce: partial counts -> device 0 (sum) -> every device
      if (n) {
        tg_ctx* c0 = ctxs[0];
        DeviceGuard dg(c0->device);
        cudaEvent_t t0, t1;
        TGB_CUDA(cudaEventCreate(&t0));
        TGB_CUDA(cudaEventCreate(&t1));
        TGB_CUDA(cudaEventRecord(t0, c0->stream));
        TGB_CUDA(cudaMemcpyAsync(m->indeg[0], m->g[0]->indeg, 4 * n, cudaMemcpyDeviceToDevice,
                                 c0->stream));
        uint32_t* tmp = c0->scratch_t<uint32_t>(kScratchA, n);
        for (uint32_t r = 1; r < ndev; ++r) {
          TGB_CUDA(cudaMemcpyPeerAsync(tmp, c0->device, m->g[r]->indeg, ctxs[r]->device, 4 * n,
                                       c0->stream));
          add_u32_kernel<<<grid_for(n, 256), 256, 0, c0->stream>>>(m->indeg[0], tmp, n);
          TGB_LAUNCHED();
        }
        for (uint32_t r = 1; r < ndev; ++r)
          TGB_CUDA(cudaMemcpyPeerAsync(m->indeg[r], ctxs[r]->device, m->indeg[0], c0->device,
                                       4 * n, c0->stream));
        TGB_CUDA(cudaEventRecord(t1, c0->stream));
        TGB_CUDA(cudaEventSynchronize(t1));
        TGB_CUDA(cudaEventElapsedTime(&m->indeg_ms, t0, t1));
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
      }
    } catch (...) {
      tg_mgraph_destroy(m);
      throw;
    }
    *out = m;
  });
}

int tg_mgraph_info(const tg_mgraph* m, uint64_t* bounds, uint64_t* edges, double* indeg_ms) {
  return guard([&] {
    for (uint32_t r = 0; r < m->G; ++r) {
      if (bounds) bounds[r] = m->bounds[r];
      if (edges) edges[r] = m->g[r]->e;
    }
    if (bounds) bounds[m->G] = m->bounds[m->G];
    if (indeg_ms) *indeg_ms = m->indeg_ms;
  });
}

int tg_mgraph_in_degrees(tg_mgraph* m, uint64_t* out) {
  return guard([&] {
    if (!m->n) return;
    tg_ctx* c0 = m->ctx[0];
    DeviceGuard dg(c0->device);
    DevOut<uint64_t> o(c0, out, m->n, kStageOut0);
    widen_kernel<<<grid_for(m->n, 256), 256, 0, c0->stream>>>(m->indeg[0], o.dev(), m->n);
    TGB_LAUNCHED();
    o.finish();
  });
}

int tg_mgraph_pagerank(tg_mgraph* m, uint32_t iterations, double damp, const uint64_t* tid,
                       uint64_t ntid, int weighted, double* out) {
  return guard([&] {
    check_config(iterations, damp);
    if (weighted && ntid == 0)
      domain_error(
          "weighted reverse pagerank needs a non-empty train id set; "
          "use reverse_pagerank when no nodes are labeled");  // scoring.cpp:89-91
    const uint64_t n = m->n;
    if (n == 0) return;
    const uint32_t G = m->G;
    double *na[TG_MAX_DEVICES], *nb[TG_MAX_DEVICES], *sc[TG_MAX_DEVICES];
    for (uint32_t r = 0; r < G; ++r) {
      tg_ctx* c = m->ctx[r];
      DeviceGuard dg(c->device);
      na[r] = c->scratch_t<double>(kScratchB, n);
      nb[r] = c->scratch_t<double>(kScratchC, n);
      sc[r] = c->scratch_t<double>(kScratchD, n);
      const uint64_t* td = weighted ? dev_in(c, tid, ntid, kStageIn0) : nullptr;
      const int rc = tg_pagerank_init_async(c, n, td, weighted ? ntid : 0, m->indeg[r], na[r]);
      if (rc != TG_OK) throw Error(rc, tg_last_error());
    }
    // init ran on every device before any push lands in its vectors
    exchange_barrier(m);
    for (uint32_t it = 0; it < iterations; ++it) {
      const int last = it + 1 == iterations ? 1 : 0;
      for (uint32_t r = 0; r < G; ++r) {
        DeviceGuard dg(m->ctx[r]->device);
        pagerank_step(m->ctx[r], m->g[r], m->indeg[r], damp, na[r], nb[r], sc[r], m->bounds[r],
                      m->bounds[r + 1], last);
        push_block(m, r, last ? sc[r] : nb[r], last ? sc : nb, m->bounds[r], m->bounds[r + 1]);
      }
      exchange_barrier(m);
      std::swap(na, nb);
    }
    tg_ctx* c0 = m->ctx[0];
    DeviceGuard dg(c0->device);
    DevOut<double> o(c0, out, n, kStageOut0);
    TGB_CUDA(cudaMemcpyAsync(o.dev(), sc[0], 8 * n, cudaMemcpyDeviceToDevice, c0->stream));
    o.finish();
    for (uint32_t r = 1; r < G; ++r) m->ctx[r]->sync();
  });
}

}  // extern "C"
