// Graph-structure tiering: the sampler's graph placed
// by the same TierLayout as the feature rows. Shared by structure.cu
// (placement) and sampling.cu (the sampler reads neighbour lists through it).
//
// "we expand the idea of multi-GPU node feature data
// placement strategy to the graph structure as well and distribute the graph
// structure over multiple GPUs"; the reference only estimates it
// (tools/tiergraph_cli.cpp:389-406, --structure-of: one pseudo-row per node
// fed to hot_fraction_sweep). Here row v of the TRANSPOSED, score-reordered
// graph (v's in-neighbours, new ids) lives where resolve() puts row v
// (tiering.cpp:48-65):
//   [0, lb)   replicated: every device holds these rows' neighbour ids;
//   [lb, mb)  interleaved: device (v-lb) % D holds them, in slot order;
//   [mb, N)   cold: pinned, mapped host memory, read by UVA zero-copy loads.
// The offsets (N+1 u32) are on every device: a node's degree decides how
// many of its neighbour ids are read (all, or `fanout` Floyd picks), and they
// are 4 B per node against the lists' 4 B per edge.
#pragma once
#include <cstdint>

#include "internal.cuh"

namespace tgb {

// What a sampler kernel needs to find row v's neighbour ids. An untiered
// graph is the view with lb = mb = N (every row "replicated", rep = targets).
struct SGraphView {
  const uint32_t* off = nullptr;        // N+1 (device)
  const uint32_t* rep = nullptr;        // rows [0, lb): index off[v]
  const uint32_t* ilv[TG_MAX_DEVICES] = {};  // device d's interleaved slice (local or peer)
  const uint32_t* ilv_start = nullptr;  // mb-lb: row's start within its device's slice
  const uint32_t* cold = nullptr;       // rows [mb, N): index off[v] - cold_base (UVA)
  uint64_t cold_base = 0;
  uint32_t lb = 0, mb = 0, n = 0, D = 1, self = 0;
  // neighbour ids read per tier (0 local, 1 peer, 2 host), or null
  unsigned long long* reads = nullptr;

  // Row v's first neighbour id and its tier (0 local, 1 peer, 2 host).
  __device__ __forceinline__ const uint32_t* row(uint32_t v, uint32_t b, int* tier) const {
    if (v < lb) {
      *tier = 0;
      return rep + b;
    }
    if (v < mb) {
      const uint32_t o = v - lb;
      const uint32_t d = D == 1 ? 0u : o % D;
      *tier = d == self ? 0 : 1;
      return ilv[d] + ilv_start[o];
    }
    *tier = 2;
    return cold + (b - cold_base);
  }
};

}  // namespace tgb

struct tg_sgraph {
  tg_ctx* ctx = nullptr;
  tg_layout L{};
  uint32_t dev = 0;
  uint64_t n = 0, e = 0;
  uint32_t* off = nullptr;        // device, n+1
  uint32_t* rep = nullptr;        // device, off[lb] entries
  uint32_t* slice = nullptr;      // device, this device's interleaved rows
  uint64_t slice_len = 0;
  uint32_t* ilv_start = nullptr;  // device, mb-lb
  uint32_t* cold_host = nullptr;  // pinned mapped host (owned unless attached)
  const uint32_t* cold_dev = nullptr;
  uint64_t cold_len = 0;          // E - off[mb]
  bool own_cold = false, cold_attached = false, cold_fill = true;
  const uint32_t* peer[TG_MAX_DEVICES] = {};
  bool placed = false;

  tgb::SGraphView view() const;
};
