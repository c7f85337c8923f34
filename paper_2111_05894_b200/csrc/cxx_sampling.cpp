// cxx_sampling.cpp — the reference's sampling API (proj/include/tiergraph/
// sampling.hpp) with build_minibatch and run_training_trace on the GPU.
//
// Drop-in replacement for the reference translation unit proj/src/
// sampling.cpp: the minibatch expansion and the
// access-counter trace run in csrc/sampling.cu through the C-ABI and are
// bit-identical to the reference. The one-node helper sample_in_neighbors
// (it advances a caller-owned host RngStream) and the O(n) analysis
// cumulative_access_curve stay host code, as does argument validation.
// Compiles against this repo's include/ and, unchanged, against the
// reference's headers (oracle/Makefile target dropin).
#include <algorithm>
#include <string>
#include <vector>

#include "cxx_common.hpp"
#include "tg_capi.h"
#include "tiergraph/sampling.hpp"

namespace tiergraph {

namespace {

constexpr std::uint64_t kSampleTag = 0x534Dull;  // sampling.cpp:15 (stream domain)

// The GPU sampler state lives in the device-graph cache (cxx_common.hpp
// GraphLease): consecutive build_minibatch calls on the same graph reuse the
// upload, the stamps and the member bitmap.

}  // namespace

// sampling.cpp:18-25
void validate_fanouts(const FanoutSpec& spec) {
  if (spec.fanouts.empty()) throw DomainError("fanouts must be non-empty");
  if (spec.fanouts.size() > 5)
    throw DomainError("fanout depth " + std::to_string(spec.fanouts.size()) +
                      " exceeds the supported maximum of 5");
  for (const std::uint32_t f : spec.fanouts)
    if (f == 0) throw DomainError("every fanout must be >= 1");
}

// sampling.cpp:27-33
AccessCounter make_access_counter(std::vector<std::uint64_t> counts) {
  AccessCounter c;
  for (const std::uint64_t v : counts) c.total += v;
  c.counts = std::move(counts);
  return c;
}

// sampling.cpp:35-37
RngStream BatchRng::stream(std::uint32_t layer, NodeId node) const {
  return RngStream(derive_stream_key(rng_seed, {kSampleTag, epoch, batch_index, layer, node}));
}

// sampling.cpp:39-54 — one node, host (the stream object is the caller's).
std::vector<NodeId> sample_in_neighbors(const CsrGraph& gt, NodeId node, std::uint32_t fanout,
                                        RngStream& rng) {
  if (node >= gt.num_nodes()) throw DomainError("node " + std::to_string(node) + " out of range");
  const auto nbrs = gt.row(node);
  if (nbrs.size() <= fanout) return std::vector<NodeId>(nbrs.begin(), nbrs.end());
  std::vector<std::uint64_t> idx;
  sample_index_subset(rng, nbrs.size(), fanout, idx);
  std::vector<NodeId> out;
  out.reserve(idx.size());
  for (const std::uint64_t i : idx) out.push_back(nbrs[i]);
  return out;
}

// sampling.cpp:56-90 on the GPU (K-sampler, csrc/sampling.cu).
std::vector<NodeId> build_minibatch(const CsrGraph& gt, std::span<const NodeId> seeds,
                                    const FanoutSpec& fanouts, const BatchRng& rng,
                                    std::vector<NodeId>* raw_draws) {
  validate_fanouts(fanouts);
  if (seeds.empty()) throw DomainError("build_minibatch: seeds must be non-empty");
  for (const NodeId s : seeds)
    if (s >= gt.num_nodes()) throw DomainError("seed " + std::to_string(s) + " out of range");
  b200::GraphLease dg(gt);
  tg_sampler* smp = dg.sampler();
  const uint64_t n = gt.num_nodes();
  const auto& f = fanouts.fanouts;
  // layered bounds: frontier_{l+1} <= min(n, frontier_l * k_l); members <=
  // min(n, sum of frontiers); raw draws <= |seeds| + sum frontier_l * k_l
  uint64_t fr = std::min<uint64_t>(seeds.size(), n), mem = fr, raw_cap = seeds.size();
  for (const std::uint32_t k : f) {
    raw_cap += fr * k;
    fr = std::min<uint64_t>(n, fr * k);
    mem += fr;
  }
  mem = std::min<uint64_t>(mem, n);
  std::vector<NodeId> members(mem);
  uint64_t count = 0;
  if (!raw_draws) {
    b200::check(tg_sample_minibatch(smp, seeds.data(), seeds.size(), f.data(),
                                    static_cast<uint32_t>(f.size()), rng.rng_seed, rng.epoch,
                                    rng.batch_index, members.data(), mem, &count));
  } else {
    const uint64_t cap = raw_cap;
    std::vector<NodeId> raw(cap);
    uint64_t raw_n = 0;
    b200::check(tg_sample_minibatch_raw(smp, seeds.data(), seeds.size(), f.data(),
                                        static_cast<uint32_t>(f.size()), rng.rng_seed, rng.epoch,
                                        rng.batch_index, members.data(), mem, &count, raw.data(),
                                        cap, &raw_n));
    raw_draws->insert(raw_draws->end(), raw.begin(), raw.begin() + static_cast<long>(raw_n));
  }
  members.resize(count);
  return members;
}

// sampling.cpp:92-140 on the GPU.
AccessCounter run_training_trace(const CsrGraph& g, const TrainIdSet& tid,
                                 const FanoutSpec& fanouts, const TraceConfig& cfg) {
  validate_fanouts(fanouts);
  if (tid.ids.empty()) throw DomainError("run_training_trace: train id set is empty");
  if (cfg.batch_size < 1) throw DomainError("batch_size must be >= 1");
  if (cfg.epochs < 1) throw DomainError("epochs must be >= 1");
  const NodeId n = g.num_nodes();
  for (const NodeId id : tid.ids)
    if (id >= n) throw DomainError("train id " + std::to_string(id) + " out of range");
  // the sampler runs on transpose(g), built on the device (tg_transpose)
  // and cached with g's entry
  b200::GraphLease dg(g);
  b200::CachedGraph* e = dg.entry();
  if (!e->sampler_t) {
    tg_ctx* ctx = dg.ctx();
    const uint64_t m = g.targets.size();
    void *toff = nullptr, *ttgt = nullptr;
    b200::check(tg_device_alloc(ctx, 8 * (n + 1), &toff));
    const int rc0 = tg_device_alloc(ctx, 8 * std::max<uint64_t>(m, 1), &ttgt);
    int rc = rc0;
    static const uint64_t kNone = 0;
    if (rc == TG_OK)
      rc = tg_transpose(ctx, g.offsets.data(), m ? g.targets.data() : &kNone, n, m,
                        static_cast<uint64_t*>(toff), static_cast<uint64_t*>(ttgt));
    if (rc == TG_OK)
      rc = tg_graph_create(ctx, static_cast<uint64_t*>(toff), static_cast<uint64_t*>(ttgt), n, m,
                           &e->gt);
    if (rc == TG_OK) rc = tg_sampler_create(ctx, e->gt, &e->sampler_t);
    tg_ctx_sync(ctx);
    tg_device_free(ctx, toff);
    if (ttgt) tg_device_free(ctx, ttgt);
    b200::check(rc);
  }
  std::vector<std::uint64_t> counts(n);
  const auto& f = fanouts.fanouts;
  b200::check(tg_sampler_trace(e->sampler_t, tid.ids.data(), tid.ids.size(), f.data(),
                               static_cast<uint32_t>(f.size()), cfg.batch_size, cfg.epochs,
                               cfg.rng_seed, cfg.dedup_per_batch ? 1 : 0, counts.data()));
  return make_access_counter(std::move(counts));
}

// sampling.cpp:142-165 — host analysis over the counter.
std::vector<double> cumulative_access_curve(const AccessCounter& counter,
                                            std::span<const NodeId> ordering) {
  const NodeId n = counter.counts.size();
  if (counter.total == 0) throw DomainError("cumulative_access_curve: counter total is zero");
  if (ordering.size() != n)
    throw DomainError("ordering length " + std::to_string(ordering.size()) + " != num_nodes " +
                      std::to_string(n));
  std::vector<char> hit(n, 0);
  for (const NodeId u : ordering) {
    if (u >= n || hit[u]) throw DomainError("ordering is not a permutation of node ids");
    hit[u] = 1;
  }
  std::vector<double> curve(n);
  const double total = static_cast<double>(counter.total);
  std::uint64_t covered = 0;
  for (NodeId k = 0; k < n; ++k) {
    covered += counter.counts[ordering[k]];
    curve[k] = static_cast<double>(covered) / total;
  }
  return curve;
}

}  // namespace tiergraph
