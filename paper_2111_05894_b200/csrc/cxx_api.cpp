// cxx_api.cpp — the reference's scoring / reorder / tiering C++ API on the B200.
//
// Drop-in replacement for the reference translation units proj/src/scoring.cpp,
// proj/src/reorder.cpp and proj/src/tiering.cpp: every function declared in
// proj/include/tiergraph/{scoring,reorder,tiering}.hpp is defined here, with
// the same semantics and error messages, and does its work on the GPU through
// the C-ABI (include/tg_capi.h). This file includes only the per-subsystem
// header names, so it compiles against this repo's include/ (libtiergraph_b200_cxx.so)
// and, unchanged, against the reference's own headers (the drop-in build in
// oracle/Makefile, target `dropin`, which links the reference's unit and
// acceptance tests against it).
//
// Host-side work left here is what the reference itself does outside its
// loops: argument checks, O(1) scalar layout arithmetic, the train-id
// canonicalisation of TrainIdSet::from_ids, sequential_reorder_oracle (a
// documented single-threaded oracle) and the CSV writer.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <string>
#include <vector>

#include "cxx_common.hpp"
#include "tg_capi.h"
#include "tiergraph/reorder.hpp"
#include "tiergraph/scoring.hpp"
#include "tiergraph/tiering.hpp"

namespace tiergraph {

using b200::check;
using b200::Ctx;
using b200::nonnull;

namespace {

tg_layout to_c(const TierLayout& l) {
  return tg_layout{l.num_rows, l.local_boundary, l.multi_boundary,
                   l.num_devices, l.feature_dim, l.elem_bytes};
}

TierLayout from_c(const tg_layout& l) {
  TierLayout t;
  t.num_rows = l.num_rows;
  t.local_boundary = l.local_boundary;
  t.multi_boundary = l.multi_boundary;
  t.num_devices = l.num_devices;
  t.feature_dim = l.feature_dim;
  t.elem_bytes = l.elem_bytes;
  return t;
}

tg_report to_c(const TrafficReport& r) {
  return tg_report{r.local_accesses, r.peer_accesses, r.host_accesses,
                   r.local_bytes, r.peer_bytes, r.host_bytes};
}

void load(TrafficReport& r, const tg_report& c) {
  r.local_accesses = c.local_accesses;
  r.peer_accesses = c.peer_accesses;
  r.host_accesses = c.host_accesses;
  r.local_bytes = c.local_bytes;
  r.peer_bytes = c.peer_bytes;
  r.host_bytes = c.host_bytes;
}

// reorder.cpp:41-43 / :70-72 / :99-101 — every permuting call checks length
// before anything else.
void check_perm_length(const NodePermutation& perm, uint64_t n, const char* what = "num_nodes") {
  if (perm.size() != n)
    throw DomainError("permutation length " + std::to_string(perm.size()) + " != " + what + " " +
                      std::to_string(n));
}

}  // namespace

// ================================================================ scoring
// scoring.cpp:13-20 — canonicalise the labeled-node ids (host: a one-off
// O(|tid| log |tid|) input preparation, not part of any loop).
TrainIdSet TrainIdSet::from_ids(std::vector<NodeId> raw, NodeId num_nodes) {
  std::sort(raw.begin(), raw.end());
  raw.resize(static_cast<size_t>(std::unique(raw.begin(), raw.end()) - raw.begin()));
  if (!raw.empty() && raw.back() >= num_nodes)
    throw DomainError("train id " + std::to_string(raw.back()) + " out of range for num_nodes=" +
                      std::to_string(num_nodes));
  TrainIdSet t;
  t.ids = std::move(raw);
  return t;
}

// scoring.cpp:22-31 — the seeded Floyd subset, restated bit-exactly in
// csrc/host_producers.cpp.
TrainIdSet draw_random_train_ids(NodeId num_nodes, NodeId count, std::uint64_t seed) {
  TrainIdSet t;
  t.ids.resize(count ? count : 1);
  const int rc = tg_draw_random_train_ids(num_nodes, count, seed, t.ids.data());
  if (rc != TG_OK) throw DomainError(tg_host_last_error());
  t.ids.resize(count);
  return t;
}

// scoring.cpp:33-38
ScoreVector degree_score(const CsrGraph& g) {
  ScoreVector out(g.num_nodes());
  if (out.empty()) return out;
  b200::GraphLease dg(g);
  check(tg_degree_score(dg.ctx(), dg.graph(), out.data()));
  return out;
}

// scoring.cpp:78-102 on the device copy cached for g (K1 in-degrees with the
// upload, K2 init, K3 SpMV x iterations). With several TIERGRAPH_DEVICES the
// rows are partitioned over them (tg_mgraph), bit-identical to one device.
static ScoreVector run_pagerank(const CsrGraph& g, const PagerankConfig& cfg,
                                const TrainIdSet* tid) {
  ScoreVector out(g.num_nodes());
  if (out.empty() || (tid && tid->ids.empty())) {
    // the argument checks of scoring.cpp:42-47 / :89-91 (the library runs
    // them before touching a context or graph), then {} for an empty graph
    check(tid ? tg_weighted_reverse_pagerank(nullptr, nullptr, cfg.iterations, cfg.damp,
                                             nonnull(tid->ids), tid->ids.size(), nullptr)
              : tg_reverse_pagerank(nullptr, nullptr, cfg.iterations, cfg.damp, nullptr));
    return out;
  }
  b200::GraphLease dg(g);
  if (dg.devices() > 1) {
    check(tg_mgraph_pagerank(dg.partitioned(), cfg.iterations, cfg.damp,
                             tid ? nonnull(tid->ids) : nullptr, tid ? tid->ids.size() : 0,
                             tid ? 1 : 0, out.data()));
  } else if (tid) {
    check(tg_weighted_reverse_pagerank(dg.ctx(), dg.graph(), cfg.iterations, cfg.damp,
                                       nonnull(tid->ids), tid->ids.size(), out.data()));
  } else {
    check(tg_reverse_pagerank(dg.ctx(), dg.graph(), cfg.iterations, cfg.damp, out.data()));
  }
  return out;
}

// scoring.cpp:78-84
ScoreVector reverse_pagerank(const CsrGraph& g, const PagerankConfig& cfg) {
  return run_pagerank(g, cfg, nullptr);
}

// scoring.cpp:86-102
ScoreVector weighted_reverse_pagerank(const CsrGraph& g, const PagerankConfig& cfg,
                                      const TrainIdSet& tid) {
  return run_pagerank(g, cfg, &tid);
}

// scoring.cpp:104-115 (K4 key transform + K5 radix sort)
std::vector<NodeId> score_ordering(const ScoreVector& scores) {
  std::vector<NodeId> order(scores.size());
  if (scores.empty()) return order;
  Ctx ctx;
  check(tg_score_ordering(ctx, scores.data(), scores.size(), order.data()));
  return order;
}

// ================================================================ reorder
// reorder.cpp:10-21
void validate_permutation(const NodePermutation& perm) {
  if (perm.size() == 0) return;
  Ctx ctx;
  check(tg_validate_permutation(ctx, perm.new_id_of.data(), perm.size()));
}

// reorder.cpp:23-29 (K4 + K5 + K6 scatter)
NodePermutation permutation_from_scores(const ScoreVector& scores) {
  NodePermutation p;
  p.new_id_of.resize(scores.size());
  if (scores.empty()) return p;
  Ctx ctx;
  check(tg_permutation_from_scores(ctx, scores.data(), scores.size(), p.new_id_of.data(),
                                   nullptr));
  return p;
}

// reorder.cpp:31-37
NodePermutation invert(const NodePermutation& perm) {
  NodePermutation inv;
  inv.new_id_of.resize(perm.size());
  if (perm.size() == 0) return inv;
  Ctx ctx;
  check(tg_invert(ctx, perm.new_id_of.data(), perm.size(), inv.new_id_of.data()));
  return inv;
}

// reorder.cpp:39-66 (Algorithm 2: scatter lengths, scan, remapped copy)
CsrGraph reorder_graph(const CsrGraph& g, const NodePermutation& perm) {
  const uint64_t n = g.num_nodes(), e = g.num_edges();
  CsrGraph out;
  out.offsets.resize(n + 1);
  out.targets.resize(e);
  Ctx ctx;
  static const uint64_t kZeroOffset = 0;
  uint64_t scratch = 0;
  check(tg_reorder_graph(ctx, g.offsets.empty() ? &kZeroOffset : g.offsets.data(),
                         nonnull(g.targets), n, e, nonnull(perm.new_id_of), perm.size(),
                         out.offsets.data(), e ? out.targets.data() : &scratch));
  return out;
}

// reorder.cpp:68-95 — the API's single-threaded equivalence oracle for
// reorder_graph. It is sequential by contract (reorder.hpp:35-37), so it
// stays a plain host loop; the product path is reorder_graph above.
CsrGraph sequential_reorder_oracle(const CsrGraph& g, const NodePermutation& perm) {
  const NodeId n = g.num_nodes();
  check_perm_length(perm, n);
  validate_permutation(perm);
  std::vector<NodeId> old_of(n);
  for (NodeId u = 0; u < n; ++u) old_of[perm[u]] = u;
  CsrGraph out;
  out.offsets.assign(n + 1, 0);
  out.targets.reserve(g.num_edges());
  for (NodeId r = 0; r < n; ++r) {
    for (const NodeId v : g.row(old_of[r])) out.targets.push_back(perm[v]);
    out.offsets[r + 1] = out.targets.size();
  }
  return out;
}

// reorder.cpp:97-117 — new row perm[u] = old row u
FeatureMatrix reorder_features(const FeatureMatrix& f, const NodePermutation& perm) {
  const uint64_t want = f.num_rows * f.dim * f.elem_bytes;
  if (f.data.size() != want)  // validate_features, feature_matrix.cpp:9-14
    throw FormatError("features: data holds " + std::to_string(f.data.size()) +
                      " bytes, expected " + std::to_string(want));
  check_perm_length(perm, f.num_rows, "num_rows");
  FeatureMatrix out;
  out.num_rows = f.num_rows;
  out.dim = f.dim;
  out.elem_bytes = f.elem_bytes;
  out.data.resize(f.data.size());
  Ctx ctx;
  uint8_t scratch = 0;
  check(tg_reorder_features(ctx, f.data.empty() ? &scratch : f.data.data(), f.num_rows,
                            f.row_bytes(), nonnull(perm.new_id_of), perm.size(),
                            out.data.empty() ? &scratch : out.data.data()));
  return out;
}

// ================================================================ tiering
// tiering.cpp:10-18
void validate_layout(const TierLayout& layout) {
  const tg_layout l = to_c(layout);
  check(tg_validate_layout(&l));
}

// tiering.cpp:20-23
void validate_cost_model(const LinkCostModel& cost) {
  check(tg_validate_cost_model(cost.local_gbps, cost.peer_gbps, cost.host_gbps));
}

// tiering.cpp:25-29
double TrafficReport::hit_ratio() const {
  const tg_report r = to_c(*this);
  return tg_report_hit_ratio(&r);
}

// tiering.cpp:31-36
double TrafficReport::est_transfer_seconds(const LinkCostModel& cost) const {
  const tg_report r = to_c(*this);
  return tg_report_est_transfer_seconds(&r, cost.local_gbps, cost.peer_gbps, cost.host_gbps);
}

// tiering.cpp:38-46
TrafficReport& TrafficReport::operator+=(const TrafficReport& o) {
  local_accesses += o.local_accesses;
  peer_accesses += o.peer_accesses;
  host_accesses += o.host_accesses;
  local_bytes += o.local_bytes;
  peer_bytes += o.peer_bytes;
  host_bytes += o.host_bytes;
  return *this;
}

// tiering.cpp:48-65
Location resolve(const TierLayout& layout, std::uint64_t row_id, std::uint32_t requesting_device) {
  const tg_layout l = to_c(layout);
  tg_location c{};
  check(tg_resolve(&l, row_id, requesting_device, &c));
  Location loc;
  loc.tier = c.tier == TG_TIER_LOCAL_HOT     ? Tier::LocalHot
             : c.tier == TG_TIER_INTERLEAVED ? Tier::InterleavedDevice
                                             : Tier::ColdHost;
  loc.device = c.device;
  loc.row_within_tier = c.row_within_tier;
  return loc;
}

// tiering.cpp:67-98
TierLayout plan_layout(std::uint64_t num_rows, double hot_fraction, double replicated_fraction,
                       std::uint32_t num_devices, std::uint64_t feature_dim,
                       std::uint32_t elem_bytes, std::uint64_t per_device_budget_bytes) {
  tg_layout l{};
  check(tg_plan_layout(num_rows, hot_fraction, replicated_fraction, num_devices, feature_dim,
                       elem_bytes, per_device_budget_bytes, &l));
  return from_c(l);
}

// tiering.cpp:100-125 — accounting only, on the GPU (K8's counter path).
void gather(const TierLayout& layout, std::span<const std::uint64_t> row_ids,
            std::uint32_t requesting_device, TrafficReport& report) {
  if (row_ids.empty()) return;
  const tg_layout l = to_c(layout);
  tg_report r = to_c(report);
  Ctx ctx;
  const int rc = tg_gather_account(ctx, &l, row_ids.data(), row_ids.size(), requesting_device, &r);
  load(report, r);  // the prefix before a bad id stays accounted (reference loop semantics)
  check(rc);
}

// tiering.cpp:127-162
TrafficReport simulate_trace(const AccessCounter& counter, const TierLayout& layout) {
  validate_layout(layout);
  if (counter.counts.size() != layout.num_rows)
    throw DomainError("counter covers " + std::to_string(counter.counts.size()) +
                      " rows but the layout has " + std::to_string(layout.num_rows));
  if (counter.total == 0) throw DomainError("simulate_trace: counter total is zero");
  TrafficReport rep;
  if (layout.num_rows == 0) return rep;
  const tg_layout l = to_c(layout);
  tg_report r{};
  Ctx ctx;
  const int rc = tg_simulate_trace(ctx, counter.counts.data(), counter.counts.size(), &l, &r);
  // The reference trusts counter.total; the device sums the counts. An
  // all-zero counter whose total field is non-zero replays to an empty report.
  if (rc == TG_ERR_DOMAIN && std::strstr(tg_last_error(), "total is zero")) return rep;
  check(rc);
  load(rep, r);
  return rep;
}

// tiering.cpp:164-175
std::vector<std::uint64_t> counts_in_row_order(const AccessCounter& counter,
                                               std::span<const NodeId> ordering) {
  std::vector<std::uint64_t> out(ordering.size());
  if (ordering.size() != counter.counts.size())
    throw DomainError("ordering length != counter length");
  if (out.empty()) return out;
  Ctx ctx;
  check(tg_counts_in_row_order(ctx, counter.counts.data(), counter.counts.size(), ordering.data(),
                               ordering.size(), out.data()));
  return out;
}

// tiering.cpp:177-202 — one device replay pass for all fractions.
std::vector<SweepRow> hot_fraction_sweep(const AccessCounter& counter,
                                         std::span<const NodeId> ordering,
                                         std::span<const double> fractions,
                                         double replicated_fraction, std::uint32_t num_devices,
                                         std::uint64_t feature_dim, std::uint32_t elem_bytes,
                                         std::uint64_t per_device_budget_bytes) {
  for (size_t i = 1; i < fractions.size(); ++i)
    if (fractions[i] < fractions[i - 1])
      throw DomainError("sweep fractions must be sorted ascending");
  if (ordering.size() != counter.counts.size())
    throw DomainError("ordering length != counter length");
  const size_t nf = fractions.size();
  std::vector<tg_layout> lays(nf ? nf : 1);
  std::vector<tg_report> reps(nf ? nf : 1);
  std::vector<double> rep_frac(nf ? nf : 1);
  static const double kNoFraction = 0.0;
  Ctx ctx;
  check(tg_hot_fraction_sweep(ctx, nonnull(counter.counts), counter.counts.size(),
                              ordering.empty() ? nonnull(counter.counts) : ordering.data(),
                              nf ? fractions.data() : &kNoFraction, nf, replicated_fraction,
                              num_devices, feature_dim, elem_bytes, per_device_budget_bytes,
                              lays.data(), reps.data(), rep_frac.data()));
  std::vector<SweepRow> rows(nf);
  for (size_t i = 0; i < nf; ++i) {
    rows[i].hot_fraction = fractions[i];
    rows[i].replicated_fraction = rep_frac[i];
    rows[i].layout = from_c(lays[i]);
    load(rows[i].report, reps[i]);
  }
  return rows;
}

// tiering.cpp:204-231 — report CSV (host file I/O, same columns and format).
void write_report_csv(std::span<const SweepRow> rows, const LinkCostModel& cost,
                      const std::string& path) {
  std::ofstream f(path, std::ios::trunc);
  if (!f) throw IoError("cannot open for writing: " + path);
  f << std::setprecision(17);
  if (!rows.empty()) {
    const TierLayout& l = rows.front().layout;
    f << "# num_rows=" << l.num_rows << "\n# num_devices=" << l.num_devices
      << "\n# feature_dim=" << l.feature_dim << "\n# elem_bytes=" << l.elem_bytes
      << "\n# local_gbps=" << cost.local_gbps << "\n# peer_gbps=" << cost.peer_gbps
      << "\n# host_gbps=" << cost.host_gbps << '\n';
  }
  f << "hot_fraction,replicated_fraction,num_devices,total_accesses,local_accesses,"
       "peer_accesses,host_accesses,local_bytes,peer_bytes,host_bytes,hit_ratio,"
       "est_transfer_seconds\n";
  for (const SweepRow& s : rows) {
    const TrafficReport& r = s.report;
    const char c = ',';
    f << s.hot_fraction << c << s.replicated_fraction << c << s.layout.num_devices << c
      << r.total_accesses() << c << r.local_accesses << c << r.peer_accesses << c
      << r.host_accesses << c << r.local_bytes << c << r.peer_bytes << c << r.host_bytes << c
      << r.hit_ratio() << c << r.est_transfer_seconds(cost) << '\n';
  }
  f.flush();
  if (!f) throw IoError("write failed: " + path);
}

}  // namespace tiergraph
