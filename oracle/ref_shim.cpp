// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp), compiled out-of-tree by oracle/Makefile
// with -Dtiergraph=tiergraph_ref so it can share a process with the B200
// library. Only tests/, __graft_entry__.smoke() and bench.py's CPU legs load
// the resulting oracle/_ref/libtgref.so, and only as the checker / CPU
// baseline. Every entry point forwards to the reference function named in its
// comment; nothing here re-implements reference arithmetic.
//
// Error convention mirrors the reference CLI (tools/tiergraph_cli.cpp:589-601):
// 0 ok, 2 DomainError, 3 FormatError, 4 IoError, 5 anything else.

#include <omp.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "tiergraph/csr_graph.hpp"
#include "tiergraph/feature_matrix.hpp"
#include "tiergraph/io.hpp"
#include "tiergraph/parallel.hpp"
#include "tiergraph/reorder.hpp"
#include "tiergraph/rng.hpp"
#include "tiergraph/sampling.hpp"
#include "tiergraph/scoring.hpp"
#include "tiergraph/tiering.hpp"
#include "tiergraph/types.hpp"

namespace tg = tiergraph;  // expands to tiergraph_ref under -Dtiergraph=tiergraph_ref

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const tg::DomainError& e) {
    g_err = e.what();
    return 2;
  } catch (const tg::FormatError& e) {
    g_err = e.what();
    return 3;
  } catch (const tg::IoError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

tg::CsrGraph make_graph(const uint64_t* offsets, const uint64_t* targets, uint64_t n,
                        uint64_t e) {
  tg::CsrGraph g;
  g.offsets.assign(offsets, offsets + n + 1);
  g.targets.assign(targets, targets + e);
  return g;
}

tg::TierLayout make_layout(const uint64_t* l) {
  // l = {num_rows, local_boundary, multi_boundary, num_devices, feature_dim, elem_bytes}
  tg::TierLayout t;
  t.num_rows = l[0];
  t.local_boundary = l[1];
  t.multi_boundary = l[2];
  t.num_devices = static_cast<uint32_t>(l[3]);
  t.feature_dim = l[4];
  t.elem_bytes = static_cast<uint32_t>(l[5]);
  return t;
}

void put_report(const tg::TrafficReport& r, uint64_t* out) {
  out[0] = r.local_accesses;
  out[1] = r.peer_accesses;
  out[2] = r.host_accesses;
  out[3] = r.local_bytes;
  out[4] = r.peer_bytes;
  out[5] = r.host_bytes;
}

tg::TrafficReport get_report(const uint64_t* in) {
  tg::TrafficReport r;
  r.local_accesses = in[0];
  r.peer_accesses = in[1];
  r.host_accesses = in[2];
  r.local_bytes = in[3];
  r.peer_bytes = in[4];
  r.host_bytes = in[5];
  return r;
}

uint64_t* dup_vec(const std::vector<uint64_t>& v) {
  auto* p = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (v.size() ? v.size() : 1)));
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(uint64_t) * v.size());
  return p;
}

struct RefGraph {
  tg::CsrGraph g;
};
struct RefFeatures {
  tg::FeatureMatrix f;
};
}  // namespace

extern "C" {

const char* tgref_last_error() { return g_err.c_str(); }
void tgref_free(void* p) { std::free(p); }

// parallel.hpp:8-9
void tgref_set_worker_count(int n) { tg::set_worker_count(n); }
int tgref_worker_count() { return tg::worker_count(); }

// ---- graph handles (construction copies; it is not part of any timed call)
void* tgref_graph_create(const uint64_t* offsets, const uint64_t* targets, uint64_t n,
                         uint64_t e) {
  auto* h = new RefGraph;
  h->g = make_graph(offsets, targets, n, e);
  return h;
}
void tgref_graph_destroy(void* h) { delete static_cast<RefGraph*>(h); }
uint64_t tgref_graph_num_edges(void* h) { return static_cast<RefGraph*>(h)->g.num_edges(); }
uint64_t tgref_graph_num_nodes(void* h) { return static_cast<RefGraph*>(h)->g.num_nodes(); }
void tgref_graph_export(void* h, uint64_t* offsets, uint64_t* targets) {
  const auto& g = static_cast<RefGraph*>(h)->g;
  std::memcpy(offsets, g.offsets.data(), sizeof(uint64_t) * g.offsets.size());
  if (!g.targets.empty())
    std::memcpy(targets, g.targets.data(), sizeof(uint64_t) * g.targets.size());
}

// csr_graph.cpp:36-65 from_edge_list
int tgref_from_edge_list(uint64_t n, const uint64_t* src, const uint64_t* dst, uint64_t m,
                         void** out_graph) {
  return guard([&] {
    tg::EdgeList el;
    el.num_nodes = n;
    el.pairs.resize(m);
    for (uint64_t i = 0; i < m; ++i) el.pairs[i] = {src[i], dst[i]};
    auto* h = new RefGraph;
    h->g = tg::from_edge_list(el);
    *out_graph = h;
  });
}

// csr_graph.cpp:95-132 generate_power_law
int tgref_generate_power_law(uint64_t n, uint64_t m, uint64_t seed, void** out_graph) {
  return guard([&] {
    auto* h = new RefGraph;
    h->g = tg::generate_power_law(n, m, seed);
    *out_graph = h;
  });
}

// csr_graph.cpp:67-80 transpose
void* tgref_graph_transpose(void* h) {
  auto* t = new RefGraph;
  t->g = tg::transpose(static_cast<RefGraph*>(h)->g);
  return t;
}

// csr_graph.cpp:10-34 validate_csr
int tgref_validate_csr(void* h, int require_sorted) {
  return guard([&] { tg::validate_csr(static_cast<RefGraph*>(h)->g, require_sorted != 0); });
}

// csr_graph.cpp:89-93 in_degrees
void tgref_in_degrees(void* h, uint64_t* out) {
  const auto d = tg::in_degrees(static_cast<RefGraph*>(h)->g);
  if (!d.empty()) std::memcpy(out, d.data(), sizeof(uint64_t) * d.size());
}

// scoring.cpp:13-20 TrainIdSet::from_ids ; returns malloc'ed sorted unique ids
int tgref_train_ids_from(const uint64_t* raw, uint64_t m, uint64_t num_nodes, uint64_t** out,
                         uint64_t* out_n) {
  return guard([&] {
    const auto t = tg::TrainIdSet::from_ids(std::vector<uint64_t>(raw, raw + m), num_nodes);
    *out = dup_vec(t.ids);
    *out_n = t.ids.size();
  });
}

// scoring.cpp:22-31 draw_random_train_ids ; out has `count` entries
int tgref_draw_random_train_ids(uint64_t num_nodes, uint64_t count, uint64_t seed,
                                uint64_t* out) {
  return guard([&] {
    const auto t = tg::draw_random_train_ids(num_nodes, count, seed);
    std::memcpy(out, t.ids.data(), sizeof(uint64_t) * t.ids.size());
  });
}

// scoring.cpp:33-38 degree_score
void tgref_degree_score(void* h, double* out) {
  const auto s = tg::degree_score(static_cast<RefGraph*>(h)->g);
  if (!s.empty()) std::memcpy(out, s.data(), sizeof(double) * s.size());
}

// scoring.cpp:78-84 reverse_pagerank
int tgref_reverse_pagerank(void* h, uint32_t iterations, double damp, double* out) {
  return guard([&] {
    const auto s = tg::reverse_pagerank(static_cast<RefGraph*>(h)->g, {iterations, damp});
    if (!s.empty()) std::memcpy(out, s.data(), sizeof(double) * s.size());
  });
}

// scoring.cpp:86-102 weighted_reverse_pagerank ; tid must already be sorted-unique
// (the caller's TrainIdSet), exactly like the reference signature.
int tgref_weighted_reverse_pagerank(void* h, uint32_t iterations, double damp,
                                    const uint64_t* tid, uint64_t ntid, double* out) {
  return guard([&] {
    tg::TrainIdSet t;
    t.ids.assign(tid, tid + ntid);
    const auto s =
        tg::weighted_reverse_pagerank(static_cast<RefGraph*>(h)->g, {iterations, damp}, t);
    if (!s.empty()) std::memcpy(out, s.data(), sizeof(double) * s.size());
  });
}

// scoring.cpp:104-115 score_ordering
int tgref_score_ordering(const double* scores, uint64_t n, uint64_t* out) {
  return guard([&] {
    const auto o = tg::score_ordering(std::vector<double>(scores, scores + n));
    if (!o.empty()) std::memcpy(out, o.data(), sizeof(uint64_t) * n);
  });
}

// reorder.cpp:23-29 permutation_from_scores
int tgref_permutation_from_scores(const double* scores, uint64_t n, uint64_t* out) {
  return guard([&] {
    const auto p = tg::permutation_from_scores(std::vector<double>(scores, scores + n));
    if (n) std::memcpy(out, p.new_id_of.data(), sizeof(uint64_t) * n);
  });
}

// reorder.cpp:10-21 validate_permutation
int tgref_validate_permutation(const uint64_t* perm, uint64_t n) {
  return guard([&] {
    tg::NodePermutation p;
    p.new_id_of.assign(perm, perm + n);
    tg::validate_permutation(p);
  });
}

// reorder.cpp:31-37 invert
int tgref_invert(const uint64_t* perm, uint64_t n, uint64_t* out) {
  return guard([&] {
    tg::NodePermutation p;
    p.new_id_of.assign(perm, perm + n);
    const auto q = tg::invert(p);
    if (n) std::memcpy(out, q.new_id_of.data(), sizeof(uint64_t) * n);
  });
}

// reorder.cpp:39-66 reorder_graph ; returns a new graph handle
int tgref_reorder_graph(void* h, const uint64_t* perm, uint64_t n, void** out_graph) {
  return guard([&] {
    tg::NodePermutation p;
    p.new_id_of.assign(perm, perm + n);
    auto* r = new RefGraph;
    try {
      r->g = tg::reorder_graph(static_cast<RefGraph*>(h)->g, p);
    } catch (...) {
      delete r;
      throw;
    }
    *out_graph = r;
  });
}

// reorder.cpp:68-95 sequential_reorder_oracle
int tgref_sequential_reorder_oracle(void* h, const uint64_t* perm, uint64_t n,
                                    void** out_graph) {
  return guard([&] {
    tg::NodePermutation p;
    p.new_id_of.assign(perm, perm + n);
    auto* r = new RefGraph;
    try {
      r->g = tg::sequential_reorder_oracle(static_cast<RefGraph*>(h)->g, p);
    } catch (...) {
      delete r;
      throw;
    }
    *out_graph = r;
  });
}

// ---- feature matrices
void* tgref_features_create(const uint8_t* data, uint64_t rows, uint64_t dim,
                            uint32_t elem_bytes) {
  auto* h = new RefFeatures;
  h->f.num_rows = rows;
  h->f.dim = dim;
  h->f.elem_bytes = elem_bytes;
  h->f.data.assign(data, data + rows * dim * elem_bytes);
  return h;
}
// feature_matrix.cpp:16-28 make_test_features
void* tgref_make_test_features(uint64_t rows, uint64_t dim) {
  auto* h = new RefFeatures;
  h->f = tg::make_test_features(rows, dim);
  return h;
}
void tgref_features_destroy(void* h) { delete static_cast<RefFeatures*>(h); }
const uint8_t* tgref_features_data(void* h) { return static_cast<RefFeatures*>(h)->f.data.data(); }
uint64_t tgref_features_nbytes(void* h) { return static_cast<RefFeatures*>(h)->f.data.size(); }

// reorder.cpp:97-117 reorder_features ; returns a new feature handle
int tgref_reorder_features(void* h, const uint64_t* perm, uint64_t n, void** out) {
  return guard([&] {
    tg::NodePermutation p;
    p.new_id_of.assign(perm, perm + n);
    auto* r = new RefFeatures;
    try {
      r->f = tg::reorder_features(static_cast<RefFeatures*>(h)->f, p);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  });
}

// CPU byte gather baseline: FeatureMatrix::row(id) (feature_matrix.hpp:22-24)
// copied into a contiguous buffer with the reorder_features memcpy pattern
// (reorder.cpp:113-115), plus the reference's own accounting gather()
// (tiering.cpp:100-125). The reference moves no bytes itself; this is the
// CPU path a reference user would write, timed as the CPU baseline.
int tgref_features_gather(void* h, const uint64_t* layout6, const uint64_t* ids, uint64_t n,
                          uint32_t requesting_device, uint8_t* out, uint64_t* report6) {
  return guard([&] {
    const auto& f = static_cast<RefFeatures*>(h)->f;
    const uint64_t rb = f.row_bytes();
    const auto layout = make_layout(layout6);
    tg::TrafficReport rep = get_report(report6);
    tg::gather(layout, std::span<const uint64_t>(ids, n), requesting_device, rep);
    const int workers = tg::worker_count();
#pragma omp parallel for schedule(static) num_threads(workers)
    for (int64_t i = 0; i < static_cast<int64_t>(n); ++i)
      std::memcpy(out + static_cast<uint64_t>(i) * rb, f.row(ids[i]).data(), rb);
    put_report(rep, report6);
  });
}

// The same CPU byte gather from the ORIGINAL (un-reordered) matrix held by the
// caller: new row `id` of reorder_features(f, perm) is old row inv[id]
// (reorder.cpp:113-115 writes old row u to new row perm[u]), so this copies
// FeatureMatrix::row(inv[id]) (feature_matrix.hpp:22-24: data + id*row_bytes)
// -- byte-identical to gathering from the reordered copy without a second
// N x R matrix (used where two copies do not fit in host RAM).
int tgref_features_gather_inv(const uint8_t* data, uint64_t rows, uint64_t row_bytes,
                              const uint64_t* inv, const uint64_t* layout6, const uint64_t* ids,
                              uint64_t n, uint32_t requesting_device, uint8_t* out,
                              uint64_t* report6) {
  return guard([&] {
    const auto layout = make_layout(layout6);
    tg::TrafficReport rep = get_report(report6);
    tg::gather(layout, std::span<const uint64_t>(ids, n), requesting_device, rep);
    const int workers = tg::worker_count();
#pragma omp parallel for schedule(static) num_threads(workers)
    for (int64_t i = 0; i < static_cast<int64_t>(n); ++i) {
      const uint64_t old = inv[ids[i]];
      if (old < rows) std::memcpy(out + static_cast<uint64_t>(i) * row_bytes,
                                  data + old * row_bytes, row_bytes);
    }
    put_report(rep, report6);
  });
}

// ---- tiering (tiering.cpp)
int tgref_validate_layout(const uint64_t* layout6) {
  return guard([&] { tg::validate_layout(make_layout(layout6)); });
}

int tgref_validate_cost_model(double local_gbps, double peer_gbps, double host_gbps) {
  return guard([&] { tg::validate_cost_model({local_gbps, peer_gbps, host_gbps}); });
}

// tiering.cpp:48-65 resolve ; out3 = {tier, device, row_within_tier}
int tgref_resolve(const uint64_t* layout6, uint64_t row, uint32_t dev, uint64_t* out3) {
  return guard([&] {
    const auto loc = tg::resolve(make_layout(layout6), row, dev);
    out3[0] = static_cast<uint64_t>(loc.tier);
    out3[1] = loc.device;
    out3[2] = loc.row_within_tier;
  });
}

// tiering.cpp:67-98 plan_layout ; out6 = layout
int tgref_plan_layout(uint64_t num_rows, double hot, double rep, uint32_t devices,
                      uint64_t dim, uint32_t elem_bytes, uint64_t budget, uint64_t* out6) {
  return guard([&] {
    const auto l = tg::plan_layout(num_rows, hot, rep, devices, dim, elem_bytes, budget);
    out6[0] = l.num_rows;
    out6[1] = l.local_boundary;
    out6[2] = l.multi_boundary;
    out6[3] = l.num_devices;
    out6[4] = l.feature_dim;
    out6[5] = l.elem_bytes;
  });
}

// tiering.cpp:100-125 gather (accounting only) ; report6 is accumulated into
int tgref_gather(const uint64_t* layout6, const uint64_t* ids, uint64_t n, uint32_t dev,
                 uint64_t* report6) {
  tg::TrafficReport rep = get_report(report6);
  const int rc = guard([&] {
    tg::gather(make_layout(layout6), std::span<const uint64_t>(ids, n), dev, rep);
  });
  put_report(rep, report6);  // partial accounting survives an exception, as in the reference
  return rc;
}

// tiering.cpp:127-162 simulate_trace
int tgref_simulate_trace(const uint64_t* counts, uint64_t n, const uint64_t* layout6,
                         uint64_t* report6) {
  return guard([&] {
    const auto c = tg::make_access_counter(std::vector<uint64_t>(counts, counts + n));
    put_report(tg::simulate_trace(c, make_layout(layout6)), report6);
  });
}

// tiering.cpp:164-175 counts_in_row_order
int tgref_counts_in_row_order(const uint64_t* counts, uint64_t n, const uint64_t* ordering,
                              uint64_t m, uint64_t* out) {
  return guard([&] {
    const auto c = tg::make_access_counter(std::vector<uint64_t>(counts, counts + n));
    const auto r = tg::counts_in_row_order(c, std::span<const uint64_t>(ordering, m));
    if (!r.empty()) std::memcpy(out, r.data(), sizeof(uint64_t) * r.size());
  });
}

// tiering.cpp:177-202 hot_fraction_sweep ; per fraction: layout6 then report6
int tgref_hot_fraction_sweep(const uint64_t* counts, uint64_t n, const uint64_t* ordering,
                             const double* fractions, uint64_t nf, double replicated,
                             uint32_t devices, uint64_t dim, uint32_t elem_bytes,
                             uint64_t budget, uint64_t* out_layouts, uint64_t* out_reports,
                             double* out_rep_fractions) {
  return guard([&] {
    const auto c = tg::make_access_counter(std::vector<uint64_t>(counts, counts + n));
    const auto rows =
        tg::hot_fraction_sweep(c, std::span<const uint64_t>(ordering, n),
                               std::span<const double>(fractions, nf), replicated, devices,
                               dim, elem_bytes, budget);
    for (size_t i = 0; i < rows.size(); ++i) {
      const auto& l = rows[i].layout;
      uint64_t* o = out_layouts + 6 * i;
      o[0] = l.num_rows;
      o[1] = l.local_boundary;
      o[2] = l.multi_boundary;
      o[3] = l.num_devices;
      o[4] = l.feature_dim;
      o[5] = l.elem_bytes;
      put_report(rows[i].report, out_reports + 6 * i);
      out_rep_fractions[i] = rows[i].replicated_fraction;
    }
  });
}

// TrafficReport::hit_ratio / est_transfer_seconds (tiering.cpp:25-36)
double tgref_hit_ratio(const uint64_t* report6) { return get_report(report6).hit_ratio(); }
double tgref_est_transfer_seconds(const uint64_t* report6, double l, double p, double h) {
  return get_report(report6).est_transfer_seconds({l, p, h});
}

// ---- sampling (sampling.cpp) — the producer of the gather's id lists
int tgref_build_minibatch(void* gt_handle, const uint64_t* seeds, uint64_t nseeds,
                          const uint32_t* fanouts, uint32_t nf, uint64_t rng_seed,
                          uint64_t epoch, uint64_t batch, uint64_t** out, uint64_t* out_n) {
  return guard([&] {
    tg::FanoutSpec spec;
    spec.fanouts.assign(fanouts, fanouts + nf);
    const tg::BatchRng rng{rng_seed, epoch, batch};
    const auto ids = tg::build_minibatch(static_cast<RefGraph*>(gt_handle)->g,
                                         std::span<const uint64_t>(seeds, nseeds), spec, rng);
    *out = dup_vec(ids);
    *out_n = ids.size();
  });
}

// The per-epoch schedule of run_training_trace (sampling.cpp:106-123): shuffle the
// train ids with key {0x5348, epoch}, split into batches, expand batch b with
// BatchRng{seed, epoch, b}. Returns the CSR of all the epoch's minibatch id lists
// (batch b = ids[off[b]..off[b+1])). Uses the reference's own shuffle_in_place,
// derive_stream_key and build_minibatch; the loop is the trace's own loop.
int tgref_epoch_minibatches(void* gt_handle, const uint64_t* tid, uint64_t ntid,
                            const uint32_t* fanouts, uint32_t nf, uint64_t batch_size,
                            uint64_t rng_seed, uint64_t epoch, uint64_t max_batches,
                            uint64_t** out_off, uint64_t* out_nb, uint64_t** out_ids) {
  return guard([&] {
    tg::FanoutSpec spec;
    spec.fanouts.assign(fanouts, fanouts + nf);
    std::vector<uint64_t> order(tid, tid + ntid);
    tg::RngStream shuffle_rng(tg::derive_stream_key(rng_seed, {0x5348ull, epoch}));
    tg::shuffle_in_place(shuffle_rng, order);
    uint64_t nb = (order.size() + batch_size - 1) / batch_size;
    if (max_batches && nb > max_batches) nb = max_batches;
    std::vector<std::vector<uint64_t>> lists(nb);
    const auto& gt = static_cast<RefGraph*>(gt_handle)->g;
    const int workers = tg::worker_count();
#pragma omp parallel for schedule(dynamic) num_threads(workers)
    for (int64_t b = 0; b < static_cast<int64_t>(nb); ++b) {
      const uint64_t begin = static_cast<uint64_t>(b) * batch_size;
      const uint64_t end = std::min<uint64_t>(begin + batch_size, order.size());
      lists[b] = tg::build_minibatch(gt, std::span<const uint64_t>(order.data() + begin, end - begin),
                                     spec, tg::BatchRng{rng_seed, epoch, static_cast<uint64_t>(b)});
    }
    std::vector<uint64_t> off(nb + 1, 0), all;
    for (uint64_t b = 0; b < nb; ++b) off[b + 1] = off[b] + lists[b].size();
    all.reserve(off[nb]);
    for (auto& l : lists) all.insert(all.end(), l.begin(), l.end());
    *out_off = dup_vec(off);
    *out_nb = nb;
    *out_ids = dup_vec(all);
  });
}

// sampling.cpp:92-140 run_training_trace ; out has num_nodes counts
int tgref_run_training_trace(void* g_handle, const uint64_t* tid, uint64_t ntid,
                             const uint32_t* fanouts, uint32_t nf, uint64_t batch_size,
                             uint64_t epochs, uint64_t rng_seed, int dedup, uint64_t* out) {
  return guard([&] {
    tg::TrainIdSet t;
    t.ids.assign(tid, tid + ntid);
    tg::FanoutSpec spec;
    spec.fanouts.assign(fanouts, fanouts + nf);
    tg::TraceConfig cfg;
    cfg.batch_size = batch_size;
    cfg.epochs = epochs;
    cfg.rng_seed = rng_seed;
    cfg.dedup_per_batch = dedup != 0;
    const auto c = tg::run_training_trace(static_cast<RefGraph*>(g_handle)->g, t, spec, cfg);
    if (!c.counts.empty()) std::memcpy(out, c.counts.data(), sizeof(uint64_t) * c.counts.size());
  });
}

// rng.hpp:13-18 mix64 and rng.hpp:23-28 derive_stream_key (for fixture pinning)
uint64_t tgref_mix64(uint64_t x) { return tg::mix64(x); }
uint64_t tgref_derive_stream_key(uint64_t seed, const uint64_t* coords, uint32_t n) {
  uint64_t h = 0;
  switch (n) {  // initializer_list cannot be built at run time; cover the arities used
    case 0: h = tg::derive_stream_key(seed, {}); break;
    case 1: h = tg::derive_stream_key(seed, {coords[0]}); break;
    case 2: h = tg::derive_stream_key(seed, {coords[0], coords[1]}); break;
    case 3: h = tg::derive_stream_key(seed, {coords[0], coords[1], coords[2]}); break;
    case 4: h = tg::derive_stream_key(seed, {coords[0], coords[1], coords[2], coords[3]}); break;
    default:
      h = tg::derive_stream_key(seed, {coords[0], coords[1], coords[2], coords[3], coords[4]});
  }
  return h;
}

// io.cpp: the binary containers (golden files for the device loaders)
int tgref_save_csr(void* h, const char* path) {
  return guard([&] { tg::save_csr(static_cast<RefGraph*>(h)->g, path); });
}
int tgref_load_csr(const char* path, void** out_graph) {
  return guard([&] {
    auto* h = new RefGraph;
    try {
      h->g = tg::load_csr(path);
    } catch (...) {
      delete h;
      throw;
    }
    *out_graph = h;
  });
}
int tgref_save_features(void* h, const char* path) {
  return guard([&] { tg::save_features(static_cast<RefFeatures*>(h)->f, path); });
}
int tgref_load_features(const char* path, void** out) {
  return guard([&] {
    auto* h = new RefFeatures;
    try {
      h->f = tg::load_features(path);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
int tgref_save_perm(const uint64_t* perm, uint64_t n, const char* path) {
  return guard([&] { tg::save_u64_vector(std::vector<uint64_t>(perm, perm + n), "PERM", path); });
}

}  // extern "C"
