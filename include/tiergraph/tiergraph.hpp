// tiergraph.hpp — the C++ drop-in API of the B200 tiergraph hot path.
//
// Same namespace, type layouts and signatures as the reference C++ toolkit
// (arXiv 2111.05894 `tiergraph`, proj/include/tiergraph/*.hpp) for the part
// of it on the data-tiering hot path: scoring (hot-set prediction), reorder
// (permutation and row layout), tiering (address map, accounting, replay),
// and the sampler that produces the gather's id lists. The computations run
// on the GPU through the C-ABI in tg_capi.h; the bodies live in
// paper_2111_05894_b200/csrc/cxx_api.cpp and cxx_sampling.cpp, which compile
// unchanged against either this header or the reference's own headers (that
// second build is the drop-in proof).
//
// The per-subsystem header names of the reference (tiergraph/scoring.hpp, ...)
// exist in this directory as forwarders to this file.
//
// Results are returned by value and calls are synchronous, as in the
// reference. Internally each call borrows a device context (one CUDA stream +
// scratch) from a process-wide pool on the device named by TIERGRAPH_DEVICES
// (default 0), mirroring TIERGRAPH_THREADS (reference parallel.cpp:13-19).
#pragma once

#include <cstdint>
#include <initializer_list>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace tiergraph {

// ---------------------------------------------------------------- types
// reference types.hpp:9-29. Error classes keep the reference's bases so
// `catch (const std::invalid_argument&)` still sees DomainError.
using NodeId = std::uint64_t;
using EdgeIdx = std::uint64_t;

struct IoError : std::runtime_error {
  explicit IoError(const std::string& what) : std::runtime_error(what) {}
};
struct FormatError : std::runtime_error {
  explicit FormatError(const std::string& what) : std::runtime_error(what) {}
};
struct DomainError : std::invalid_argument {
  explicit DomainError(const std::string& what) : std::invalid_argument(what) {}
};

// ---------------------------------------------------------------- graph
// reference csr_graph.hpp:22-35: row u = targets[offsets[u] .. offsets[u+1])
// holds u's OUT-neighbours. Two vectors, offsets first (layout-identical).
struct CsrGraph {
  std::vector<EdgeIdx> offsets;
  std::vector<NodeId> targets;

  NodeId num_nodes() const { return offsets.size() ? offsets.size() - 1 : 0; }
  EdgeIdx num_edges() const { return targets.size(); }
  std::span<const NodeId> row(NodeId u) const {
    return std::span<const NodeId>(targets).subspan(offsets[u], offsets[u + 1] - offsets[u]);
  }
  EdgeIdx out_degree(NodeId u) const { return offsets[u + 1] - offsets[u]; }
  bool operator==(const CsrGraph&) const = default;
};

// reference csr_graph.cpp:89-93 — K1 on the GPU (standalone library only; a
// drop-in build keeps the reference's own csr_graph.cpp).
std::vector<EdgeIdx> in_degrees(const CsrGraph& g);

// ------------------------------------------------------------- features
// reference feature_matrix.hpp:14-28: row-major, element type opaque.
struct FeatureMatrix {
  std::uint64_t num_rows = 0;
  std::uint64_t dim = 0;
  std::uint32_t elem_bytes = 0;
  std::vector<std::uint8_t> data;

  std::uint64_t row_bytes() const { return dim * elem_bytes; }
  std::span<const std::uint8_t> row(std::uint64_t r) const {
    return std::span<const std::uint8_t>(data).subspan(r * row_bytes(), row_bytes());
  }
  std::span<std::uint8_t> row(std::uint64_t r) {
    return std::span<std::uint8_t>(data).subspan(r * row_bytes(), row_bytes());
  }
};

// reference feature_matrix.cpp:9-14 (FormatError on a size mismatch).
void validate_features(const FeatureMatrix& f);

// -------------------------------------------------------------- scoring
// reference scoring.hpp:12-49.
using ScoreVector = std::vector<double>;

struct TrainIdSet {
  std::vector<NodeId> ids;  // sorted, unique, < num_nodes
  static TrainIdSet from_ids(std::vector<NodeId> raw, NodeId num_nodes);
};

TrainIdSet draw_random_train_ids(NodeId num_nodes, NodeId count, std::uint64_t seed);

struct PagerankConfig {
  std::uint32_t iterations = 5;
  double damp = 0.85;
};

ScoreVector degree_score(const CsrGraph& g);
// Bit-identical to the reference (fp64, per-row left-to-right sums, no FMA).
ScoreVector reverse_pagerank(const CsrGraph& g, const PagerankConfig& cfg);
ScoreVector weighted_reverse_pagerank(const CsrGraph& g, const PagerankConfig& cfg,
                                      const TrainIdSet& tid);
// Descending score, ties by ascending id (GPU radix sort).
std::vector<NodeId> score_ordering(const ScoreVector& scores);

// -------------------------------------------------------------- reorder
// reference reorder.hpp:13-40.
struct NodePermutation {
  std::vector<NodeId> new_id_of;
  NodeId size() const { return new_id_of.size(); }
  NodeId operator[](NodeId old_id) const { return new_id_of[old_id]; }
};

void validate_permutation(const NodePermutation& perm);
NodePermutation permutation_from_scores(const ScoreVector& scores);
NodePermutation invert(const NodePermutation& perm);
CsrGraph reorder_graph(const CsrGraph& g, const NodePermutation& perm);
CsrGraph sequential_reorder_oracle(const CsrGraph& g, const NodePermutation& perm);
FeatureMatrix reorder_features(const FeatureMatrix& f, const NodePermutation& perm);

// --------------------------------------------------------- graph helpers
// reference csr_graph.hpp:48 — canonical transpose (host; standalone library
// only, a drop-in build keeps the reference's csr_graph.cpp).
CsrGraph transpose(const CsrGraph& g);

// ------------------------------------------------------------------- rng
// reference rng.hpp:13-73: splitmix64, stream keys and the counter-based
// stream the samplers draw from (header-only there, restated here).
constexpr std::uint64_t mix64(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

inline std::uint64_t derive_stream_key(std::uint64_t seed,
                                       std::initializer_list<std::uint64_t> coords) {
  std::uint64_t key = mix64(seed ^ 0x6A09E667F3BCC908ull);
  for (const std::uint64_t c : coords) key = mix64(key ^ mix64(c));
  return key;
}

class RngStream {
 public:
  explicit RngStream(std::uint64_t key) : counter_(key) {}
  std::uint64_t next_u64() { return mix64(counter_++); }
  // uniform in [0, bound): Lemire's multiply-shift, rejecting the biased low part
  std::uint64_t next_below(std::uint64_t bound) {
    unsigned __int128 prod = static_cast<unsigned __int128>(next_u64()) * bound;
    if (static_cast<std::uint64_t>(prod) < bound) {
      const std::uint64_t floor = (0 - bound) % bound;
      while (static_cast<std::uint64_t>(prod) < floor)
        prod = static_cast<unsigned __int128>(next_u64()) * bound;
    }
    return static_cast<std::uint64_t>(prod >> 64);
  }
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

 private:
  std::uint64_t counter_;
};

// reference rng.cpp:8-40 (Floyd's k-subset; standalone library only).
void sample_index_subset(RngStream& rng, std::uint64_t population, std::uint64_t k,
                         std::vector<std::uint64_t>& out);

template <typename T>
void shuffle_in_place(RngStream& rng, std::vector<T>& items) {  // rng.hpp:67-73
  for (std::size_t i = items.size(); i > 1; --i)
    std::swap(items[i - 1], items[static_cast<std::size_t>(rng.next_below(i))]);
}

// -------------------------------------------------------------- sampling
// reference sampling.hpp:12-72. build_minibatch and run_training_trace run on
// the GPU (csrc/sampling.cu, bit-identical); sample_in_neighbors (one node,
// a caller-owned stream) and cumulative_access_curve stay on the host.
struct FanoutSpec {
  std::vector<std::uint32_t> fanouts;
};
void validate_fanouts(const FanoutSpec& spec);

struct TraceConfig {
  std::uint64_t batch_size = 1000;
  std::uint64_t epochs = 1;
  std::uint64_t rng_seed = 0;
  bool dedup_per_batch = true;
};

struct AccessCounter {
  std::vector<std::uint64_t> counts;
  std::uint64_t total = 0;
};
AccessCounter make_access_counter(std::vector<std::uint64_t> counts);

struct BatchRng {
  std::uint64_t rng_seed = 0;
  std::uint64_t epoch = 0;
  std::uint64_t batch_index = 0;
  RngStream stream(std::uint32_t layer, NodeId node) const;
};

std::vector<NodeId> sample_in_neighbors(const CsrGraph& gt, NodeId node, std::uint32_t fanout,
                                        RngStream& rng);
std::vector<NodeId> build_minibatch(const CsrGraph& gt, std::span<const NodeId> seeds,
                                    const FanoutSpec& fanouts, const BatchRng& rng,
                                    std::vector<NodeId>* raw_draws = nullptr);
AccessCounter run_training_trace(const CsrGraph& g, const TrainIdSet& tid,
                                 const FanoutSpec& fanouts, const TraceConfig& cfg);
std::vector<double> cumulative_access_curve(const AccessCounter& counter,
                                            std::span<const NodeId> ordering);

// -------------------------------------------------------------- tiering
// reference tiering.hpp:16-121.
struct TierLayout {
  std::uint64_t num_rows = 0;
  std::uint64_t local_boundary = 0;  // [0, lb): replicated on every device
  std::uint64_t multi_boundary = 0;  // [lb, mb): interleaved; [mb, N): host
  std::uint32_t num_devices = 1;
  std::uint64_t feature_dim = 0;
  std::uint32_t elem_bytes = 0;
  std::uint64_t bytes_per_row() const { return feature_dim * elem_bytes; }
};
void validate_layout(const TierLayout& layout);

enum class Tier : std::uint8_t { LocalHot, InterleavedDevice, ColdHost };

struct Location {
  Tier tier = Tier::ColdHost;
  std::uint32_t device = 0;
  std::uint64_t row_within_tier = 0;
  bool operator==(const Location&) const = default;
};

struct LinkCostModel {
  double local_gbps = 900.0;
  double peer_gbps = 150.0;
  double host_gbps = 16.0;
};
void validate_cost_model(const LinkCostModel& cost);

struct TrafficReport {
  std::uint64_t local_accesses = 0;
  std::uint64_t peer_accesses = 0;
  std::uint64_t host_accesses = 0;
  std::uint64_t local_bytes = 0;
  std::uint64_t peer_bytes = 0;
  std::uint64_t host_bytes = 0;

  std::uint64_t total_accesses() const { return local_accesses + peer_accesses + host_accesses; }
  double hit_ratio() const;
  double est_transfer_seconds(const LinkCostModel& cost) const;
  TrafficReport& operator+=(const TrafficReport& other);
  bool operator==(const TrafficReport&) const = default;
};

Location resolve(const TierLayout& layout, std::uint64_t row_id, std::uint32_t requesting_device);
TierLayout plan_layout(std::uint64_t num_rows, double hot_fraction, double replicated_fraction,
                       std::uint32_t num_devices, std::uint64_t feature_dim,
                       std::uint32_t elem_bytes, std::uint64_t per_device_budget_bytes = 0);
// Accounting only (the reference moves no bytes); TieredFeatureStore::gather_rows
// (tiergraph/tiered_store.hpp) moves them.
void gather(const TierLayout& layout, std::span<const std::uint64_t> row_ids,
            std::uint32_t requesting_device, TrafficReport& report);
TrafficReport simulate_trace(const AccessCounter& counter, const TierLayout& layout);
std::vector<std::uint64_t> counts_in_row_order(const AccessCounter& counter,
                                               std::span<const NodeId> ordering);

struct SweepRow {
  double hot_fraction = 0.0;
  double replicated_fraction = 0.0;
  TierLayout layout;
  TrafficReport report;
};
std::vector<SweepRow> hot_fraction_sweep(const AccessCounter& counter,
                                         std::span<const NodeId> ordering,
                                         std::span<const double> fractions,
                                         double replicated_fraction, std::uint32_t num_devices,
                                         std::uint64_t feature_dim, std::uint32_t elem_bytes,
                                         std::uint64_t per_device_budget_bytes = 0);
void write_report_csv(std::span<const SweepRow> rows, const LinkCostModel& cost,
                      const std::string& path);

}  // namespace tiergraph
