// cxx_support.cpp — the few non-hot-path reference symbols the standalone C++
// library needs so that tiergraph.hpp is self-sufficient. A drop-in build
// against the reference headers links the reference's own csr_graph.cpp,
// feature_matrix.cpp and sampling.cpp instead, and does not compile this file.
#include <algorithm>
#include <string>
#include <utility>
#include <vector>

#include "cxx_common.hpp"
#include "tiergraph/tiergraph.hpp"

namespace tiergraph {

// csr_graph.cpp:89-93 — K1 (shared-memory privatised histogram) on the GPU.
std::vector<EdgeIdx> in_degrees(const CsrGraph& g) {
  std::vector<EdgeIdx> out(g.num_nodes());
  if (out.empty()) return out;
  b200::GraphLease dg(g);
  b200::check(tg_in_degrees(dg.ctx(), dg.graph(), out.data()));
  return out;
}

// feature_matrix.cpp:9-14
void validate_features(const FeatureMatrix& f) {
  const std::uint64_t want = f.num_rows * f.dim * f.elem_bytes;
  if (f.data.size() != want)
    throw FormatError("features: data holds " + std::to_string(f.data.size()) +
                      " bytes, expected " + std::to_string(want));
}

// csr_graph.cpp:67-80 — canonical transpose on the device (tg_transpose: a
// stable radix sort of the edges by target in CSR order, so every transposed
// row lists its sources ascending, bit-identical to the reference).
CsrGraph transpose(const CsrGraph& g) {
  const uint64_t n = g.num_nodes();
  CsrGraph t;
  t.offsets.assign(n + 1, 0);
  t.targets.resize(g.num_edges());
  if (n == 0) return t;
  static const uint64_t kNone = 0;
  uint64_t scratch = 0;
  b200::Ctx ctx;
  b200::check(tg_transpose(ctx, g.offsets.data(), g.targets.empty() ? &kNone : g.targets.data(), n,
                           g.num_edges(), t.offsets.data(),
                           t.targets.empty() ? &scratch : t.targets.data()));
  return t;
}

// rng.cpp:8-40 — Floyd's k-subset: draw t in [0, j] for j = pop-k .. pop-1 and
// take t unless already taken, else j.
void sample_index_subset(RngStream& rng, std::uint64_t population, std::uint64_t k,
                         std::vector<std::uint64_t>& out) {
  out.clear();
  if (k >= population) {
    for (std::uint64_t i = 0; i < population; ++i) out.push_back(i);
    return;
  }
  for (std::uint64_t j = population - k; j < population; ++j) {
    const std::uint64_t t = rng.next_below(j + 1);
    out.push_back(std::find(out.begin(), out.end(), t) == out.end() ? t : j);
  }
}

}  // namespace tiergraph
