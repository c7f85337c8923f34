// cxx_support.cpp — the few non-hot-path reference symbols the standalone C++
// library needs so that tiergraph.hpp is self-sufficient. A drop-in build
// against the reference headers links the reference's own csr_graph.cpp,
// feature_matrix.cpp and sampling.cpp instead, and does not compile this file.
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
  b200::Ctx ctx;
  b200::DevGraph dg(ctx, g);
  b200::check(tg_in_degrees(ctx, dg.get(), out.data()));
  return out;
}

// feature_matrix.cpp:9-14
void validate_features(const FeatureMatrix& f) {
  const std::uint64_t want = f.num_rows * f.dim * f.elem_bytes;
  if (f.data.size() != want)
    throw FormatError("features: data holds " + std::to_string(f.data.size()) +
                      " bytes, expected " + std::to_string(want));
}

// sampling.cpp:27-33 — total is the sum of the counts.
AccessCounter make_access_counter(std::vector<std::uint64_t> counts) {
  AccessCounter c;
  for (const std::uint64_t v : counts) c.total += v;
  c.counts = std::move(counts);
  return c;
}

}  // namespace tiergraph
