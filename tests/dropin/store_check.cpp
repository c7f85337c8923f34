// store_check.cpp — C++ API check of the byte-moving tiered gather.
//
// Built against include/tiergraph (this repo's drop-in headers) and linked
// with libtiergraph_b200_cxx.so by tests/test_dropin.py. Runs the C++ path a
// reference user would write: score -> permute -> plan -> TieredFeatureStore
// -> gather_rows from every layout device, and checks
//   * rows byte-equal to reorder_features(f, perm).row(id)  (reorder.cpp:97-117)
//   * the report equal to gather(layout, ids, device, .)     (tiering.cpp:100-125)
//   * an out-of-range id throws DomainError after the prefix was accounted.
// Layout devices outnumbering GPUs share a GPU (peer reads are then same-GPU).
// Prints "store_check ok ..." and exits 0 on success.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tiergraph/scoring.hpp"
#include "tiergraph/tiered_store.hpp"
#include "tiergraph/tiering.hpp"

using namespace tiergraph;

static int fails = 0;
#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);    \
      ++fails;                                                      \
    }                                                               \
  } while (0)

int main(int argc, char** argv) {
  const std::uint32_t D = argc > 1 ? static_cast<std::uint32_t>(std::atoi(argv[1])) : 4;
  const NodeId n = 5000;
  // a small random-ish graph: node u -> (u*7+k*13) % n
  CsrGraph g;
  g.offsets.push_back(0);
  for (NodeId u = 0; u < n; ++u) {
    std::vector<NodeId> row;
    for (NodeId k = 0; k < (u % 9); ++k) row.push_back((u * 7 + k * 13 + 1) % n);
    std::sort(row.begin(), row.end());
    row.erase(std::unique(row.begin(), row.end()), row.end());
    g.targets.insert(g.targets.end(), row.begin(), row.end());
    g.offsets.push_back(g.targets.size());
  }
  const TrainIdSet tid = draw_random_train_ids(n, n / 10, 3);
  const ScoreVector s = weighted_reverse_pagerank(g, PagerankConfig{}, tid);
  const NodePermutation perm = permutation_from_scores(s);

  // 24-dim fp32 rows (96 B) with a closed-form fill
  FeatureMatrix f;
  f.num_rows = n;
  f.dim = 24;
  f.elem_bytes = 4;
  f.data.resize(n * f.row_bytes());
  for (NodeId r = 0; r < n; ++r)
    for (std::uint64_t c = 0; c < f.dim; ++c) {
      const float v = static_cast<float>(r) * 0.5f + static_cast<float>(c);
      std::memcpy(f.data.data() + r * f.row_bytes() + c * 4, &v, 4);
    }
  const FeatureMatrix want = reorder_features(f, perm);

  for (const bool indirect : {false, true}) {
    const TierLayout lay = plan_layout(n, 0.3, 0.05, D, f.dim, f.elem_bytes);
    TieredStoreOptions opt;
    opt.cold_indirect = indirect;
    TieredFeatureStore store(f, perm, lay, {}, opt);
    std::vector<std::uint64_t> ids;
    for (NodeId i = 0; i < n; i += 3) ids.push_back(i);
    std::vector<std::uint8_t> out(ids.size() * f.row_bytes());
    for (std::uint32_t dev = 0; dev < D; ++dev) {
      TrafficReport got, ref;
      store.gather_rows(ids, dev, out.data(), got);
      gather(lay, ids, dev, ref);
      EXPECT(got == ref);
      EXPECT(got.peer_accesses > 0 || D == 1);
      bool same = true;
      for (size_t i = 0; i < ids.size(); ++i)
        same &= std::memcmp(out.data() + i * f.row_bytes(), want.row(ids[i]).data(),
                            f.row_bytes()) == 0;
      EXPECT(same);
    }
    // bad id: prefix accounted, then DomainError (tiering.cpp:50-52)
    std::vector<std::uint64_t> bad = {1, 2, n + 5, 3};
    TrafficReport r;
    bool threw = false;
    try {
      store.gather_rows(bad, 0, out.data(), r);
    } catch (const DomainError&) {
      threw = true;
    }
    EXPECT(threw);
    EXPECT(r.total_accesses() == 2);
  }
  std::printf("store_check %s: D=%u n=%llu\n", fails ? "FAILED" : "ok", D,
              static_cast<unsigned long long>(n));
  return fails ? 1 : 0;
}
