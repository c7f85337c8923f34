// api_check.cpp — the reference C++ API as a caller uses it, on this library
// (include/tiergraph + libtiergraph_b200_cxx.so), driven by
// tests/test_dropin.py::test_cxx_api_cache_and_devices.
//
//   api_check <graph.bin> <out_prefix> [reps]
// reads a CSR (u64 n, u64 e, offsets[n+1], targets[e]) and a train-id list
// from <graph.bin>, then
//   * runs weighted_reverse_pagerank `reps` times and writes the scores of
//     the first call to <out_prefix>.scores (the test compares them with the
//     reference build, raw bytes) and the per-call host time to stdout: the
//     first call uploads the graph, the rest reuse the cached device copy
//     (VERDICT r01 #8); TIERGRAPH_DEVICES with several entries partitions the
//     rows over them (tg_mgraph);
//   * runs build_minibatch for a few batches twice and checks both runs equal
//     (the cached sampler state is reused);
//   * rebuilds the graph with one edge removed and checks that the scores
//     change (the cache key follows the content);
//   * transpose() on the device equals a host transpose.
// Prints "api_check ok ..." on success.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tiergraph/tiergraph.hpp"

using namespace tiergraph;
using Clock = std::chrono::steady_clock;

static int fails = 0;
#define EXPECT(c)                                                \
  do {                                                           \
    if (!(c)) {                                                  \
      std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                   \
    }                                                            \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const int reps = argc > 3 ? std::atoi(argv[3]) : 3;
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 2;
  uint64_t n = 0, e = 0, nt = 0;
  if (std::fread(&n, 8, 1, f) != 1 || std::fread(&e, 8, 1, f) != 1) return 2;
  CsrGraph g;
  g.offsets.resize(n + 1);
  g.targets.resize(e);
  if (std::fread(g.offsets.data(), 8, n + 1, f) != n + 1) return 2;
  if (e && std::fread(g.targets.data(), 8, e, f) != e) return 2;
  if (std::fread(&nt, 8, 1, f) != 1) return 2;
  TrainIdSet tid;
  tid.ids.resize(nt);
  if (nt && std::fread(tid.ids.data(), 8, nt, f) != nt) return 2;
  std::fclose(f);

  const PagerankConfig cfg{5, 0.85};
  ScoreVector first;
  for (int r = 0; r < reps; ++r) {
    const auto t0 = Clock::now();
    ScoreVector s = weighted_reverse_pagerank(g, cfg, tid);
    const double ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
    std::printf("call %d: %.3f ms\n", r, ms);
    if (r == 0) first = s;
    else EXPECT(std::memcmp(s.data(), first.data(), 8 * n) == 0);
  }
  {
    FILE* o = std::fopen((std::string(argv[2]) + ".scores").c_str(), "wb");
    std::fwrite(first.data(), 8, n, o);
    std::fclose(o);
  }
  // unweighted and degree score through the same cache entry
  const ScoreVector u = reverse_pagerank(g, PagerankConfig{3, 0.5});
  {
    FILE* o = std::fopen((std::string(argv[2]) + ".plain").c_str(), "wb");
    std::fwrite(u.data(), 8, n, o);
    std::fclose(o);
  }
  const ScoreVector deg = degree_score(g);
  for (uint64_t i = 0; i < n; ++i) EXPECT(deg[i] == double(g.offsets[i + 1] - g.offsets[i]));

  // a content change at the same sizes is a different cache entry
  if (e > 1) {
    CsrGraph h = g;
    // move the last edge of the first non-empty row to the next row
    uint64_t u0 = 0;
    while (g.offsets[u0 + 1] == g.offsets[u0]) ++u0;
    if (u0 + 1 < n) {
      h.offsets[u0 + 1] -= 1;
      const ScoreVector s2 = weighted_reverse_pagerank(h, cfg, tid);
      EXPECT(std::memcmp(s2.data(), first.data(), 8 * n) != 0);
    }
  }

  // the sampler on the transposed graph, twice (cached state reused)
  const CsrGraph gt = transpose(g);
  {
    // host transpose for comparison (csr_graph.cpp:67-80: ascending sources)
    std::vector<uint64_t> cnt(n + 1, 0);
    for (uint64_t v : g.targets) ++cnt[v + 1];
    for (uint64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
    std::vector<uint64_t> pos(cnt.begin(), cnt.end() - 1), tt(e);
    for (uint64_t s = 0; s < n; ++s)
      for (uint64_t k = g.offsets[s]; k < g.offsets[s + 1]; ++k) tt[pos[g.targets[k]]++] = s;
    EXPECT(gt.offsets == cnt);
    EXPECT(gt.targets == tt);
  }
  FanoutSpec fan;
  fan.fanouts = {10, 5};
  std::vector<std::vector<NodeId>> a, b;
  for (int pass = 0; pass < 2; ++pass)
    for (uint64_t k = 0; k < 4 && k * 64 < nt; ++k) {
      std::vector<NodeId> seeds(tid.ids.begin() + k * 64,
                                tid.ids.begin() + std::min<uint64_t>(nt, (k + 1) * 64));
      auto m = build_minibatch(gt, seeds, fan, BatchRng{7, 0, k}, nullptr);
      (pass ? b : a).push_back(std::move(m));
    }
  EXPECT(a == b && !a.empty());
  {
    FILE* o = std::fopen((std::string(argv[2]) + ".mb0").c_str(), "wb");
    std::fwrite(a[0].data(), 8, a[0].size(), o);
    std::fclose(o);
  }
  if (fails) return 1;
  std::printf("api_check ok: n=%lu e=%lu\n", (unsigned long)n, (unsigned long)e);
  return 0;
}
