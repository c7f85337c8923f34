// Host-side producers of the hot path's inputs (NOT the hot path): the
// seeded train-id draw, the graph transpose and the GraphSAGE minibatch
// expansion that yields the per-minibatch node-id lists the tiered gather
// consumes. They restate the reference's counter-based algorithms so the id
// lists are bit-identical to the reference's (tests/test_gpu_gather.py
// checks them against the reference build):
//   rng.hpp:13-59 (mix64, derive_stream_key, RngStream, Lemire next_below)
//   rng.cpp:8-40 (Floyd k-subset), rng.hpp:67-73 (Fisher-Yates)
//   scoring.cpp:22-31 (draw_random_train_ids)
//   csr_graph.cpp:67-80 (transpose)
//   sampling.cpp:35-90 (BatchRng streams, sample_in_neighbors, build_minibatch)
//   sampling.cpp:106-123 (per-epoch shuffle + batching of run_training_trace)
// Moving sampling onto the GPU is SURVEY §8(f) row 1 ("next").
#include <omp.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "tg_capi.h"

namespace {

thread_local std::string t_err;

inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t stream_key(uint64_t seed, const uint64_t* c, int n) {
  uint64_t h = mix64(seed ^ 0x6A09E667F3BCC908ull);
  for (int i = 0; i < n; ++i) h = mix64(h ^ mix64(c[i]));
  return h;
}

struct Rng {
  uint64_t s;
  uint64_t next() { return mix64(s++); }
  uint64_t below(uint64_t bound) {
    uint64_t x = next();
    unsigned __int128 m = static_cast<unsigned __int128>(x) * bound;
    uint64_t lo = static_cast<uint64_t>(m);
    if (lo < bound) {
      const uint64_t t = (0 - bound) % bound;
      while (lo < t) {
        x = next();
        m = static_cast<unsigned __int128>(x) * bound;
        lo = static_cast<uint64_t>(m);
      }
    }
    return static_cast<uint64_t>(m >> 64);
  }
};

// Floyd: emits t unless already emitted, else j (membership over emitted values).
void k_subset(Rng& rng, uint64_t pop, uint64_t k, std::vector<uint64_t>& out) {
  out.clear();
  if (k >= pop) {
    for (uint64_t i = 0; i < pop; ++i) out.push_back(i);
    return;
  }
  if (k <= 64) {
    for (uint64_t j = pop - k; j < pop; ++j) {
      const uint64_t t = rng.below(j + 1);
      out.push_back(std::find(out.begin(), out.end(), t) != out.end() ? j : t);
    }
    return;
  }
  uint64_t cap = 1;
  while (cap < 4 * k) cap <<= 1;
  std::vector<uint64_t> tab(cap, ~0ull);
  auto insert = [&](uint64_t v) {
    uint64_t h = mix64(v) & (cap - 1);
    while (tab[h] != ~0ull) {
      if (tab[h] == v) return false;
      h = (h + 1) & (cap - 1);
    }
    tab[h] = v;
    return true;
  };
  for (uint64_t j = pop - k; j < pop; ++j) {
    const uint64_t t = rng.below(j + 1);
    if (insert(t)) {
      out.push_back(t);
    } else {
      insert(j);
      out.push_back(j);
    }
  }
}

void sort_unique(std::vector<uint64_t>& v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}

std::vector<uint64_t> build_minibatch(const uint64_t* off, const uint64_t* tgt, const uint64_t* seeds,
                                      uint64_t ns, const uint32_t* fan, uint32_t nf, uint64_t seed,
                                      uint64_t epoch, uint64_t batch) {
  std::vector<uint64_t> frontier(seeds, seeds + ns), next, picks;
  sort_unique(frontier);
  std::vector<uint64_t> members = frontier;
  for (uint32_t layer = 0; layer < nf; ++layer) {
    next.clear();
    for (const uint64_t v : frontier) {
      const uint64_t b = off[v], deg = off[v + 1] - b;
      if (deg <= fan[layer]) {
        next.insert(next.end(), tgt + b, tgt + b + deg);
      } else {
        const uint64_t c[5] = {0x534Dull, epoch, batch, layer, v};  // sampling.cpp:35-37
        Rng rng{stream_key(seed, c, 5)};
        k_subset(rng, deg, fan[layer], picks);
        for (const uint64_t p : picks) next.push_back(tgt[b + p]);
      }
    }
    sort_unique(next);
    frontier.swap(next);
    members.insert(members.end(), frontier.begin(), frontier.end());
    if (frontier.empty()) break;
  }
  sort_unique(members);
  return members;
}

uint64_t* dup(const std::vector<uint64_t>& v) {
  auto* p = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * std::max<size_t>(v.size(), 1)));
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(uint64_t) * v.size());
  return p;
}

}  // namespace

extern "C" {

const char* tg_host_last_error(void) { return t_err.c_str(); }
void tg_free(void* p) { std::free(p); }

int tg_draw_random_train_ids(uint64_t num_nodes, uint64_t count, uint64_t seed, uint64_t* out) {
  if (count < 1 || count > num_nodes) {
    t_err = "need 1 <= count <= num_nodes, got count=" + std::to_string(count) + " for " +
            std::to_string(num_nodes) + " nodes";
    return TG_ERR_DOMAIN;
  }
  const uint64_t tag = 0x6C61ull;
  Rng rng{stream_key(seed, &tag, 1)};
  std::vector<uint64_t> picks;
  k_subset(rng, num_nodes, count, picks);
  std::sort(picks.begin(), picks.end());
  std::memcpy(out, picks.data(), sizeof(uint64_t) * count);
  return TG_OK;
}

int tg_transpose_host(const uint64_t* off, const uint64_t* tgt, uint64_t n, uint64_t* t_off,
                      uint64_t* t_tgt) {
  const uint64_t e = off[n];
  std::vector<std::atomic<uint64_t>> cnt(n + 1);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < static_cast<int64_t>(n + 1); ++i) cnt[i].store(0, std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < static_cast<int64_t>(e); ++i)
    cnt[tgt[i] + 1].fetch_add(1, std::memory_order_relaxed);
  t_off[0] = 0;
  for (uint64_t v = 0; v < n; ++v) t_off[v + 1] = t_off[v] + cnt[v + 1].load(std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < static_cast<int64_t>(n); ++v) cnt[v].store(t_off[v], std::memory_order_relaxed);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t u = 0; u < static_cast<int64_t>(n); ++u)
    for (uint64_t k = off[u]; k < off[u + 1]; ++k)
      t_tgt[cnt[tgt[k]].fetch_add(1, std::memory_order_relaxed)] = static_cast<uint64_t>(u);
  // every transposed row ascending, as the reference's source-order walk leaves it
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < static_cast<int64_t>(n); ++v) std::sort(t_tgt + t_off[v], t_tgt + t_off[v + 1]);
  return TG_OK;
}

int tg_epoch_order(const uint64_t* tid, uint64_t ntid, uint64_t seed, uint64_t epoch,
                   uint64_t* out) {
  std::memcpy(out, tid, sizeof(uint64_t) * ntid);
  const uint64_t sc[2] = {0x5348ull, epoch};  // sampling.cpp:108
  Rng sh{stream_key(seed, sc, 2)};
  for (size_t i = ntid; i > 1; --i) std::swap(out[i - 1], out[sh.below(i)]);  // rng.hpp:67-73
  return TG_OK;
}

int tg_epoch_minibatches(const uint64_t* gt_off, const uint64_t* gt_tgt, uint64_t n,
                         const uint64_t* tid, uint64_t ntid, const uint32_t* fanouts, uint32_t nf,
                         uint64_t batch_size, uint64_t seed, uint64_t epoch, uint64_t first_batch,
                         uint64_t max_batches, int threads, uint64_t** out_off, uint64_t* out_nb,
                         uint64_t** out_ids) {
  if (nf == 0 || nf > 5) {
    t_err = "fanout depth must be 1..5";
    return TG_ERR_DOMAIN;
  }
  for (uint32_t i = 0; i < nf; ++i)
    if (fanouts[i] < 1) {
      t_err = "every fanout must be >= 1";
      return TG_ERR_DOMAIN;
    }
  if (batch_size < 1 || ntid == 0) {
    t_err = "batch_size and the train id set must be non-empty";
    return TG_ERR_DOMAIN;
  }
  for (uint64_t i = 0; i < ntid; ++i)
    if (tid[i] >= n) {
      t_err = "train id " + std::to_string(tid[i]) + " out of range";
      return TG_ERR_DOMAIN;
    }
  std::vector<uint64_t> order(tid, tid + ntid);
  const uint64_t sc[2] = {0x5348ull, epoch};  // sampling.cpp:108
  Rng sh{stream_key(seed, sc, 2)};
  for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[sh.below(i)]);
  const uint64_t total = (order.size() + batch_size - 1) / batch_size;
  const uint64_t b0 = std::min(first_batch, total);
  uint64_t nb = total - b0;
  if (max_batches && nb > max_batches) nb = max_batches;
  std::vector<std::vector<uint64_t>> lists(nb);
  const int th = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic) num_threads(th)
  for (int64_t i = 0; i < static_cast<int64_t>(nb); ++i) {
    const uint64_t b = b0 + static_cast<uint64_t>(i);
    const uint64_t beg = b * batch_size, end = std::min<uint64_t>(beg + batch_size, order.size());
    lists[i] = build_minibatch(gt_off, gt_tgt, order.data() + beg, end - beg, fanouts, nf, seed,
                               epoch, b);
  }
  std::vector<uint64_t> off(nb + 1, 0), all;
  for (uint64_t i = 0; i < nb; ++i) off[i + 1] = off[i] + lists[i].size();
  all.reserve(off[nb]);
  for (auto& l : lists) all.insert(all.end(), l.begin(), l.end());
  *out_off = dup(off);
  *out_nb = nb;
  *out_ids = dup(all);
  return TG_OK;
}

}  // extern "C"
