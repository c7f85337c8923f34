// cxx_common.hpp — shared plumbing of the C++ drop-in layer (cxx_*.cpp).
//
// Error mapping (C-ABI code -> the reference exception class, types.hpp:13-29)
// and a process-wide pool of device contexts: the reference API is free
// functions on value types and is safe to call from several threads at once
// (SPEC.md:97), so each call leases a tg_ctx (stream + scratch) of its own
// instead of sharing one.
#pragma once

#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "tg_capi.h"
#include "tiergraph/types.hpp"

namespace tiergraph::b200 {

[[noreturn]] inline void raise(int rc) {
  std::string msg = tg_last_error();
  switch (rc) {
    case TG_ERR_DOMAIN: throw DomainError(msg);
    case TG_ERR_FORMAT: throw FormatError(msg);
    case TG_ERR_IO: throw IoError(msg);
    default: throw std::runtime_error("tiergraph_b200: " + msg);
  }
}

inline void check(int rc) {
  if (rc != TG_OK) raise(rc);
}

// Contexts are created on first use and kept for the life of the process
// (destroying CUDA objects from static destructors races the runtime's own
// teardown).
class CtxPool {
 public:
  static CtxPool& get() {
    static CtxPool* pool = new CtxPool;
    return *pool;
  }
  tg_ctx* acquire(int device) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (size_t i = 0; i < free_.size(); ++i)
        if (tg_ctx_device(free_[i]) == device) {
          tg_ctx* c = free_[i];
          free_.erase(free_.begin() + static_cast<long>(i));
          return c;
        }
    }
    tg_ctx* c = nullptr;
    check(tg_ctx_create(device, &c));
    return c;
  }
  void release(tg_ctx* c) {
    std::lock_guard<std::mutex> lk(mu_);
    free_.push_back(c);
  }

 private:
  std::mutex mu_;
  std::vector<tg_ctx*> free_;
};

// RAII lease of a context on the default device (TIERGRAPH_DEVICES).
class Ctx {
 public:
  explicit Ctx(int device = tg_default_device()) : c_(CtxPool::get().acquire(device)) {}
  ~Ctx() { CtxPool::get().release(c_); }
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
  operator tg_ctx*() const { return c_; }

 private:
  tg_ctx* c_;
};

// Device copy of a host CsrGraph for the duration of one call.
class DevGraph {
 public:
  template <class Graph>
  DevGraph(tg_ctx* ctx, const Graph& g) {
    const uint64_t n = g.num_nodes();
    if (n == 0) return;
    static const uint64_t kNoEdge = 0;
    check(tg_graph_create(ctx, g.offsets.data(), g.targets.empty() ? &kNoEdge : g.targets.data(),
                          n, g.targets.size(), &h_));
  }
  ~DevGraph() { tg_graph_destroy(h_); }
  DevGraph(const DevGraph&) = delete;
  DevGraph& operator=(const DevGraph&) = delete;
  const tg_graph* get() const { return h_; }

 private:
  tg_graph* h_ = nullptr;
};

// ---------------------------------------------------------------------------
// Device copies of host graphs kept ACROSS calls: a caller
// that runs weighted_reverse_pagerank / build_minibatch repeatedly on the same
// CsrGraph pays the O(E) upload, the K3 row schedule, K1 and the sampler state
// once, not per call.
//
// An entry is keyed by the graph's array addresses and sizes plus a content
// fingerprint: a hash of EVERY offset and of 4,096 evenly strided targets and
// the first / last 512. A graph rebuilt (other addresses) or edited in a way
// that changes the offsets or any sampled target is uploaded again; an
// in-place rewrite of unsampled targets that keeps every row length is not
// detected -- set TIERGRAPH_DEVICE_CACHE=0 to upload on every call.
// TIERGRAPH_DEVICE_CACHE=<k> keeps at most k graphs (default 2), least
// recently used evicted first. Each entry owns its contexts; calls on one
// entry are serialised by its mutex, calls on different graphs run
// concurrently, as the reference allows.
//
// With several devices in TIERGRAPH_DEVICES the entry also holds the graph
// partitioned over them (tg_mgraph): PageRank then runs row-partitioned on
// every listed device, bit-identical to one device.
inline uint64_t hash_words(const uint64_t* p, uint64_t n, uint64_t h) {
  uint64_t a = h ^ 0x9E3779B97F4A7C15ull, b = h + 0xBF58476D1CE4E5B9ull, c = ~h, d = h * 31;
  uint64_t i = 0;
  for (; i + 4 <= n; i += 4) {
    a = (a ^ p[i]) * 0x100000001B3ull;
    b = (b ^ p[i + 1]) * 0x100000001B3ull;
    c = (c ^ p[i + 2]) * 0x100000001B3ull;
    d = (d ^ p[i + 3]) * 0x100000001B3ull;
  }
  for (; i < n; ++i) a = (a ^ p[i]) * 0x100000001B3ull;
  return a ^ (b << 1) ^ (c << 2) ^ (d << 3) ^ n;
}

struct CachedGraph {
  std::mutex mu;  // one call at a time on this entry
  uint64_t key[5] = {};
  std::vector<tg_ctx*> ctxs;     // own contexts: one per listed device
  tg_graph* g = nullptr;         // whole graph on ctxs[0] (lazy)
  tg_mgraph* mg = nullptr;       // partitioned over every listed device (lazy)
  tg_sampler* sampler = nullptr; // sampler over g (lazy)
  tg_graph* gt = nullptr;        // transpose(g) on ctxs[0] (lazy, run_training_trace)
  tg_sampler* sampler_t = nullptr;
  ~CachedGraph() {
    tg_sampler_destroy(sampler_t);
    tg_graph_destroy(gt);
    tg_sampler_destroy(sampler);
    tg_graph_destroy(g);
    tg_mgraph_destroy(mg);
    for (tg_ctx* c : ctxs) tg_ctx_destroy(c);
  }
};

class GraphCache {
 public:
  static GraphCache& get() {
    static GraphCache* c = new GraphCache;  // never destroyed (CUDA teardown order)
    return *c;
  }
  static int capacity() {
    const char* e = std::getenv("TIERGRAPH_DEVICE_CACHE");
    return e ? std::atoi(e) : 2;
  }
  // The entry for g (created empty, or found); the caller locks entry->mu.
  template <class Graph>
  std::shared_ptr<CachedGraph> lease(const Graph& g) {
    const uint64_t n = g.offsets.size(), e = g.targets.size();
    uint64_t h = hash_words(g.offsets.data(), n, 1);
    std::vector<uint64_t> smp;
    if (e) {
      const uint64_t k = std::min<uint64_t>(e, 4096), st = std::max<uint64_t>(e / k, 1);
      for (uint64_t i = 0; i < e; i += st) smp.push_back(g.targets[i]);
      const uint64_t edge = std::min<uint64_t>(e, 512);
      h = hash_words(g.targets.data(), edge, h);
      h = hash_words(g.targets.data() + (e - edge), edge, h);
    }
    h = hash_words(smp.data(), smp.size(), h);
    const uint64_t key[5] = {reinterpret_cast<uint64_t>(g.offsets.data()),
                             reinterpret_cast<uint64_t>(g.targets.data()), n, e, h};
    const int cap = capacity();
    std::lock_guard<std::mutex> lk(mu_);
    for (auto it = lru_.begin(); it != lru_.end(); ++it)
      if (std::memcmp((*it)->key, key, sizeof key) == 0) {
        auto p = *it;
        lru_.erase(it);
        lru_.push_front(p);
        return p;
      }
    auto p = std::make_shared<CachedGraph>();
    std::memcpy(p->key, key, sizeof key);
    int devs[TG_MAX_DEVICES];
    const int nd = std::min(tg_device_list(devs, TG_MAX_DEVICES), TG_MAX_DEVICES);
    for (int i = 0; i < nd; ++i) {
      tg_ctx* c = nullptr;
      check(tg_ctx_create(devs[i], &c));
      p->ctxs.push_back(c);
    }
    if (cap > 0) {
      lru_.push_front(p);
      while (static_cast<int>(lru_.size()) > cap) lru_.pop_back();  // freed when unleased
    }
    return p;
  }
  void clear() {
    std::lock_guard<std::mutex> lk(mu_);
    lru_.clear();
  }

 private:
  std::mutex mu_;
  std::list<std::shared_ptr<CachedGraph>> lru_;
};

// A locked lease of the cached device state of host graph g.
class GraphLease {
 public:
  template <class Graph>
  explicit GraphLease(const Graph& g) : e_(GraphCache::get().lease(g)), lk_(e_->mu), host_(&g) {
    upload_ = [](CachedGraph* e, const void* hg) {
      const auto& gg = *static_cast<const Graph*>(hg);
      static const uint64_t kNoEdge = 0;
      check(tg_graph_create(e->ctxs[0], gg.offsets.data(),
                            gg.targets.empty() ? &kNoEdge : gg.targets.data(), gg.num_nodes(),
                            gg.targets.size(), &e->g));
    };
    mupload_ = [](CachedGraph* e, const void* hg) {
      const auto& gg = *static_cast<const Graph*>(hg);
      static const uint64_t kNoEdge = 0;
      check(tg_mgraph_create(e->ctxs.data(), static_cast<uint32_t>(e->ctxs.size()),
                             gg.offsets.data(), gg.targets.empty() ? &kNoEdge : gg.targets.data(),
                             gg.num_nodes(), gg.targets.size(), &e->mg));
    };
  }
  GraphLease(const GraphLease&) = delete;
  GraphLease& operator=(const GraphLease&) = delete;
  tg_ctx* ctx() const { return e_->ctxs[0]; }
  size_t devices() const { return e_->ctxs.size(); }
  const tg_graph* graph() {
    if (!e_->g) upload_(e_.get(), host_);
    return e_->g;
  }
  tg_mgraph* partitioned() {
    if (!e_->mg) mupload_(e_.get(), host_);
    return e_->mg;
  }
  tg_sampler* sampler() {
    if (!e_->sampler) check(tg_sampler_create(ctx(), graph(), &e_->sampler));
    return e_->sampler;
  }
  CachedGraph* entry() { return e_.get(); }

 private:
  std::shared_ptr<CachedGraph> e_;
  std::unique_lock<std::mutex> lk_;
  const void* host_;
  void (*upload_)(CachedGraph*, const void*);
  void (*mupload_)(CachedGraph*, const void*);
};

template <class T>
const T* nonnull(const std::vector<T>& v) {
  static const T kZero{};
  return v.empty() ? &kZero : v.data();
}

}  // namespace tiergraph::b200
