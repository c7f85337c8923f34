// cxx_common.hpp — shared plumbing of the C++ drop-in layer (cxx_*.cpp).
//
// Error mapping (C-ABI code -> the reference exception class, types.hpp:13-29)
// and a process-wide pool of device contexts: the reference API is free
// functions on value types and is safe to call from several threads at once
// (SPEC.md:97), so each call leases a tg_ctx (stream + scratch) of its own
// instead of sharing one.
#pragma once

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

template <class T>
const T* nonnull(const std::vector<T>& v) {
  static const T kZero{};
  return v.empty() ? &kZero : v.data();
}

}  // namespace tiergraph::b200
