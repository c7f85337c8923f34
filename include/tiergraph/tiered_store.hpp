// tiered_store.hpp — the byte-moving tiered feature gather (B200 addition).
//
// The reference places rows into a simulated three-tier memory and its
// gather() only counts bytes (proj/src/tiering.cpp:100-125). This class is
// the real thing the paper describes (Listing 1 at
// PAPER.md:683-709): rows are placed by the reference's address map
// (resolve(), tiering.cpp:48-65) into
//   * [0, lb)   — replicated into the HBM of every device,
//   * [lb, mb)  — interleaved: row r on device (r-lb) % D, slot (r-lb) / D,
//                 read by the other devices with direct NVLink peer loads,
//   * [mb, N)   — pinned, mapped host memory read by UVA zero-copy,
// and gather_rows() copies a minibatch's rows into one contiguous buffer with
// accounting identical to gather(layout, ids, device, report).
//
// Only uses types that exist in the reference headers, so it compiles against
// either header set (see tiergraph.hpp).
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "tiergraph/reorder.hpp"
#include "tiergraph/tiering.hpp"

namespace tiergraph {

struct TieredStoreOptions {
  // Cold tier format: a pinned copy in new-id order (default), or the caller's
  // ORIGINAL matrix registered in place and indexed through the inverse
  // permutation (no second host copy, PAPER.md:659-668 cudaHostRegister).
  bool cold_indirect = false;
  // Pad cold rows to a 128-byte stride (whole PCIe read requests).
  bool pad128 = true;
  // Rows whose size is not a multiple of 128 B: keep each cold row's whole
  // 128 B lines in host memory and the remainder in HBM (one PCIe read
  // request fewer per cold row: C2's 400 B rows read as 384 + 16).
  bool split_tail = true;
  // K8 through TMA bulk copies staged in shared memory (else 16 B loads).
  bool bulk = true;
  // Deal consecutive row batches across CTAs, so the cold (PCIe) rows, taken
  // first, are issued from every SM (address translation of a large host
  // region is per-SM limited: 148 -> 89 us per C3 minibatch).
  bool spread = true;
  // After the first (spread) round, warps claim row batches from a device
  // counter, so warps waiting on cold (PCIe) batches hold no HBM batches
  // behind them (C3 minibatch 91.5 -> 83.4 us).
  bool dynamic = true;
};

class TieredFeatureStore {
 public:
  // `features` in ORIGINAL (old-id) order; `perm` = permutation_from_scores;
  // `devices` = CUDA ordinals of the layout's devices 0..D-1 (default: the
  // first D of TIERGRAPH_DEVICES / the visible devices). Peer access is
  // enabled between all of them.
  TieredFeatureStore(const FeatureMatrix& features, const NodePermutation& perm,
                     const TierLayout& layout, std::vector<int> devices = {},
                     TieredStoreOptions opts = {});
  ~TieredFeatureStore();
  TieredFeatureStore(const TieredFeatureStore&) = delete;
  TieredFeatureStore& operator=(const TieredFeatureStore&) = delete;

  // Copy rows `ids` (NEW ids) as seen from layout device `device` into dst
  // (ids.size() x row_bytes; host or device memory) and accumulate the same
  // counters as gather(layout(), ids, device, report). An out-of-range id
  // throws DomainError after the ids before it were accounted.
  void gather_rows(std::span<const std::uint64_t> ids, std::uint32_t device, void* dst,
                   TrafficReport& report);

  const TierLayout& layout() const;
  std::uint64_t row_bytes() const;
  // CUDA ordinal serving layout device d.
  int cuda_device(std::uint32_t d) const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

}  // namespace tiergraph
