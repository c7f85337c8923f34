// The tiered store's state, shared by tiering.cu (placement, K8) and io.cu
// (placement straight from a FEAT file).
#pragma once
#include <cstdint>
#include <initializer_list>

#include "internal.cuh"

struct tg_store {
  tg_ctx* ctx = nullptr;
  tg_layout L{};
  uint32_t dev = 0;
  uint32_t flags = 0;
  uint64_t R = 0;
  uint64_t local_rows = 0;
  uint8_t* local = nullptr;                       // device
  const uint8_t* inter[TG_MAX_DEVICES] = {};      // per-device interleaved slice base
  uint8_t* cold_host = nullptr;                   // host view (owned when own_cold)
  const uint8_t* cold_dev = nullptr;              // device view of the cold tier
  uint64_t cold_stride = 0;
  // TG_COLD_SPLIT_TAIL: the host row holds cold_head bytes (whole 128 B
  // lines); the remaining R - cold_head bytes of each cold row sit in HBM
  uint64_t cold_head = 0;                         // 0: the whole row is in host memory
  uint8_t* cold_tail = nullptr;                   // device, (N-mb) x (R - cold_head)
  bool own_cold_tail = false;
  bool own_cold = false;
  bool cold_attached = false;                     // cold_host is caller memory (tg_store_attach_cold)
  bool cold_fill = true;                          // ... and this store writes the cold rows
  void* registered = nullptr;                     // caller matrix registered for INDIRECT
  uint32_t* cold_src = nullptr;                   // INDIRECT: cold slot -> original row
  bool own_cold_src = false;
  const tg_store* cold_owner = nullptr;
  bool placed = false;
  uint64_t* counters = nullptr;                   // device: 3 x u64 + err
  uint64_t* result_host = nullptr;                // mapped pinned: the counters read back
  uint64_t* result_dev = nullptr;                 // its device address
  uint64_t fin_seq = 0;                           // sequence number of the last synchronous gather
};

namespace tgb {
// Widest vector the row size and every base/stride allow.
int vec_width(uint64_t R, std::initializer_list<uint64_t> addrs);
// Validates a device permutation (reorder.cpp:10-21 messages); inv_dev may be null.
void check_permutation(tg_ctx* ctx, const uint64_t* perm_dev, uint64_t n, uint32_t* inv_dev);
// The reordered (own, pinned, mapped) cold tier of the store, allocated on
// first use; returns its device address.
const uint8_t* ensure_cold_tier(tg_store* s);
}  // namespace tgb

struct tg_graph;
namespace tgb {
// A tg_graph from device offsets (u64, validated + narrowed here) and
// targets already narrowed to u32 and range-checked (ownership taken).
void graph_from_device(tg_ctx* ctx, const uint64_t* off64_dev, uint32_t* tgt32_dev, uint64_t n,
                       uint64_t e, tg_graph** out);
}  // namespace tgb
