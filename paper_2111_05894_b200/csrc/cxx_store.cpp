// cxx_store.cpp — TieredFeatureStore (include/tiergraph/tiered_store.hpp):
// one tg_store per layout device, peers wired to each other's HBM slices,
// one shared pinned cold tier. Compiles against either header set.
#include <string>
#include <vector>

#include "cxx_common.hpp"
#include "tg_capi.h"
#include "tiergraph/tiered_store.hpp"

namespace tiergraph {

struct TieredFeatureStore::Impl {
  TierLayout layout;
  std::vector<int> devices;
  std::vector<tg_ctx*> ctxs;
  std::vector<tg_store*> stores;

  ~Impl() {
    for (size_t d = stores.size(); d-- > 0;) tg_store_destroy(stores[d]);
    for (tg_ctx* c : ctxs) tg_ctx_destroy(c);
  }
};

TieredFeatureStore::TieredFeatureStore(const FeatureMatrix& features, const NodePermutation& perm,
                                       const TierLayout& layout, std::vector<int> devices,
                                       TieredStoreOptions opts)
    : impl_(new Impl) {
  validate_layout(layout);
  const std::uint64_t want = features.num_rows * features.dim * features.elem_bytes;
  if (features.data.size() != want)
    throw FormatError("features: data holds " + std::to_string(features.data.size()) +
                      " bytes, expected " + std::to_string(want));
  if (features.num_rows != layout.num_rows ||
      features.row_bytes() != layout.bytes_per_row())
    throw DomainError("tiered store: feature matrix does not match the layout");
  if (perm.size() != layout.num_rows)
    throw DomainError("permutation length " + std::to_string(perm.size()) + " != num_rows " +
                      std::to_string(layout.num_rows));
  const std::uint32_t D = layout.num_devices;
  if (devices.empty()) {
    // layout device d -> CUDA ordinal; with fewer GPUs than layout devices the
    // slices share GPUs (the peer path then reads same-GPU memory).
    const int visible = tg_device_count();
    const int first = tg_default_device();
    for (std::uint32_t d = 0; d < D; ++d) devices.push_back((first + static_cast<int>(d)) % visible);
  }
  if (devices.size() != D)
    throw DomainError("tiered store: " + std::to_string(devices.size()) +
                      " CUDA devices given for a layout of " + std::to_string(D));
  Impl& m = *impl_;
  m.layout = layout;
  m.devices = devices;
  for (std::uint32_t a = 0; a < D; ++a)
    for (std::uint32_t b = 0; b < D; ++b)
      if (devices[a] != devices[b]) b200::check(tg_enable_peer_access(devices[a], devices[b]));
  const tg_layout l{layout.num_rows, layout.local_boundary, layout.multi_boundary,
                    layout.num_devices, layout.feature_dim, layout.elem_bytes};
  const std::uint32_t flags = (opts.cold_indirect ? TG_COLD_INDIRECT : TG_COLD_REORDERED) |
                              (opts.pad128 ? TG_COLD_PAD128 : 0u) |
                              (opts.split_tail ? TG_COLD_SPLIT_TAIL : 0u) |
                              (opts.bulk ? TG_GATHER_BULK : 0u) |
                              (opts.spread ? TG_GATHER_SPREAD : 0u) |
                              (opts.dynamic ? TG_GATHER_DYNAMIC : 0u);
  static const std::uint64_t kNoRow = 0;
  static const std::uint8_t kNoByte = 0;
  const void* src = features.data.empty() ? &kNoByte : features.data.data();
  const std::uint64_t* p = perm.new_id_of.empty() ? &kNoRow : perm.new_id_of.data();
  for (std::uint32_t d = 0; d < D; ++d) {
    tg_ctx* c = nullptr;
    b200::check(tg_ctx_create(devices[d], &c));
    m.ctxs.push_back(c);
    tg_store* s = nullptr;
    b200::check(tg_store_create(c, &l, d, flags, &s));
    m.stores.push_back(s);
    // K7: device 0 also fills the cold tier; the others map it
    if (d > 0) b200::check(tg_store_share_cold(s, m.stores[0]));
    b200::check(tg_store_place(s, src, p));
  }
  for (std::uint32_t d = 0; d < D; ++d)
    for (std::uint32_t q = 0; q < D; ++q)
      if (q != d) b200::check(tg_store_set_peer(m.stores[d], q, tg_store_local_base(m.stores[q])));
}

TieredFeatureStore::~TieredFeatureStore() = default;

void TieredFeatureStore::gather_rows(std::span<const std::uint64_t> ids, std::uint32_t device,
                                     void* dst, TrafficReport& report) {
  const TierLayout& L = impl_->layout;
  if (device >= L.num_devices)
    throw DomainError("requesting device " + std::to_string(device) + " out of range for " +
                      std::to_string(L.num_devices) + " devices");
  if (ids.empty()) return;
  tg_report r{report.local_accesses, report.peer_accesses, report.host_accesses,
              report.local_bytes, report.peer_bytes, report.host_bytes};
  const int rc = tg_gather_rows(impl_->stores[device], ids.data(), ids.size(), dst, &r);
  report.local_accesses = r.local_accesses;
  report.peer_accesses = r.peer_accesses;
  report.host_accesses = r.host_accesses;
  report.local_bytes = r.local_bytes;
  report.peer_bytes = r.peer_bytes;
  report.host_bytes = r.host_bytes;
  b200::check(rc);
}

const TierLayout& TieredFeatureStore::layout() const { return impl_->layout; }
std::uint64_t TieredFeatureStore::row_bytes() const { return impl_->layout.bytes_per_row(); }
int TieredFeatureStore::cuda_device(std::uint32_t d) const { return impl_->devices.at(d); }

}  // namespace tiergraph
