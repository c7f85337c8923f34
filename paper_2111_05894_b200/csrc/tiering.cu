// Hot path B: the tier address map, placement (K7), the tiered feature gather
// (K8) and the reference's byte accounting, plus the trace replays.
//
// Reference: proj/src/tiering.cpp (resolve :48-65, plan_layout :67-98,
// gather :100-125, simulate_trace :127-162, counts_in_row_order :164-175,
// hot_fraction_sweep :177-202) and the byte-moving gather the paper describes
// (PAPER.md:683-709 Listing 1, :346-353): a per-row pointer from a small table
// {local HBM, peer HBM slices, pinned host}, chosen by comparing the row id to
// the hot boundaries.
//
// Address map (resolve): row r < lb            -> local replicated row r
//                        lb <= r < mb          -> device (r-lb)%D, slot (r-lb)/D
//                        r >= mb               -> cold row r-mb (pinned host)
// Each device's HBM region holds its lb replicated rows followed by its slice
// of the interleaved rows. Peers' slices are read by direct loads through
// peer pointers (same process, cudaDeviceEnablePeerAccess) or CUDA-IPC
// mappings (one process per GPU); cold rows by UVA zero-copy loads.
//
// K8 copies rows with 16-byte vector loads: a warp takes a batch of B rows
// (B*R/16 <= 256 chunks), resolves one row per lane, then every lane issues
// up to 8 independent 16 B loads before storing them, so each warp keeps
// ~4 KB in flight — the queue depth the PCIe zero-copy path needs.
#include <cuda_runtime.h>
#include <errno.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstring>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <chrono>
#include <map>
#include <mutex>
#include <string>

#include "internal.cuh"

#include "store_internal.cuh"

namespace tgb {

// --------------------------------------------------------------- host logic
void validate_layout(const tg_layout& l) {  // tiering.cpp:10-18
  if (l.num_devices < 1) domain_error("layout: num_devices must be >= 1");
  if (l.local_boundary > l.multi_boundary || l.multi_boundary > l.num_rows)
    domain_error("layout: need 0 <= local_boundary <= multi_boundary <= num_rows, got " +
                 std::to_string(l.local_boundary) + ", " + std::to_string(l.multi_boundary) +
                 ", " + std::to_string(l.num_rows));
}

tg_layout plan_layout(uint64_t num_rows, double hot, double rep, uint32_t devices, uint64_t dim,
                      uint32_t eb, uint64_t budget) {  // tiering.cpp:67-98
  if (!(rep >= 0.0 && rep <= hot && hot <= 1.0))
    domain_error("plan_layout: need 0 <= replicated_fraction <= hot_fraction <= 1");
  if (devices < 1) domain_error("plan_layout: num_devices must be >= 1");
  tg_layout l{};
  l.num_rows = num_rows;
  l.local_boundary = static_cast<uint64_t>(std::llround(rep * static_cast<double>(num_rows)));
  l.multi_boundary = static_cast<uint64_t>(std::llround(hot * static_cast<double>(num_rows)));
  l.num_devices = devices;
  l.feature_dim = dim;
  l.elem_bytes = eb;
  validate_layout(l);
  if (budget > 0) {
    const uint64_t inter = l.multi_boundary - l.local_boundary;
    const uint64_t per_dev = l.local_boundary + (inter + devices - 1) / devices;
    const uint64_t required = per_dev * (dim * eb);
    if (required > budget)
      domain_error("layout needs " + std::to_string(required) +
                   " bytes per device but the budget is " + std::to_string(budget));
  }
  return l;
}

void range_error(const tg_layout& l, uint64_t row) {  // tiering.cpp:50-52
  domain_error("row " + std::to_string(row) + " out of range for " + std::to_string(l.num_rows) +
               " rows");
}
void device_error(const tg_layout& l, uint32_t dev) {  // tiering.cpp:53-55
  domain_error("requesting device " + std::to_string(dev) + " out of range for " +
               std::to_string(l.num_devices) + " devices");
}

// ------------------------------------------------------------ device resolve
struct TierMap {
  uint64_t lb, mb, nrows;
  uint32_t D, dev;
};

// 0 local (replicated, or interleaved on the requesting device), 1 peer, 2 host, 3 invalid.
__device__ __forceinline__ int tier_of(const TierMap& m, uint64_t id, uint32_t* owner,
                                       uint64_t* slot) {
  if (id >= m.nrows) return 3;
  if (id < m.lb) {
    *slot = id;
    return 0;
  }
  if (id < m.mb) {
    const uint64_t off = id - m.lb;
    uint32_t d;
    uint64_t s;
    if (m.D == 1) {
      d = 0;
      s = off;
    } else if (off < 0xffffffffull) {  // 32-bit divide is far cheaper
      const uint32_t o = static_cast<uint32_t>(off);
      d = o % m.D;
      s = o / m.D;
    } else {
      d = static_cast<uint32_t>(off % m.D);
      s = off / m.D;
    }
    *owner = d;
    *slot = s;
    return d == m.dev ? 0 : 1;
  }
  *slot = id - m.mb;
  return 2;
}

__device__ __forceinline__ void block_add_counters(uint64_t cl, uint64_t cp, uint64_t ch,
                                                   uint64_t* counters) {
  __shared__ unsigned long long sc[3];
  if (threadIdx.x < 3) sc[threadIdx.x] = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    if (cl) atomicAdd(&sc[0], (unsigned long long)cl);
    if (cp) atomicAdd(&sc[1], (unsigned long long)cp);
    if (ch) atomicAdd(&sc[2], (unsigned long long)ch);
  }
  __syncthreads();
  if (threadIdx.x < 3 && sc[threadIdx.x])
    atomicAdd(reinterpret_cast<unsigned long long*>(counters) + threadIdx.x, sc[threadIdx.x]);
}

// tiering.cpp:100-125 gather(): accounting only, one id per thread.
__global__ void __launch_bounds__(256) account_kernel(TierMap m, const uint64_t* __restrict__ ids,
                                                      uint64_t n, uint64_t* counters,
                                                      unsigned long long* err) {
  uint64_t cl = 0, cp = 0, ch = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t owner;
    uint64_t slot;
    const int t = tier_of(m, ids[i], &owner, &slot);
    if (t == 3) atomicMin(err, (unsigned long long)i);
    cl += t == 0;
    cp += t == 1;
    ch += t == 2;
  }
  // warp reduce then block
  for (int o = 16; o; o >>= 1) {
    cl += __shfl_xor_sync(0xffffffffu, cl, o);
    cp += __shfl_xor_sync(0xffffffffu, cp, o);
    ch += __shfl_xor_sync(0xffffffffu, ch, o);
  }
  block_add_counters(cl, cp, ch, counters);
}

// ------------------------------------------------------------- row copies
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_l2pf_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// PF: ask L2 to fetch the surrounding 256 B sector group (TG_GATHER_L2PF).
template <typename V, bool PF = false>
__device__ __forceinline__ V ld_row(const V* p) {
  return *p;
}
template <>
__device__ __forceinline__ uint4 ld_row<uint4, false>(const uint4* p) {
  return ld_stream_v4(p);
}
template <>
__device__ __forceinline__ uint4 ld_row<uint4, true>(const uint4* p) {
  return ld_l2pf_v4(p);
}

constexpr int kCopyChunks = 256;            // chunks per warp batch (8 per lane)
constexpr int kCopyPerLane = kCopyChunks / 32;

// Copies a batch of B rows: src[j]/dst[j] held by lane j (j < B, nullptr =
// skip). C = row_bytes / sizeof(V) chunks per row; B*C <= kCopyChunks.
// tail/Hc: a split cold row's chunks [Hc, C) come from `tail` (per lane, or null).
template <typename V, bool PF = false>
__device__ __forceinline__ void copy_batch(const uint8_t* src, uint8_t* dst, uint32_t B,
                                           uint32_t C, int lane, const uint8_t* tail = nullptr,
                                           uint32_t Hc = 0) {
  const uint32_t total = B * C;
  V buf[kCopyPerLane];
  const V* sp[kCopyPerLane];
  V* dp[kCopyPerLane];
#pragma unroll
  for (int u = 0; u < kCopyPerLane; ++u) {
    const uint32_t idx = lane + 32u * u;
    const uint32_t row = idx < total ? idx / C : 0;
    const uint32_t ch = idx - row * C;
    const uint8_t* s = reinterpret_cast<const uint8_t*>(
        __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src), row));
    uint8_t* d = reinterpret_cast<uint8_t*>(
        __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(dst), row));
    const uint8_t* tl = reinterpret_cast<const uint8_t*>(
        __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(tail), row));
    const bool ok = idx < total && s != nullptr;
    sp[u] = !ok ? nullptr
                : (tl && ch >= Hc) ? reinterpret_cast<const V*>(tl) + (ch - Hc)
                                   : reinterpret_cast<const V*>(s) + ch;
    dp[u] = ok ? reinterpret_cast<V*>(d) + ch : nullptr;
  }
#pragma unroll
  for (int u = 0; u < kCopyPerLane; ++u)
    if (sp[u]) buf[u] = ld_row<V, PF>(sp[u]);
#pragma unroll
  for (int u = 0; u < kCopyPerLane; ++u)
    if (dp[u]) *dp[u] = buf[u];
}

// Large rows (C > kCopyChunks): one row per warp, looped.
template <typename V>
__device__ __forceinline__ void copy_row_looped(const uint8_t* src, uint8_t* dst, uint64_t C,
                                                int lane, const uint8_t* tail = nullptr,
                                                uint64_t Hc = 0) {
  const V* s = reinterpret_cast<const V*>(src);
  const V* tl = reinterpret_cast<const V*>(tail);
  V* d = reinterpret_cast<V*>(dst);
  for (uint64_t c0 = 0; c0 < C; c0 += kCopyChunks) {
    V buf[kCopyPerLane];
#pragma unroll
    for (int u = 0; u < kCopyPerLane; ++u) {
      const uint64_t c = c0 + lane + 32u * u;
      if (c < C) buf[u] = ld_row<V>((tl && c >= Hc) ? tl + (c - Hc) : s + c);
    }
#pragma unroll
    for (int u = 0; u < kCopyPerLane; ++u) {
      const uint64_t c = c0 + lane + 32u * u;
      if (c < C) d[c] = buf[u];
    }
  }
}

struct GatherTable {
  TierMap m;
  const uint8_t* local;
  const uint8_t* inter[TG_MAX_DEVICES];
  const uint8_t* cold;
  const uint32_t* cold_src;
  const uint8_t* cold_tail;  // TG_COLD_SPLIT_TAIL: bytes [cold_head, R) of cold rows, in HBM
  uint64_t R;
  uint64_t cold_stride;
  uint64_t cold_head;
  // synchronous C-ABI path: the last CTA to finish copies {counters, err} to
  // mapped pinned host memory and re-arms them (no memset / D2H copy calls)
  uint64_t* fin_host;
  unsigned* fin_done;
  uint64_t fin_seq;  // written to fin_host[4] last: the host's "this call is done" flag
  // TG_GATHER_DYNAMIC: after the first (statically spread) round, warps claim
  // batches from this counter, so a warp waiting on a cold (PCIe) batch does
  // not hold HBM batches behind it; the last CTA re-arms it
  unsigned long long* claim;
  unsigned* claim_done;
};

__device__ __forceinline__ void claim_finalize(const GatherTable& t) {
  if (!t.claim) return;
  __syncthreads();  // every warp of this CTA has made its last claim
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(t.claim_done, 1u) == gridDim.x - 1) {
      *reinterpret_cast<volatile unsigned long long*>(t.claim) = 0ull;
      *reinterpret_cast<volatile unsigned*>(t.claim_done) = 0u;
      __threadfence();
    }
  }
}

__device__ __forceinline__ void gather_finalize(const GatherTable& t, uint64_t* counters,
                                                unsigned long long* err) {
  if (!t.fin_host) return;
  __syncthreads();  // this CTA's counter atomics are issued
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned ticket = atomicAdd(t.fin_done, 1u);
    if (ticket == gridDim.x - 1) {
      __threadfence();
      volatile uint64_t* c = counters;
      volatile unsigned long long* e = err;
      volatile uint64_t* h = t.fin_host;
      h[0] = c[0];
      h[1] = c[1];
      h[2] = c[2];
      h[3] = e[0];
      c[0] = 0;
      c[1] = 0;
      c[2] = 0;
      e[0] = ~0ull;
      *reinterpret_cast<volatile unsigned*>(t.fin_done) = 0u;
      __threadfence_system();
      h[4] = t.fin_seq;  // every CTA's rows and the counters above are out
      __threadfence_system();
    }
  }
}

// *tail: for a split cold row, where its bytes [cold_head, R) live (else null)
__device__ __forceinline__ const uint8_t* row_ptr(const GatherTable& t, uint64_t id, int* tier,
                                                  const uint8_t** tail) {
  uint32_t owner = 0;
  uint64_t slot = 0;
  const int k = tier_of(t.m, id, &owner, &slot);
  *tier = k;
  *tail = nullptr;
  if (k == 3) return nullptr;
  if (id < t.m.lb) return t.local + slot * t.R;
  if (k == 2) {
    const uint64_t row = t.cold_src ? t.cold_src[slot] : slot;
    if (t.cold_tail) *tail = t.cold_tail + row * (t.R - t.cold_head);
    return t.cold + row * t.cold_stride;
  }
  return t.inter[owner] + slot * t.R;
}

// K8: the tiered gather. dst row i <- feature row ids[i].
template <typename V, bool PF = false>
__global__ void __launch_bounds__(256) gather_kernel(GatherTable t, const uint64_t* __restrict__ ids,
                                                     uint64_t n, uint8_t* __restrict__ dst,
                                                     uint32_t B, uint32_t C, uint64_t* counters,
                                                     unsigned long long* err, uint32_t spread) {
  const int lane = threadIdx.x & 31;
  // spread: consecutive batches go to different CTAs (so the cold batches,
  // taken first, are issued from every SM rather than the first few CTAs)
  const uint64_t warp = spread ? (threadIdx.x >> 5) * (uint64_t)gridDim.x + blockIdx.x
                               : (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t cl = 0, cp = 0, ch = 0;
  // Batches run from the END of the id list: minibatch lists are sorted, so
  // the cold (highest) ids go first and their PCIe latency overlaps the
  // HBM-resident rows that follow.
  const uint64_t nb = (n + B - 1) / B;
  for (uint64_t k = warp; k < nb; k += nwarps) {
    const uint64_t b0 = (nb - 1 - k) * B;
    const uint8_t* src = nullptr;
    const uint8_t* tail = nullptr;
    uint8_t* d = nullptr;
    int tier = -1;
    if (lane < (int)B && b0 + lane < n) {
      src = row_ptr(t, ids[b0 + lane], &tier, &tail);
      if (tier == 3) atomicMin(err, (unsigned long long)(b0 + lane));
      else d = dst + (b0 + lane) * t.R;
    }
    cl += __popc(__ballot_sync(0xffffffffu, tier == 0));
    cp += __popc(__ballot_sync(0xffffffffu, tier == 1));
    ch += __popc(__ballot_sync(0xffffffffu, tier == 2));
    const uint32_t Hc = static_cast<uint32_t>(t.cold_head / sizeof(V));
    if (C <= (uint32_t)kCopyChunks) {
      copy_batch<V, PF>(src, d, B, C, lane, tail, Hc);
    } else {
      for (uint32_t j = 0; j < B; ++j) {
        const uint8_t* s = reinterpret_cast<const uint8_t*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src), j));
        const uint8_t* tl = reinterpret_cast<const uint8_t*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(tail), j));
        uint8_t* o = reinterpret_cast<uint8_t*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(d), j));
        if (s) copy_row_looped<V>(s, o, C, lane, tl, Hc);
      }
    }
  }
  if (lane != 0) cl = cp = ch = 0;
  block_add_counters(cl, cp, ch, counters);
  gather_finalize(t, counters, err);
}

// K8, TMA bulk-copy variant (TG_GATHER_BULK): each warp stages a batch of
// rows in shared memory with one cp.async.bulk per row (global/host-mapped ->
// smem, completion on an mbarrier), then writes them out with bulk stores
// (smem -> HBM). The copy engine issues whole-row requests, which is what
// the PCIe zero-copy path prefers. Two staging buffers per warp: the loads of
// batch k+1 are in flight while batch k drains.
constexpr int kBulkWarps = 8;
constexpr int kBulkStage = 6144;  // bytes per staging buffer (x2 per warp)

__device__ __forceinline__ void bulk_g2s(uint32_t smem_dst, const void* src, uint32_t bytes,
                                         uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_dst), "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_init_s(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
               ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAITB_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITB_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(kBulkWarps * 32) gather_bulk_kernel(
    GatherTable t, const uint64_t* __restrict__ ids, uint64_t n, uint8_t* __restrict__ dst,
    uint32_t B, uint32_t Rpad, uint64_t* counters, unsigned long long* err, uint32_t spread) {
  extern __shared__ __align__(128) uint8_t bulk_smem[];  // [warps][2][kBulkStage]
  __shared__ __align__(8) uint64_t bars[kBulkWarps][2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(&bars[w][0]));
  const uint32_t bar1 = static_cast<uint32_t>(__cvta_generic_to_shared(&bars[w][1]));
  const uint32_t s0 =
      static_cast<uint32_t>(__cvta_generic_to_shared(bulk_smem + (2 * w) * kBulkStage));
  const uint32_t s1 = s0 + kBulkStage;
  if (lane == 0) {
    mbar_init_s(bar0, 1);
    mbar_init_s(bar1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint64_t warp = spread ? (uint64_t)w * gridDim.x + blockIdx.x
                               : (uint64_t)blockIdx.x * kBulkWarps + w;
  const uint64_t nwarps = (uint64_t)gridDim.x * kBulkWarps;
  const uint64_t nb = (n + B - 1) / B;
  const uint32_t R = static_cast<uint32_t>(t.R);
  uint64_t cl = 0, cp = 0, ch = 0;
  uint32_t phase[2] = {0, 0};
  // in-flight batch state (one per buffer)
  int buf = 0;
  // the next batch's ids are loaded one batch ahead (ids may sit in host
  // memory, read in place: their PCIe latency then overlaps this batch)
  auto id_of = [&](uint64_t k) -> uint64_t {
    const uint64_t i = (nb - 1 - k) * B + lane;
    return (k < nb && lane < (int)B && i < n) ? ids[i] : 0ull;
  };
  // first round static (spread over the SMs: it holds the cold batches of a
  // sorted list), then dynamic claims (TG_GATHER_DYNAMIC) or the static stride
  auto next_of = [&](uint64_t k) -> uint64_t {
    if (!t.claim) return k + nwarps;
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(t.claim, 1ull);
    return nwarps + __shfl_sync(0xffffffffu, c, 0);
  };
  uint64_t k_next = warp;
  uint64_t id_next = id_of(k_next);
  while (k_next < nb) {
    const uint64_t k = k_next;
    const uint64_t b0 = (nb - 1 - k) * B;  // cold (highest ids) first
    const uint64_t id = id_next;
    k_next = next_of(k);
    id_next = id_of(k_next);
    const uint32_t bar = buf ? bar1 : bar0;
    const uint32_t sb = buf ? s1 : s0;
    // the buffer we are about to fill was stored from two batches ago
    bulk_wait_read<1>();
    __syncwarp();
    const uint8_t* src = nullptr;
    const uint8_t* tail = nullptr;
    int tier = -1;
    if (lane < (int)B && b0 + lane < n) {
      src = row_ptr(t, id, &tier, &tail);
      if (tier == 3) atomicMin(err, (unsigned long long)(b0 + lane));
    }
    cl += __popc(__ballot_sync(0xffffffffu, tier == 0));
    cp += __popc(__ballot_sync(0xffffffffu, tier == 1));
    ch += __popc(__ballot_sync(0xffffffffu, tier == 2));
    const uint32_t nrows = __popc(__ballot_sync(0xffffffffu, src != nullptr));
    if (lane == 0) mbar_expect_tx(bar, nrows * R);
    __syncwarp();
    if (tail) {  // split cold row: whole lines over PCIe, the remainder from HBM
      const uint32_t H = static_cast<uint32_t>(t.cold_head);
      bulk_g2s(sb + lane * Rpad, src, H, bar);
      bulk_g2s(sb + lane * Rpad + H, tail, R - H, bar);
    } else if (src) {
      bulk_g2s(sb + lane * Rpad, src, R, bar);
    }
    // drain the OTHER buffer's batch (issued last iteration) while this one loads
    mbar_wait_s(bar, phase[buf]);
    phase[buf] ^= 1;
    if (src) bulk_s2g(dst + (b0 + lane) * t.R, sb + lane * Rpad, R);
    bulk_commit();
    buf ^= 1;
  }
  bulk_wait_read<0>();
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (lane != 0) cl = cp = ch = 0;
  block_add_counters(cl, cp, ch, counters);
  gather_finalize(t, counters, err);
  claim_finalize(t);
}

// Generic row mover: dst + dst_row(i)*dst_stride <- src + src_row(i)*src_stride
// with the rows named by optional u64/u32 index arrays. Used for placement
// (K7: hot slots and the cold copy) and reorder_features.
struct MoveArgs {
  const uint8_t* src;
  uint8_t* dst;
  uint64_t src_stride, dst_stride;
  const uint32_t* src_idx32;  // src row = src_idx32[i] (else i)
  const uint64_t* dst_idx64;  // dst row = dst_idx64[i] (else i)
  uint64_t src_row_base;      // added to i before src_idx32 lookup
  uint32_t slot_mode;         // 1: src row index from slot i of a store (see below)
  uint64_t lb;
  uint32_t D, dev;
};

__device__ __forceinline__ uint64_t store_slot_row(uint64_t s, uint64_t lb, uint32_t D,
                                                   uint32_t dev) {
  return s < lb ? s : lb + (s - lb) * D + dev;
}

template <typename V>
__global__ void __launch_bounds__(256) move_rows_kernel(MoveArgs a, uint64_t n, uint32_t B,
                                                        uint32_t C) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t b0 = warp * B; b0 < n; b0 += nwarps * B) {
    const uint8_t* s = nullptr;
    uint8_t* d = nullptr;
    if (lane < (int)B && b0 + lane < n) {
      const uint64_t i = b0 + lane;
      uint64_t k = a.src_row_base + (a.slot_mode ? store_slot_row(i, a.lb, a.D, a.dev) : i);
      const uint64_t sr = a.src_idx32 ? a.src_idx32[k] : k;
      const uint64_t dr = a.dst_idx64 ? a.dst_idx64[i] : i;
      s = a.src + sr * a.src_stride;
      d = a.dst + dr * a.dst_stride;
    }
    if (C <= (uint32_t)kCopyChunks) {
      copy_batch<V>(s, d, B, C, lane);
    } else {
      for (uint32_t j = 0; j < B; ++j) {
        const uint8_t* ss = reinterpret_cast<const uint8_t*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(s), j));
        uint8_t* dd = reinterpret_cast<uint8_t*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(d), j));
        if (ss) copy_row_looped<V>(ss, dd, C, lane);
      }
    }
  }
}

// Widest vector the row size and every base/stride allow.
int vec_width(uint64_t R, std::initializer_list<uint64_t> addrs) {
  int w = 16;
  while (w > 1) {
    bool ok = R % w == 0;
    for (uint64_t a : addrs) ok = ok && a % w == 0;
    if (ok) break;
    w >>= 1;
  }
  return w;
}

void batch_shape(uint64_t R, int w, uint32_t* B, uint32_t* C) {
  const uint64_t c = R / w;
  *C = static_cast<uint32_t>(c);
  *B = c >= (uint64_t)kCopyChunks ? 1u : static_cast<uint32_t>(std::min<uint64_t>(32, kCopyChunks / c));
}

void launch_move(tg_ctx* ctx, const MoveArgs& a, uint64_t n, uint64_t R) {
  if (n == 0 || R == 0) return;
  const int w = vec_width(R, {reinterpret_cast<uint64_t>(a.src), reinterpret_cast<uint64_t>(a.dst),
                             a.src_stride, a.dst_stride});
  uint32_t B, C;
  batch_shape(R, w, &B, &C);
  const uint64_t warps = (n + B - 1) / B;
  const unsigned grid = grid_for(warps * 32, 256, ctx->num_sms * 16);
  switch (w) {
    case 16: move_rows_kernel<uint4><<<grid, 256, 0, ctx->stream>>>(a, n, B, C); break;
    case 8: move_rows_kernel<uint2><<<grid, 256, 0, ctx->stream>>>(a, n, B, C); break;
    case 4: move_rows_kernel<uint32_t><<<grid, 256, 0, ctx->stream>>>(a, n, B, C); break;
    case 2: move_rows_kernel<uint16_t><<<grid, 256, 0, ctx->stream>>>(a, n, B, C); break;
    default: move_rows_kernel<uint8_t><<<grid, 256, 0, ctx->stream>>>(a, n, B, C); break;
  }
  TGB_LAUNCHED();
}

// ---------------------------------------------------------- permutation util
// Pass 1: seen[v] = the lowest position holding new id v.
__global__ void perm_first_kernel(const uint64_t* __restrict__ p, uint64_t n,
                                  uint32_t* __restrict__ seen) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = p[u];
    if (v < n) atomicMin(&seen[v], static_cast<uint32_t>(u));
  }
}

// Pass 2: position u offends iff p[u] >= n or an earlier position holds p[u]
// -- exactly the positions the reference's sequential scan throws at
// (reorder.cpp:10-21); the minimum of them is its first throw.
__global__ void perm_check_kernel(const uint64_t* __restrict__ p, uint64_t n,
                                  const uint32_t* __restrict__ seen, uint32_t* __restrict__ inv,
                                  unsigned long long* bad) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = p[u];
    if (v >= n || seen[v] != static_cast<uint32_t>(u)) {
      atomicMin(bad, (unsigned long long)u);
      continue;
    }
    if (inv) inv[v] = static_cast<uint32_t>(u);
  }
}

// Validates a permutation (reorder.cpp:10-21) and optionally builds its
// inverse as u32. Throws DomainError naming the offending new id at the
// reference's first offending position.
void check_permutation(tg_ctx* ctx, const uint64_t* perm_dev, uint64_t n, uint32_t* inv_dev) {
  if (n == 0) return;
  if (n >= 0xffffffffull) domain_error("permutation: n must be < 2^32");
  uint32_t* seen = ctx->scratch_t<uint32_t>(kScratchE, n);
  auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 1);
  TGB_CUDA(cudaMemsetAsync(seen, 0xff, n * 4, ctx->stream));
  TGB_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
  perm_first_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(perm_dev, n, seen);
  TGB_LAUNCHED();
  perm_check_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(perm_dev, n, seen, inv_dev, bad);
  TGB_LAUNCHED();
  unsigned long long hb;
  TGB_CUDA(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  if (hb != ~0ull) {
    uint64_t v;
    TGB_CUDA(cudaMemcpy(&v, perm_dev + hb, 8, cudaMemcpyDeviceToHost));
    if (v >= n) domain_error("permutation: new id " + std::to_string(v) + " out of range");
    domain_error("permutation: new id " + std::to_string(v) + " assigned twice");
  }
}

__global__ void u32_to_u64_kernel(const uint32_t* __restrict__ in, uint64_t* __restrict__ out,
                                  uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

// ------------------------------------------------------------ trace replays
__global__ void row_order_kernel(const uint64_t* __restrict__ counts, uint64_t n,
                                 const uint64_t* __restrict__ ordering,
                                 uint64_t* __restrict__ out, unsigned long long* bad) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = ordering[k];
    if (u >= n) {
      atomicMin(bad, (unsigned long long)k);
      out[k] = 0;
    } else {
      out[k] = counts[u];
    }
  }
}

constexpr int kMaxSim = 16;
struct SimLayouts {
  uint64_t lb[kMaxSim], mb[kMaxSim];
  uint32_t D[kMaxSim];
  int count;
};

// tiering.cpp:137-157 for several layouts at once; out[4*f + {local,peer,host}], out[3] total
__global__ void __launch_bounds__(256) simulate_kernel(const uint64_t* __restrict__ counts, uint64_t n,
                                                       SimLayouts L, unsigned long long* out) {
  __shared__ unsigned long long acc[kMaxSim * 3 + 1];
  for (int i = threadIdx.x; i < kMaxSim * 3 + 1; i += blockDim.x) acc[i] = 0;
  __syncthreads();
  uint64_t loc[kMaxSim], peer[kMaxSim], host[kMaxSim], total = 0;
#pragma unroll
  for (int f = 0; f < kMaxSim; ++f) loc[f] = peer[f] = host[f] = 0;
  for (uint64_t row = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; row < n;
       row += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = counts[row];
    if (!c) continue;
    total += c;
#pragma unroll
    for (int f = 0; f < kMaxSim; ++f) {
      if (f >= L.count) break;
      if (row < L.lb[f]) {
        loc[f] += c;
      } else if (row < L.mb[f]) {
        const uint64_t D = L.D[f];
        const uint64_t owner = (row - L.lb[f]) % D;
        const uint64_t l = c / D + (owner < c % D ? 1 : 0);  // tiering.cpp:148
        loc[f] += l;
        peer[f] += c - l;
      } else {
        host[f] += c;
      }
    }
  }
  for (int o = 16; o; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
#pragma unroll
  for (int f = 0; f < kMaxSim; ++f) {
    if (f >= L.count) break;
    for (int o = 16; o; o >>= 1) {
      loc[f] += __shfl_xor_sync(0xffffffffu, loc[f], o);
      peer[f] += __shfl_xor_sync(0xffffffffu, peer[f], o);
      host[f] += __shfl_xor_sync(0xffffffffu, host[f], o);
    }
  }
  if ((threadIdx.x & 31) == 0) {
    for (int f = 0; f < L.count; ++f) {
      if (loc[f]) atomicAdd(&acc[3 * f], (unsigned long long)loc[f]);
      if (peer[f]) atomicAdd(&acc[3 * f + 1], (unsigned long long)peer[f]);
      if (host[f]) atomicAdd(&acc[3 * f + 2], (unsigned long long)host[f]);
    }
    if (total) atomicAdd(&acc[kMaxSim * 3], (unsigned long long)total);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxSim * 3 + 1; i += blockDim.x)
    if (acc[i]) atomicAdd(&out[i], acc[i]);
}

// Runs simulate_trace for each layout over device counts; returns total.
uint64_t simulate_many(tg_ctx* ctx, const uint64_t* counts_dev, uint64_t n,
                       const std::vector<tg_layout>& layouts, std::vector<tg_report>& out) {
  out.assign(layouts.size(), tg_report{});
  uint64_t total = 0;
  auto* acc = ctx->scratch_t<unsigned long long>(kSmall, kMaxSim * 3 + 1);
  for (size_t f0 = 0; f0 < std::max<size_t>(layouts.size(), 1); f0 += kMaxSim) {
    SimLayouts L{};
    L.count = static_cast<int>(std::min<size_t>(kMaxSim, layouts.size() - std::min(f0, layouts.size())));
    for (int f = 0; f < L.count; ++f) {
      L.lb[f] = layouts[f0 + f].local_boundary;
      L.mb[f] = layouts[f0 + f].multi_boundary;
      L.D[f] = layouts[f0 + f].num_devices;
    }
    TGB_CUDA(cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * (kMaxSim * 3 + 1), ctx->stream));
    if (n) {
      simulate_kernel<<<grid_for(n, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(counts_dev, n, L,
                                                                                  acc);
      TGB_LAUNCHED();
    }
    unsigned long long h[kMaxSim * 3 + 1];
    TGB_CUDA(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    total = h[kMaxSim * 3];
    for (int f = 0; f < L.count; ++f) {
      tg_report& r = out[f0 + f];
      const uint64_t rb = layouts[f0 + f].feature_dim * layouts[f0 + f].elem_bytes;
      r.local_accesses = h[3 * f];
      r.peer_accesses = h[3 * f + 1];
      r.host_accesses = h[3 * f + 2];
      r.local_bytes = r.local_accesses * rb;  // tiering.cpp:158-160
      r.peer_bytes = r.peer_accesses * rb;
      r.host_bytes = r.host_accesses * rb;
    }
    if (layouts.empty()) break;
  }
  return total;
}

// Reference-counted cudaHostRegister of caller matrices, so several stores
// (virtual devices, or a store and a later re-placement) can map the same
// host matrix. Memory pinned outside the library is used as is.
std::mutex g_reg_mu;
std::map<void*, std::pair<uint64_t, int>> g_reg;

const uint8_t* acquire_host_matrix(const void* p, uint64_t bytes, bool* owned) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  void* key = const_cast<void*>(p);
  auto it = g_reg.find(key);
  if (it != g_reg.end()) {
    ++it->second.second;
    *owned = true;
  } else if (void* m = mapped_device_ptr(p)) {
    *owned = false;
    return static_cast<const uint8_t*>(m);
  } else {
    TGB_CUDA(cudaHostRegister(key, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    g_reg[key] = {bytes, 1};
    *owned = true;
  }
  void* m = nullptr;
  TGB_CUDA(cudaHostGetDevicePointer(&m, key, 0));
  return static_cast<const uint8_t*>(m);
}

void release_host_matrix(void* p) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  auto it = g_reg.find(p);
  if (it == g_reg.end()) return;
  if (--it->second.second == 0) {
    cudaHostUnregister(p);
    g_reg.erase(it);
  }
}

void add_report(tg_report* r, uint64_t l, uint64_t p, uint64_t h, uint64_t rb) {
  r->local_accesses += l;
  r->peer_accesses += p;
  r->host_accesses += h;
  r->local_bytes += l * rb;
  r->peer_bytes += p * rb;
  r->host_bytes += h * rb;
}

void account(tg_ctx* ctx, const tg_layout& l, const uint64_t* ids_dev, uint64_t n, uint32_t dev,
             uint64_t* counters3, unsigned long long* err) {
  TierMap m{l.local_boundary, l.multi_boundary, l.num_rows, l.num_devices, dev};
  account_kernel<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(m, ids_dev, n,
                                                                              counters3, err);
  TGB_LAUNCHED();
}

// n sorted, distinct random ids in [base, base + span), one per stratum of
// span/n ids (a minibatch list is sorted and unique; measurement only)
__global__ void random_ids_kernel(uint64_t* __restrict__ out, uint64_t n, uint64_t base,
                                  uint64_t span, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + seed * 0x632BE59BD9B4E019ull) * 0x9E3779B97F4A7C15ull;
    x ^= x >> 31;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 29;
    const uint64_t lo = (unsigned __int128)span * i / n, hi = (unsigned __int128)span * (i + 1) / n;
    out[i] = base + lo + (hi > lo ? x % (hi - lo) : 0);
  }
}

GatherTable make_table(const tg_store* s) {
  GatherTable t{};
  t.m = TierMap{s->L.local_boundary, s->L.multi_boundary, s->L.num_rows, s->L.num_devices, s->dev};
  t.local = s->local;
  for (uint32_t d = 0; d < s->L.num_devices; ++d) t.inter[d] = s->inter[d];
  t.cold = s->cold_dev;
  t.cold_src = s->cold_src;
  t.cold_tail = s->cold_head ? s->cold_tail : nullptr;
  t.R = s->R;
  t.cold_stride = s->cold_stride;
  t.cold_head = s->cold_head;
  return t;
}

void launch_gather(tg_store* s, const uint64_t* ids_dev, uint64_t n, void* dst_dev,
                   uint64_t* counters3, unsigned long long* err, bool finalize = false) {
  tg_ctx* ctx = s->ctx;
  if (!s->placed) domain_error("tiered store: tg_store_place has not run");
  const uint64_t inter_rows = s->L.multi_boundary - s->L.local_boundary;
  for (uint32_t d = 0; d < s->L.num_devices && inter_rows > d; ++d)
    if (!s->inter[d]) domain_error("tiered store: peer slice of device " + std::to_string(d) +
                                   " is not attached (tg_store_set_peer)");
  GatherTable t = make_table(s);
  if (finalize) {
    t.fin_host = s->result_dev;
    t.fin_done = reinterpret_cast<unsigned*>(s->counters + 4);
    t.fin_seq = s->fin_seq;
  }
  if (s->flags & TG_GATHER_DYNAMIC) {  // store-owned, zero between launches
    t.claim = reinterpret_cast<unsigned long long*>(s->counters + 5);
    t.claim_done = reinterpret_cast<unsigned*>(s->counters + 6);
  }
  const uint32_t spread = (s->flags & TG_GATHER_SPREAD) ? 1u : 0u;
  uint64_t align = reinterpret_cast<uint64_t>(dst_dev) | reinterpret_cast<uint64_t>(s->local) |
                   reinterpret_cast<uint64_t>(s->cold_dev) | s->cold_stride;
  if (s->cold_head)
    align |= reinterpret_cast<uint64_t>(s->cold_tail) | s->cold_head | (s->R - s->cold_head);
  for (uint32_t d = 0; d < s->L.num_devices; ++d) align |= reinterpret_cast<uint64_t>(s->inter[d]);
  const int w = vec_width(s->R, {align});
  auto* dst = static_cast<uint8_t*>(dst_dev);
  if ((s->flags & TG_GATHER_BULK) && w == 16 && s->R <= (uint64_t)kBulkStage) {
    const uint32_t Rpad = static_cast<uint32_t>(s->R);
    // rows per warp batch: as many as a staging buffer holds, but small
    // enough that a short list still spreads over every SM (each SM's TMA
    // and address translation serve its own batches)
    const uint64_t all_warps = static_cast<uint64_t>(ctx->num_sms) * 2 * kBulkWarps;
    // TIERGRAPH_GATHER_ROWS_PER_WARP caps the batch (experiments)
    static const uint64_t cap_b = [] {
      const char* v = std::getenv("TIERGRAPH_GATHER_ROWS_PER_WARP");
      return v ? std::max<uint64_t>(1, std::strtoull(v, nullptr, 10)) : 32ull;
    }();
    const uint32_t B = static_cast<uint32_t>(std::max<uint64_t>(
        1, std::min<uint64_t>({cap_b, kBulkStage / Rpad, (n + all_warps - 1) / all_warps})));
    const uint64_t warps = (n + B - 1) / B;
    const unsigned grid = grid_for(warps * 32, kBulkWarps * 32, ctx->num_sms * 2);
    constexpr int kSmem = kBulkWarps * 2 * kBulkStage;
    static bool attr[TG_MAX_DEVICES] = {};  // a function attribute is per device
    if (!attr[ctx->device % TG_MAX_DEVICES]) {
      TGB_CUDA(cudaFuncSetAttribute(gather_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSmem));
      attr[ctx->device % TG_MAX_DEVICES] = true;
    }
    gather_bulk_kernel<<<grid, kBulkWarps * 32, kSmem, ctx->stream>>>(t, ids_dev, n, dst, B, Rpad,
                                                                      counters3, err, spread);
    TGB_LAUNCHED();
    return;
  }
  uint32_t B, C;
  batch_shape(s->R, w, &B, &C);
  const uint64_t warps = (n + B - 1) / B;
  const unsigned grid = grid_for(warps * 32, 256, ctx->num_sms * 8);
  if ((s->flags & TG_GATHER_L2PF) && w == 16) {
    gather_kernel<uint4, true><<<grid, 256, 0, ctx->stream>>>(t, ids_dev, n, dst, B, C, counters3, err, spread);
    TGB_LAUNCHED();
    return;
  }
  switch (w) {
    case 16: gather_kernel<uint4><<<grid, 256, 0, ctx->stream>>>(t, ids_dev, n, dst, B, C, counters3, err, spread); break;
    case 8: gather_kernel<uint2><<<grid, 256, 0, ctx->stream>>>(t, ids_dev, n, dst, B, C, counters3, err, spread); break;
    case 4: gather_kernel<uint32_t><<<grid, 256, 0, ctx->stream>>>(t, ids_dev, n, dst, B, C, counters3, err, spread); break;
    case 2: gather_kernel<uint16_t><<<grid, 256, 0, ctx->stream>>>(t, ids_dev, n, dst, B, C, counters3, err, spread); break;
    default: gather_kernel<uint8_t><<<grid, 256, 0, ctx->stream>>>(t, ids_dev, n, dst, B, C, counters3, err, spread); break;
  }
  TGB_LAUNCHED();
}

}  // namespace tgb

using namespace tgb;

extern "C" {

int tg_validate_layout(const tg_layout* layout) {
  return guard([&] { validate_layout(*layout); });
}

int tg_validate_cost_model(double l, double p, double h) {
  return guard([&] {  // tiering.cpp:20-23
    if (!(l > 0.0 && p > 0.0 && h > 0.0)) domain_error("cost model: all bandwidths must be positive");
  });
}

int tg_resolve(const tg_layout* l, uint64_t row, uint32_t dev, tg_location* out) {
  return guard([&] {  // tiering.cpp:48-65
    if (row >= l->num_rows) range_error(*l, row);
    if (dev >= l->num_devices) device_error(*l, dev);
    if (row < l->local_boundary) {
      *out = {TG_TIER_LOCAL_HOT, 0, row};
    } else if (row < l->multi_boundary) {
      const uint64_t off = row - l->local_boundary;
      *out = {TG_TIER_INTERLEAVED, static_cast<uint32_t>(off % l->num_devices), off / l->num_devices};
    } else {
      *out = {TG_TIER_COLD_HOST, 0, row - l->multi_boundary};
    }
  });
}

int tg_plan_layout(uint64_t num_rows, double hot, double rep, uint32_t devices, uint64_t dim,
                   uint32_t eb, uint64_t budget, tg_layout* out) {
  return guard([&] { *out = plan_layout(num_rows, hot, rep, devices, dim, eb, budget); });
}

double tg_report_hit_ratio(const tg_report* r) {  // tiering.cpp:25-29
  const uint64_t total = r->local_accesses + r->peer_accesses + r->host_accesses;
  if (total == 0) return 0.0;
  return 1.0 - static_cast<double>(r->host_accesses) / static_cast<double>(total);
}

double tg_report_est_transfer_seconds(const tg_report* r, double l, double p, double h) {
  constexpr double kGiB = 1e9;  // tiering.cpp:31-36
  return static_cast<double>(r->local_bytes) / (l * kGiB) +
         static_cast<double>(r->peer_bytes) / (p * kGiB) +
         static_cast<double>(r->host_bytes) / (h * kGiB);
}

int tg_gather_account(tg_ctx* ctx, const tg_layout* layout, const uint64_t* ids, uint64_t n,
                      uint32_t dev, tg_report* report) {
  return guard([&] {
    if (n == 0) return;  // the reference loop body never runs
    DeviceGuard dg(ctx->device);
    const uint64_t* d = dev_in(ctx, ids, n, kStageIn0);
    auto* c = ctx->scratch_t<uint64_t>(kSmall, 4);
    auto* err = reinterpret_cast<unsigned long long*>(c + 3);
    TGB_CUDA(cudaMemsetAsync(c, 0, 24, ctx->stream));
    TGB_CUDA(cudaMemsetAsync(err, 0xff, 8, ctx->stream));
    const uint64_t rb = layout->feature_dim * layout->elem_bytes;
    if (dev >= layout->num_devices) {
      // resolve() range-checks the row first, then the device (tiering.cpp:50-55)
      uint64_t id0;
      TGB_CUDA(cudaMemcpy(&id0, d, 8, cudaMemcpyDeviceToHost));
      if (id0 >= layout->num_rows) range_error(*layout, id0);
      device_error(*layout, dev);
    }
    account(ctx, *layout, d, n, dev, c, err);
    uint64_t h[4];
    TGB_CUDA(cudaMemcpyAsync(h, c, 32, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (h[3] != ~0ull) {
      // keep the prefix before the first bad id accounted, then throw
      const uint64_t first = h[3];
      TGB_CUDA(cudaMemsetAsync(c, 0, 24, ctx->stream));
      if (first) account(ctx, *layout, d, first, dev, c, err);
      TGB_CUDA(cudaMemcpyAsync(h, c, 24, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      add_report(report, h[0], h[1], h[2], rb);
      uint64_t bad;
      TGB_CUDA(cudaMemcpy(&bad, d + first, 8, cudaMemcpyDeviceToHost));
      range_error(*layout, bad);
    }
    add_report(report, h[0], h[1], h[2], rb);
  });
}

int tg_simulate_trace(tg_ctx* ctx, const uint64_t* counts, uint64_t n, const tg_layout* layout,
                      tg_report* out) {
  return guard([&] {  // tiering.cpp:127-162
    validate_layout(*layout);
    if (n != layout->num_rows)
      domain_error("counter covers " + std::to_string(n) + " rows but the layout has " +
                   std::to_string(layout->num_rows));
    DeviceGuard dg(ctx->device);
    const uint64_t* c = dev_in(ctx, counts, n, kStageIn0);
    std::vector<tg_report> reps;
    const uint64_t total = simulate_many(ctx, c, n, {*layout}, reps);
    if (total == 0) domain_error("simulate_trace: counter total is zero");
    *out = reps[0];
  });
}

int tg_counts_in_row_order(tg_ctx* ctx, const uint64_t* counts, uint64_t n,
                           const uint64_t* ordering, uint64_t m, uint64_t* out) {
  return guard([&] {  // tiering.cpp:164-175
    if (m != n) domain_error("ordering length != counter length");
    if (n == 0) return;
    DeviceGuard dg(ctx->device);
    const uint64_t* c = dev_in(ctx, counts, n, kStageIn0);
    const uint64_t* o = dev_in(ctx, ordering, n, kStageIn1);
    DevOut<uint64_t> r(ctx, out, n, kStageOut0);
    auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 1);
    TGB_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
    row_order_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(c, n, o, r.dev(), bad);
    TGB_LAUNCHED();
    unsigned long long hb;
    TGB_CUDA(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
    r.finish();
    if (hb != ~0ull) domain_error("ordering id out of range");
  });
}

int tg_hot_fraction_sweep(tg_ctx* ctx, const uint64_t* counts, uint64_t n,
                          const uint64_t* ordering, const double* fr, uint64_t nf,
                          double replicated, uint32_t devices, uint64_t dim, uint32_t eb,
                          uint64_t budget, tg_layout* out_layouts, tg_report* out_reports,
                          double* out_rep) {
  return guard([&] {  // tiering.cpp:177-202
    for (uint64_t i = 1; i < nf; ++i)
      if (fr[i] < fr[i - 1]) domain_error("sweep fractions must be sorted ascending");
    DeviceGuard dg(ctx->device);
    // counts_in_row_order (throws before any layout is planned)
    uint64_t* rc = ctx->scratch_t<uint64_t>(kScratchF, n ? n : 1);
    if (n) {
      const uint64_t* c = dev_in(ctx, counts, n, kStageIn0);
      const uint64_t* o = dev_in(ctx, ordering, n, kStageIn1);
      auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 1);
      TGB_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
      row_order_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(c, n, o, rc, bad);
      TGB_LAUNCHED();
      unsigned long long hb;
      TGB_CUDA(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      if (hb != ~0ull) domain_error("ordering id out of range");
    }
    std::vector<tg_layout> lays;
    std::vector<double> reps;
    std::vector<tg_report> out;
    bool total_checked = false;
    for (uint64_t i = 0; i < nf; ++i) {
      const double rep = std::min(replicated, fr[i]);  // :195
      lays.push_back(plan_layout(n, fr[i], rep, devices, dim, eb, budget));
      reps.push_back(rep);
      if (!total_checked) {
        // simulate_trace of the first fraction runs before the next plan_layout
        std::vector<tg_report> first;
        if (simulate_many(ctx, rc, n, {lays[0]}, first) == 0)
          domain_error("simulate_trace: counter total is zero");
        total_checked = true;
      }
    }
    simulate_many(ctx, rc, n, lays, out);
    for (uint64_t i = 0; i < nf; ++i) {
      out_layouts[i] = lays[i];
      out_reports[i] = out[i];
      out_rep[i] = reps[i];
    }
  });
}

// --------------------------------------------------------------- the store
int tg_store_create(tg_ctx* ctx, const tg_layout* layout, uint32_t device_index, uint32_t flags,
                    tg_store** out) {
  return guard([&] {
    validate_layout(*layout);
    if (layout->num_devices > TG_MAX_DEVICES)
      domain_error("tiered store: at most " + std::to_string(TG_MAX_DEVICES) + " devices");
    if (device_index >= layout->num_devices) device_error(*layout, device_index);
    DeviceGuard dg(ctx->device);
    auto* s = new tg_store;
    s->ctx = ctx;
    s->L = *layout;
    s->dev = device_index;
    s->flags = flags;
    s->R = layout->feature_dim * layout->elem_bytes;
    const uint64_t lb = layout->local_boundary, mb = layout->multi_boundary;
    const uint64_t D = layout->num_devices;
    const uint64_t inter = mb - lb;
    const uint64_t mine = inter > device_index ? (inter - device_index + D - 1) / D : 0;
    s->local_rows = lb + mine;
    try {
      TGB_CUDA(tgb::dev_malloc(&s->local, std::max<uint64_t>(s->local_rows * s->R, 16)));
      TGB_CUDA(tgb::dev_malloc(&s->counters, 64));
      // [0..2] counters, [3] first bad index (~0 = none), [4] CTA ticket
      TGB_CUDA(cudaMemsetAsync(s->counters, 0, 64, ctx->stream));
      TGB_CUDA(cudaMemsetAsync(s->counters + 3, 0xff, 8, ctx->stream));
      TGB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->result_host), 64, cudaHostAllocMapped));
      std::memset(s->result_host, 0, 64);  // [4] = 0: no call posted yet (sequence numbers start at 1)
      void* rd = nullptr;
      TGB_CUDA(cudaHostGetDevicePointer(&rd, s->result_host, 0));
      s->result_dev = static_cast<uint64_t*>(rd);
      ctx->sync();
      s->inter[device_index] = s->local + lb * s->R;
    } catch (...) {
      tg_store_destroy(s);
      throw;
    }
    *out = s;
  });
}

int tg_store_destroy(tg_store* s) {
  if (!s) return TG_OK;
  DeviceGuard dg(s->ctx->device);
  cudaFree(s->local);
  cudaFree(s->counters);
  if (s->result_host) cudaFreeHost(s->result_host);
  if (s->own_cold && s->cold_host) cudaFreeHost(s->cold_host);
  if (s->own_cold_src) cudaFree(s->cold_src);
  if (s->own_cold_tail) cudaFree(s->cold_tail);
  if (s->registered) release_host_matrix(s->registered);
  delete s;
  return TG_OK;
}

void* tg_store_local_base(const tg_store* s) { return s ? s->local : nullptr; }

int tg_store_measure_cold_us(tg_store* s, uint64_t rows, int reps, double* us) {
  return guard([&] {
    if (!s->placed) domain_error("tiered store: tg_store_place has not run");
    tg_ctx* ctx = s->ctx;
    DeviceGuard dg(ctx->device);
    const uint64_t mb = s->L.multi_boundary, N = s->L.num_rows;
    if (mb >= N) domain_error("tiered store: no cold rows");
    if (!rows) domain_error("empty measurement");
    // K8 itself over `rows` random cold ids only (L2 flushed before each launch)
    auto* ids = ctx->scratch_t<uint64_t>(kScratchD, rows);
    auto* out = ctx->scratch_t<uint8_t>(kScratchF, rows * s->R);
    auto* fl = ctx->scratch_t<uint8_t>(kScratchE, 256ull << 20);
    auto* c = ctx->scratch_t<uint64_t>(kSmall, 4);
    cudaEvent_t a, b;
    TGB_CUDA(cudaEventCreate(&a));
    TGB_CUDA(cudaEventCreate(&b));
    double tot = 0;
    for (int i = 0; i <= reps; ++i) {
      random_ids_kernel<<<grid_for(rows, 256), 256, 0, ctx->stream>>>(ids, rows, mb, N - mb, 77 + i);
      TGB_LAUNCHED();
      TGB_CUDA(cudaMemsetAsync(fl, i, 256ull << 20, ctx->stream));
      TGB_CUDA(cudaMemsetAsync(c, 0, 32, ctx->stream));
      TGB_CUDA(cudaEventRecord(a, ctx->stream));
      launch_gather(s, ids, rows, out, c, reinterpret_cast<unsigned long long*>(c + 3));
      TGB_CUDA(cudaEventRecord(b, ctx->stream));
      TGB_CUDA(cudaEventSynchronize(b));
      float ms = 0;
      TGB_CUDA(cudaEventElapsedTime(&ms, a, b));
      if (i) tot += ms;  // the first launch warms
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *us = tot / std::max(reps, 1) * 1e3;
  });
}
// The platform's ceiling for the cold part of a launch: `rows` random rows of
// the store's own cold tier (same region, stride and host bytes per row)
// read by a plain one-warp-per-row copy kernel, L2 flushed before each
// launch. Against K8's cold-only time this separates the kernel from the
// host-memory path (translation of the mapped region, PCIe).
int tg_store_measure_cold_rows_us(tg_store* s, uint64_t rows, int reps, double* us) {
  return guard([&] {
    if (!s || !us) domain_error("tg_store_measure_cold_rows_us: null argument");
    if (!s->placed) domain_error("tiered store: tg_store_place has not run");
    const uint64_t mb = s->L.multi_boundary, N = s->L.num_rows;
    if (mb >= N) domain_error("tiered store: no cold rows");
    if (s->flags & TG_COLD_INDIRECT) domain_error("tiered store: the cold tier is read in place");
    DeviceGuard dg(s->ctx->device);
    const tg_store* o = s->cold_owner ? s->cold_owner : s;
    const uint64_t hc = s->cold_head ? s->cold_head : s->R;
    *us = measure_rows_us(s->ctx, o->cold_dev, N - mb, s->cold_stride, hc, rows, reps);
  });
}

uint64_t tg_store_local_rows(const tg_store* s) { return s ? s->local_rows : 0; }
uint64_t tg_store_cold_host_bytes(const tg_store* s) {
  return s ? (s->cold_head ? s->cold_head : s->R) : 0;
}

int tg_store_set_peer(tg_store* s, uint32_t d, const void* peer_local_base) {
  return guard([&] {
    if (d >= s->L.num_devices) device_error(s->L, d);
    s->inter[d] = static_cast<const uint8_t*>(peer_local_base) + s->L.local_boundary * s->R;
  });
}

int tg_store_share_cold(tg_store* s, const tg_store* owner) {
  return guard([&] {
    if (owner->L.num_rows != s->L.num_rows || owner->L.multi_boundary != s->L.multi_boundary ||
        owner->R != s->R)
      domain_error("tiered store: cold tier layouts differ");
    s->cold_owner = owner;
  });
}

}  // extern "C"

namespace tgb {
const uint8_t* ensure_cold_tier(tg_store* s) {
  const uint64_t cold = s->L.num_rows - s->L.multi_boundary;
  s->cold_stride = (s->flags & TG_COLD_PAD128) ? (s->R + 127) / 128 * 128 : s->R;
  s->cold_head = 0;
  if ((s->flags & TG_COLD_SPLIT_TAIL) && s->R > 128 && s->R % 128 && s->R % 16 == 0) {
    // whole 128 B lines in host memory (packed: every row starts on a line),
    // the R mod 128 remainder of every cold row in HBM
    s->cold_head = s->R / 128 * 128;
    s->cold_stride = s->cold_head;
    if (!s->own_cold_tail) {
      TGB_CUDA(tgb::dev_malloc(&s->cold_tail, std::max<uint64_t>(cold * (s->R - s->cold_head), 16)));
      s->own_cold_tail = true;
    }
  }
  if (!s->own_cold && !s->cold_attached) {
    TGB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->cold_host),
                           std::max<uint64_t>(cold * s->cold_stride, 16),
                           cudaHostAllocMapped | cudaHostAllocPortable));
    s->own_cold = true;
  }
  void* cd = nullptr;
  TGB_CUDA(cudaHostGetDevicePointer(&cd, s->cold_host, 0));
  s->cold_dev = static_cast<const uint8_t*>(cd);
  return s->cold_dev;
}

// K7 placement from `src_rows` (src_nrows rows of R bytes; host or device)
// where new id i's bytes are source row order[i] (u32, device, N entries).
void place_impl(tg_store* s, const void* src_rows, uint64_t src_nrows, const uint32_t* order) {
  tg_ctx* ctx = s->ctx;
  const uint64_t N = s->L.num_rows, R = s->R, mb = s->L.multi_boundary;
  // source rows: device memory, mapped pinned memory, or pageable (registered here)
  const uint8_t* src = nullptr;
  void* reg = nullptr;
  if (is_device_ptr(src_rows)) {
    src = static_cast<const uint8_t*>(src_rows);
  } else {
    bool owned = false;
    src = acquire_host_matrix(src_rows, src_nrows * R, &owned);
    if (owned) reg = const_cast<void*>(src_rows);
  }
  // K7a: this device's HBM rows (replicated prefix + interleaved slice)
  MoveArgs a{};
  a.src = src;
  a.dst = s->local;
  a.src_stride = R;
  a.dst_stride = R;
  a.src_idx32 = order;
  a.slot_mode = 1;
  a.lb = s->L.local_boundary;
  a.D = s->L.num_devices;
  a.dev = s->dev;
  launch_move(ctx, a, s->local_rows, R);
  // K7b: the cold tier
  if (s->cold_owner) {
    s->cold_dev = s->cold_owner->cold_dev;
    s->cold_src = s->cold_owner->cold_src;
    s->cold_stride = s->cold_owner->cold_stride;
    s->cold_head = s->cold_owner->cold_head;
    s->cold_tail = s->cold_owner->cold_tail;
  } else if (s->flags & TG_COLD_INDIRECT) {
    // the caller's rows are read in place through the row map
    const uint64_t cold = N - mb;
    if (!s->cold_src) {
      TGB_CUDA(tgb::dev_malloc(&s->cold_src, sizeof(uint32_t) * std::max<uint64_t>(cold, 1)));
      s->own_cold_src = true;
    }
    if (cold)
      TGB_CUDA(cudaMemcpyAsync(s->cold_src, order + mb, cold * 4, cudaMemcpyDeviceToDevice,
                               ctx->stream));
    s->cold_dev = src;
    s->cold_stride = R;
    s->cold_head = 0;
    if (s->registered) release_host_matrix(s->registered);
    s->registered = reg;  // keep the caller's matrix mapped for the store's lifetime
    reg = nullptr;
  } else {
    const uint64_t cold = N - mb;
    ensure_cold_tier(s);
    void* cd = const_cast<uint8_t*>(s->cold_dev);
    MoveArgs c{};
    c.src = src;
    c.dst = static_cast<uint8_t*>(cd);
    c.src_stride = R;
    c.dst_stride = s->cold_stride;
    c.src_idx32 = order;
    c.src_row_base = mb;
    const uint64_t H = s->cold_head ? s->cold_head : R;
    if (!s->cold_attached || s->cold_fill) launch_move(ctx, c, cold, H);  // else filled by its owner
    if (s->cold_head) {  // the remainders into HBM
      MoveArgs t = c;
      t.src = src + H;
      t.dst = s->cold_tail;
      t.dst_stride = R - H;
      launch_move(ctx, t, cold, R - H);
    }
  }
  ctx->sync();
  if (reg) release_host_matrix(reg);
  s->placed = true;
}

__global__ void check_rows_kernel(const uint32_t* __restrict__ m, uint64_t n, uint64_t nrows,
                                  unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (m[i] >= nrows) atomicMin(bad, (unsigned long long)i);
}
}  // namespace tgb

extern "C" {

int tg_store_place(tg_store* s, const void* features, const uint64_t* new_id_of) {
  return guard([&] {
    tg_ctx* ctx = s->ctx;
    DeviceGuard dg(ctx->device);
    const uint64_t N = s->L.num_rows;
    if (N == 0) {
      s->placed = true;
      return;
    }
    // the permutation (validated like reorder_features, reorder.cpp:102) and its inverse
    const uint64_t* perm = dev_in(ctx, new_id_of, N, kStageIn0);
    uint32_t* order = ctx->scratch_t<uint32_t>(kScratchD, N);
    check_permutation(ctx, perm, N, order);
    place_impl(s, features, N, order);
  });
}

int tg_store_place_rows(tg_store* s, const void* rows, uint64_t nrows, const uint32_t* row_of) {
  return guard([&] {
    tg_ctx* ctx = s->ctx;
    DeviceGuard dg(ctx->device);
    const uint64_t N = s->L.num_rows;
    if (N == 0) {
      s->placed = true;
      return;
    }
    if (nrows == 0) domain_error("tg_store_place_rows: no source rows");
    if (nrows > 0xffffffffull) domain_error("tg_store_place_rows: at most 2^32-1 source rows");
    uint32_t* m = ctx->scratch_t<uint32_t>(kScratchD, N);
    TGB_CUDA(cudaMemcpyAsync(m, row_of, 4 * N, cudaMemcpyDefault, ctx->stream));
    auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 1);
    TGB_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
    check_rows_kernel<<<grid_for(N, 256), 256, 0, ctx->stream>>>(m, N, nrows, bad);
    TGB_LAUNCHED();
    unsigned long long hb;
    TGB_CUDA(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (hb != ~0ull)
      domain_error("tg_store_place_rows: row_of[" + std::to_string(hb) + "] >= " +
                   std::to_string(nrows));
    place_impl(s, rows, nrows, m);
  });
}

int tg_gather_rows_async(tg_store* s, const uint64_t* ids_dev, uint64_t n, void* dst_dev,
                         uint64_t* counters_dev, uint64_t* err_dev) {
  return guard([&] {
    if (n == 0) return;
    DeviceGuard dg(s->ctx->device);
    launch_gather(s, ids_dev, n, dst_dev, counters_dev,
                  reinterpret_cast<unsigned long long*>(err_dev));
  });
}

int tg_gather_rows(tg_store* s, const uint64_t* ids, uint64_t n, void* dst, tg_report* report) {
  return guard([&] {
    if (n == 0) return;
    tg_ctx* ctx = s->ctx;
    DeviceGuard dg(ctx->device);
    // ids in pinned, mapped host memory are read in place (UVA zero-copy,
    // overlapping the gather) instead of being staged by a separate copy
    const void* mapped = mapped_device_ptr(ids);
    const uint64_t* d = mapped ? static_cast<const uint64_t*>(mapped) : dev_in(ctx, ids, n, kStageIn0);
    DevOut<uint8_t> o(ctx, static_cast<uint8_t*>(dst), n * s->R, kStageOut0);
    uint64_t* c = s->counters;  // armed: zero counters, err = ~0 (re-armed by the kernel)
    auto* err = reinterpret_cast<unsigned long long*>(c + 3);
    volatile uint64_t* hv = s->result_host;
    const uint64_t seq = ++s->fin_seq;
    launch_gather(s, d, n, o.dev(), c, err, /*finalize=*/true);
    if (o.host) {
      o.finish();  // the rows come back to host memory: copy + stream sync
    } else {
      // Rows stay in HBM: return as soon as the kernel's last CTA has posted
      // the counters and the call's sequence number to mapped host memory
      // (every CTA's rows are out by then), instead of waiting for the
      // stream's completion. A kernel that never posts (a fault) falls back
      // to the stream sync after 2 s, which reports the error.
      const auto t0 = std::chrono::steady_clock::now();
      for (uint32_t k = 1; hv[4] != seq; ++k) {
        if ((k & 4095) == 0 &&
            std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) {
          ctx->sync();
          if (hv[4] != seq) throw Error(TG_ERR_INTERNAL, "gather: the kernel did not post its result");
          break;
        }
      }
    }
    uint64_t h[4] = {hv[0], hv[1], hv[2], hv[3]};
    if (h[3] != ~0ull) {  // reference semantics: prefix accounted, then DomainError
      const uint64_t first = h[3];
      TGB_CUDA(cudaMemsetAsync(c, 0, 24, ctx->stream));
      if (first) account(ctx, s->L, d, first, s->dev, c, err);
      TGB_CUDA(cudaMemcpyAsync(h, c, 24, cudaMemcpyDeviceToHost, ctx->stream));
      TGB_CUDA(cudaMemsetAsync(c, 0, 24, ctx->stream));  // re-arm for the next call
      ctx->sync();
      add_report(report, h[0], h[1], h[2], s->R);
      uint64_t bad;
      TGB_CUDA(cudaMemcpy(&bad, d + first, 8, cudaMemcpyDeviceToHost));
      range_error(s->L, bad);
    }
    add_report(report, h[0], h[1], h[2], s->R);
  });
}

int tg_time_gather_rows(tg_store* s, const uint64_t* const* ids, const uint64_t* counts, uint64_t k,
                        void* dst, int flush_l2, tg_report* report, double* seconds) {
  return guard([&] {
    tg_ctx* ctx = s->ctx;
    DeviceGuard dg(ctx->device);
    uint8_t* fl = flush_l2 ? ctx->scratch_t<uint8_t>(kScratchE, 256ull << 20) : nullptr;
    double tot = 0.0;
    for (uint64_t i = 0; i < k; ++i) {
      if (fl) {
        TGB_CUDA(cudaMemsetAsync(fl, static_cast<int>(i & 0xff), 256ull << 20, ctx->stream));
        ctx->sync();
      }
      const auto t0 = std::chrono::steady_clock::now();
      const int rc = tg_gather_rows(s, ids[i], counts[i], dst, report);
      const auto t1 = std::chrono::steady_clock::now();
      if (rc) throw Error(rc, tg_last_error());
      tot += std::chrono::duration<double>(t1 - t0).count();
    }
    *seconds = tot;
  });
}

// ------------------------------------------------------------- reorder ops
int tg_validate_permutation(tg_ctx* ctx, const uint64_t* perm, uint64_t n) {
  return guard([&] {
    if (n == 0) return;
    DeviceGuard dg(ctx->device);
    check_permutation(ctx, dev_in(ctx, perm, n, kStageIn0), n, nullptr);
  });
}

int tg_invert(tg_ctx* ctx, const uint64_t* perm, uint64_t n, uint64_t* out) {
  return guard([&] {  // reorder.cpp:31-37
    if (n == 0) return;
    DeviceGuard dg(ctx->device);
    const uint64_t* p = dev_in(ctx, perm, n, kStageIn0);
    uint32_t* inv = ctx->scratch_t<uint32_t>(kScratchD, n);
    check_permutation(ctx, p, n, inv);
    DevOut<uint64_t> o(ctx, out, n, kStageOut0);
    u32_to_u64_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(inv, o.dev(), n);
    TGB_LAUNCHED();
    o.finish();
  });
}

int tg_reorder_features(tg_ctx* ctx, const void* src, uint64_t rows, uint64_t row_bytes,
                        const uint64_t* perm, uint64_t perm_len, void* dst) {
  return guard([&] {  // reorder.cpp:97-117
    if (perm_len != rows)
      domain_error("permutation length " + std::to_string(perm_len) + " != num_rows " +
                   std::to_string(rows));
    if (rows == 0) return;
    DeviceGuard dg(ctx->device);
    const uint64_t* p = dev_in(ctx, perm, rows, kStageIn0);
    check_permutation(ctx, p, rows, nullptr);
    const uint64_t bytes = rows * row_bytes;
    const uint8_t* s = dev_in(ctx, static_cast<const uint8_t*>(src), bytes, kStageIn1);
    DevOut<uint8_t> o(ctx, static_cast<uint8_t*>(dst), bytes, kStageOut0);
    MoveArgs a{};
    a.src = s;
    a.dst = o.dev();
    a.src_stride = row_bytes;
    a.dst_stride = row_bytes;
    a.dst_idx64 = p;  // scatter: new row perm[u] <- old row u
    launch_move(ctx, a, rows, row_bytes);
    o.finish();
  });
}

// ------------------------------------------------------------- peer memory
int tg_enable_peer_access(int device, int peer) {
  return guard([&] {
    DeviceGuard dg(device);
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
      cudaGetLastError();
      return;
    }
    TGB_CUDA(e);
  });
}

int tg_ipc_get_handle(const void* p, void* out) {
  return guard([&] {
    cudaIpcMemHandle_t h;
    TGB_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(p)));
    static_assert(sizeof(h) == 64, "ipc handle size");
    std::memcpy(out, &h, 64);
  });
}

int tg_ipc_open_handle(tg_ctx* ctx, const void* handle, void** out) {
  return guard([&] {
    DeviceGuard dg(ctx->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    TGB_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int tg_ipc_close_handle(void* p) {
  return guard([&] { TGB_CUDA(cudaIpcCloseMemHandle(p)); });
}

int tg_device_alloc(tg_ctx* ctx, uint64_t bytes, void** out) {
  return guard([&] {
    DeviceGuard dg(ctx->device);
    TGB_CUDA(tgb::dev_malloc(out, std::max<uint64_t>(bytes, 16)));
    TGB_CUDA(cudaMemsetAsync(*out, 0, std::max<uint64_t>(bytes, 16), ctx->stream));
    ctx->sync();
  });
}

int tg_device_free(tg_ctx* ctx, void* p) {
  return guard([&] {
    DeviceGuard dg(ctx->device);
    TGB_CUDA(cudaFree(p));
  });
}

int tg_host_register(void* p, uint64_t bytes) {
  return guard([&] {
    TGB_CUDA(cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
  });
}
void* tg_mapped_device_ptr(const void* host) { return mapped_device_ptr(host); }

int tg_host_unregister(void* p) {
  return guard([&] { TGB_CUDA(cudaHostUnregister(p)); });
}
int tg_host_alloc(uint64_t bytes, void** out) {
  return guard([&] {
    TGB_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  });
}
int tg_host_free(void* p) {
  return guard([&] { TGB_CUDA(cudaFreeHost(p)); });
}

// One host segment per NODE shared by every process (PAPER.md:659-663:
// shared memory + cudaHostRegister in each process): POSIX shared memory
// (/dev/shm), mapped and registered (mapped | portable) in the caller.
int tg_host_shared_map(const char* name, uint64_t bytes, int create, void** out) {
  return guard([&] {
    if (!name || !out || !bytes) domain_error("tg_host_shared_map: bad argument");
    const int fd = shm_open(name, create ? (O_CREAT | O_EXCL | O_RDWR) : O_RDWR, 0600);
    if (fd < 0)
      throw Error(TG_ERR_IO, std::string("shm_open ") + name + ": " + std::strerror(errno));
    if (create && ftruncate(fd, static_cast<off_t>(bytes)) != 0) {
      const int e = errno;
      close(fd);
      shm_unlink(name);
      throw Error(TG_ERR_IO, std::string("ftruncate ") + name + ": " + std::strerror(e));
    }
    struct stat st{};
    if (fstat(fd, &st) != 0 || static_cast<uint64_t>(st.st_size) < bytes) {
      close(fd);
      throw Error(TG_ERR_IO, std::string("shared segment ") + name + " is smaller than requested");
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw Error(TG_ERR_IO, std::string("mmap ") + name + ": " + std::strerror(errno));
    const cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
      munmap(p, bytes);
      TGB_CUDA(e);
    }
    *out = p;
  });
}

int tg_host_shared_unmap(void* p, uint64_t bytes) {
  return guard([&] {
    TGB_CUDA(cudaHostUnregister(p));
    if (munmap(p, bytes) != 0) throw Error(TG_ERR_IO, std::string("munmap: ") + std::strerror(errno));
  });
}

int tg_host_shared_unlink(const char* name) {
  return guard([&] {
    if (shm_unlink(name) != 0 && errno != ENOENT)
      throw Error(TG_ERR_IO, std::string("shm_unlink ") + name + ": " + std::strerror(errno));
  });
}

// The cold tier in caller memory (e.g. a tg_host_shared_map segment shared
// by all processes of a node): `bytes` >= tg_store_cold_tier_bytes(s). With
// fill != 0 this store's placement writes the cold rows there (one process
// per node does); with fill == 0 it only reads them (the others, after the
// filler's placement finished).
int tg_store_attach_cold(tg_store* s, void* host, uint64_t bytes, int fill) {
  return guard([&] {
    if (s->flags & TG_COLD_INDIRECT)
      domain_error("tg_store_attach_cold: the store reads its cold rows in place (INDIRECT)");
    if (s->placed) domain_error("tg_store_attach_cold: call before placement");
    const uint64_t need = tg_store_cold_tier_bytes(s);
    if (bytes < need)
      domain_error("tg_store_attach_cold: " + std::to_string(bytes) + " bytes, " +
                   std::to_string(need) + " needed");
    if (!mapped_device_ptr(host))
      domain_error("tg_store_attach_cold: memory is not mapped for the device (register it)");
    if (s->own_cold && s->cold_host) cudaFreeHost(s->cold_host);
    s->cold_host = static_cast<uint8_t*>(host);
    s->own_cold = false;
    s->cold_attached = true;
    s->cold_fill = fill != 0;
  });
}

uint64_t tg_store_cold_tier_bytes(const tg_store* s) {
  const uint64_t cold = s->L.num_rows - s->L.multi_boundary;
  uint64_t stride = (s->flags & TG_COLD_PAD128) ? (s->R + 127) / 128 * 128 : s->R;
  if ((s->flags & TG_COLD_SPLIT_TAIL) && s->R > 128 && s->R % 128 && s->R % 16 == 0)
    stride = s->R / 128 * 128;
  return std::max<uint64_t>(cold * stride, 16);
}

}  // extern "C"
