// GPU GraphSAGE minibatch expansion — SURVEY §8(f) row 1, the producer of
// the tiered gather's node-id lists, moved onto the device.
//
// Reference: proj/src/sampling.cpp:35-90 (BatchRng streams,
// sample_in_neighbors, build_minibatch) over proj/include/tiergraph/rng.hpp
// (mix64, derive_stream_key, counter-based RngStream, Lemire next_below) and
// proj/src/rng.cpp:8-40 (Floyd's k-subset).
//
// Bit-identical member lists by construction: every node's draws come from
// its own stream keyed by (seed, 0x534D, epoch, batch, layer, node), so the
// SET a node samples does not depend on the order frontier nodes are
// visited. The device therefore needs no sorts:
//   * a layer's frontier is the de-duplicated set of the previous layer's
//     samples: a per-node stamp array (atomicExch(stamp) != stamp admits a
//     node once per layer) appends it to the next frontier in any order;
//   * the members (seeds + every frontier) carry a per-minibatch stamp, and
//     the final sorted unique list is a compaction of the stamped nodes in
//     node-id order — sorted for free.
// One thread per frontier node runs Floyd's algorithm exactly as rng.cpp does
// (membership among the picks already emitted; the reference switches from a
// linear scan to a hash set above 64 picks, which yields the same set).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"
#include "structure_internal.cuh"

namespace tgb {

__device__ __forceinline__ uint64_t dmix64(uint64_t x) {  // rng.hpp:13-18
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

struct DevRng {  // rng.hpp:32-59
  uint64_t s;
  __device__ uint64_t next() { return dmix64(s++); }
  __device__ uint64_t below(uint64_t bound) {  // Lemire multiply-shift with rejection
    uint64_t x = next();
    uint64_t lo = x * bound, hi = __umul64hi(x, bound);
    if (lo < bound) {
      const uint64_t t = (0 - bound) % bound;
      while (lo < t) {
        x = next();
        lo = x * bound;
        hi = __umul64hi(x, bound);
      }
    }
    return hi;
  }
};

struct SampleArgs {
  SGraphView g;  // transposed graph (row v = in-neighbours of v), tiered or not
  const uint32_t* frontier;
  const uint32_t* f_dev;  // frontier size, written by the previous launch (no host round trip)
  uint32_t fanout;
  uint64_t key_base;  // mix64(seed ^ IV) folded with {0x534D, epoch, batch, layer}
  uint32_t* picks;    // f x fanout scratch for Floyd's membership test
  uint32_t* layer_mark;
  uint32_t layer_stamp;
  uint32_t* member_bits;  // one bit per node: a member of this minibatch
  uint32_t* next;
  uint32_t* next_count;
  // optional outputs (run_training_trace, raw_draws; sampling.cpp:56-140)
  unsigned long long* counts;  // per-node access counts, or null
  int count_raw;               // 1: one per draw; 0: one per new minibatch member
  uint64_t* raw;               // every draw, or null
  unsigned long long* raw_n;
  uint64_t raw_cap;
};

__device__ __forceinline__ void admit(const SampleArgs& a, uint32_t u) {
  if (a.raw) {
    const unsigned long long k = atomicAdd(a.raw_n, 1ull);
    if (k < a.raw_cap) a.raw[k] = u;
  }
  if (a.counts && a.count_raw) atomicAdd(a.counts + u, 1ull);
  // a plain L2 read first: hot nodes are drawn by many threads per layer,
  // and only the first needs the atomic (a stale read just costs one)
  // the lanes calling here together (all of them reach the ballot below)
  const unsigned act = __activemask();
  bool fresh = false;
  if (__ldcg(a.layer_mark + u) != a.layer_stamp)
    fresh = atomicExch(a.layer_mark + u, a.layer_stamp) != a.layer_stamp;
  // append to the next frontier with one atomic per warp: every new node of
  // the layer hits the same counter
  const unsigned m = __ballot_sync(act, fresh);
  if (!m) return;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(a.next_count, static_cast<uint32_t>(__popc(m)));
  base = __shfl_sync(act, base, leader);
  if (fresh) {
    a.next[base + __popc(m & ((1u << lane) - 1u))] = u;
    const uint32_t bit = 1u << (u & 31);
    if ((__ldcg(a.member_bits + (u >> 5)) & bit) == 0 &&
        (atomicOr(a.member_bits + (u >> 5), bit) & bit) == 0 && a.counts && !a.count_raw)
      atomicAdd(a.counts + u, 1ull);
  }
}

// admit() for up to K draws of one thread at once, phase by phase so the
// memory operations of different draws are in flight together: mark reads,
// then the claiming exchanges, then one warp-aggregated append for all of
// them, then the member bits. Draw order within the thread is preserved in
// the raw list and the per-node counts are order-independent.
template <int K>
__device__ __forceinline__ void admit_batch(const SampleArgs& a, const uint32_t (&u)[K],
                                            uint32_t nvalid) {
  if (a.raw || a.counts) {
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if ((uint32_t)q >= nvalid) continue;
      if (a.raw) {
        const unsigned long long k = atomicAdd(a.raw_n, 1ull);
        if (k < a.raw_cap) a.raw[k] = u[q];
      }
      if (a.counts && a.count_raw) atomicAdd(a.counts + u[q], 1ull);
    }
  }
  uint32_t seen[K];
#pragma unroll
  for (int q = 0; q < K; ++q) seen[q] = (uint32_t)q < nvalid ? __ldcg(a.layer_mark + u[q]) : a.layer_stamp;
  uint32_t fresh = 0;  // bit q: draw q claimed its node for the next frontier
#pragma unroll
  for (int q = 0; q < K; ++q)
    if (seen[q] != a.layer_stamp && atomicExch(a.layer_mark + u[q], a.layer_stamp) != a.layer_stamp)
      fresh |= 1u << q;
  // one append for the whole warp: exclusive scan of the lanes' fresh counts
  const unsigned act = __activemask();
  const int lane = threadIdx.x & 31;
  const uint32_t mine = __popc(fresh);  // <= K <= 16: five bits
  const uint32_t total = __reduce_add_sync(act, mine);
  if (!total) return;
  // exclusive prefix over the active lanes below this one, bit by bit
  const uint32_t below = act & ((1u << lane) - 1u);
  uint32_t excl = 0;
#pragma unroll
  for (int k = 0; k < 5; ++k)
    excl += static_cast<uint32_t>(__popc(__ballot_sync(act, (mine >> k) & 1u) & below)) << k;
  const int top = 31 - __clz(act);
  uint32_t base = 0;
  if (lane == top) base = atomicAdd(a.next_count, total);
  base = __shfl_sync(act, base, top);
  uint32_t pos = base + excl;
#pragma unroll
  for (int q = 0; q < K; ++q)
    if (fresh & (1u << q)) a.next[pos++] = u[q];
#pragma unroll
  for (int q = 0; q < K; ++q) {
    if (!(fresh & (1u << q))) continue;
    const uint32_t bit = 1u << (u[q] & 31);
    if ((atomicOr(a.member_bits + (u[q] >> 5), bit) & bit) == 0 && a.counts && !a.count_raw)
      atomicAdd(a.counts + u[q], 1ull);
  }
}

// sampling.cpp:39-54 + rng.cpp:8-40 for one frontier node per thread.
// Fanouts up to kRegK keep Floyd's picks in registers and split each node's
// work into: all draws (ALU only), then all neighbour loads (independent, in
// flight together), then the admits -- one memory round trip per phase
// instead of one per draw.
constexpr uint32_t kRegK = 16;
__global__ void __launch_bounds__(256) sample_layer_kernel(const SampleArgs a) {
  const uint32_t f = *a.f_dev;  // written by the previous launch: no host round trip
  uint32_t rd0 = 0, rd1 = 0, rd2 = 0;  // neighbour ids read per tier (local, peer, host)
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < f; i += gridDim.x * blockDim.x) {
    const uint32_t v = a.frontier[i];
    const uint32_t b = a.g.off[v], deg = a.g.off[v + 1] - b;
    int tier;
    const uint32_t* nb = a.g.row(v, b, &tier);  // row v's neighbour ids, in its tier
    {
      const uint32_t c = deg < a.fanout ? deg : a.fanout;  // ids this node reads
      rd0 += tier == 0 ? c : 0u;
      rd1 += tier == 1 ? c : 0u;
      rd2 += tier == 2 ? c : 0u;
    }
    if (deg <= a.fanout) {  // all in-neighbours
      uint32_t p = 0;
      for (; p + kRegK <= deg; p += kRegK) {
        uint32_t u[kRegK];
#pragma unroll
        for (uint32_t q = 0; q < kRegK; ++q) u[q] = nb[p + q];
        admit_batch<kRegK>(a, u, kRegK);
      }
      uint32_t u[kRegK];
#pragma unroll
      for (uint32_t q = 0; q < kRegK; ++q) u[q] = p + q < deg ? nb[p + q] : 0u;
      admit_batch<kRegK>(a, u, deg - p);
      continue;
    }
    DevRng rng{dmix64(a.key_base ^ dmix64(v))};  // derive_stream_key(..., node)
    if (a.fanout <= kRegK) {
      uint32_t pk[kRegK];
#pragma unroll
      for (uint32_t jj = 0; jj < kRegK; ++jj) {
        if (jj < a.fanout) {
          const uint64_t j = deg - a.fanout + jj;
          const uint32_t t = static_cast<uint32_t>(rng.below(j + 1));
          bool seen = false;
#pragma unroll
          for (uint32_t q = 0; q < kRegK; ++q) seen |= q < jj && pk[q] == t;
          pk[jj] = seen ? static_cast<uint32_t>(j) : t;
        }
      }
      uint32_t u[kRegK];
#pragma unroll
      for (uint32_t q = 0; q < kRegK; ++q) u[q] = q < a.fanout ? nb[pk[q]] : 0u;
      admit_batch<kRegK>(a, u, a.fanout);  // draw order, as the reference emits them
      continue;
    }
    uint32_t* picks = a.picks + static_cast<uint64_t>(i) * a.fanout;
    uint32_t cnt = 0;
    for (uint64_t j = deg - a.fanout; j < deg; ++j) {
      const uint32_t t = static_cast<uint32_t>(rng.below(j + 1));
      bool seen = false;
      for (uint32_t q = 0; q < cnt; ++q) seen |= picks[q] == t;
      const uint32_t p = seen ? static_cast<uint32_t>(j) : t;
      picks[cnt++] = p;
      admit(a, nb[p]);
    }
  }
  if (a.g.reads) {  // every lane is here (blocks are whole warps)
    const uint32_t r[3] = {__reduce_add_sync(0xffffffffu, rd0), __reduce_add_sync(0xffffffffu, rd1),
                           __reduce_add_sync(0xffffffffu, rd2)};
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int t = 0; t < 3; ++t)
        if (r[t]) atomicAdd(a.g.reads + t, (unsigned long long)r[t]);
  }
}

__global__ void seed_kernel(const uint64_t* __restrict__ seeds, uint64_t ns, uint64_t n,
                            uint32_t* layer_mark, uint32_t stamp, uint32_t* member_bits,
                            uint32_t* frontier, uint32_t* count,
                            unsigned long long* bad, unsigned long long* counts, int count_raw,
                            uint64_t* raw, unsigned long long* raw_n, uint64_t raw_cap) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ns;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = seeds[i];
    if (s >= n) {
      atomicMin(bad, (unsigned long long)i);
      continue;
    }
    const uint32_t u = static_cast<uint32_t>(s);
    if (raw) {  // each seed once, as given (sampling.cpp:70)
      const unsigned long long k = atomicAdd(raw_n, 1ull);
      if (k < raw_cap) raw[k] = u;
    }
    if (counts && count_raw) atomicAdd(counts + u, 1ull);
    if (atomicExch(layer_mark + u, stamp) != stamp) {
      frontier[atomicAdd(count, 1u)] = u;
      atomicOr(member_bits + (u >> 5), 1u << (u & 31));  // the bitmap is clear per minibatch
      if (counts && !count_raw) atomicAdd(counts + u, 1ull);
    }
  }
}

// members = set bits in node-id order: per-block popcounts (BLK words =
// 32·BLK nodes per block), then positions. Reads N/8 bytes per minibatch.
// BLK = 256 words per CTA for bitmaps up to 2^20 words (C2: 300 CTAs instead
// of 75), else 1024 (the block-count prefix stays short on huge graphs).
constexpr int kCompactBlock = 256;   // the smallest block: sizes the block-count array
constexpr int kCompactBig = 1024;
constexpr uint64_t kCompactBigWords = 1ull << 20;
template <int BLK>
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, uint32_t* total) {
  __shared__ uint32_t ws[BLK / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  uint32_t before = 0, tot = 0;
  for (int k = 0; k < BLK / 32; ++k) {
    if (k < w) before += ws[k];
    tot += ws[k];
  }
  *total = tot;
  return before + x - v;
}

template <int BLK>
__global__ void __launch_bounds__(BLK) member_count_kernel(const uint32_t* __restrict__ bits,
                                                           uint64_t nwords,
                                                           uint32_t* __restrict__ counts) {
  const uint64_t i = blockIdx.x * (uint64_t)BLK + threadIdx.x;
  uint32_t tot;
  block_excl_sum<BLK>(i < nwords ? __popc(bits[i]) : 0u, &tot);
  if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) count_prefix_kernel(uint32_t* __restrict__ counts,
                                                            uint32_t m, uint32_t* total) {
  __shared__ uint32_t part[1024];
  const uint32_t per = (m + 1023) / 1024;
  const uint32_t b = threadIdx.x * per, e = min(m, b + per);
  uint32_t s = 0;
  for (uint32_t i = b; i < e; ++i) s += counts[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const uint32_t y = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += y;
    __syncthreads();
  }
  uint32_t run = part[threadIdx.x] - s;
  for (uint32_t i = b; i < e; ++i) {
    const uint32_t c = counts[i];
    counts[i] = run;
    run += c;
  }
  if (threadIdx.x == 1023) *total = part[1023];
}

template <int BLK>
__global__ void __launch_bounds__(BLK) member_write_kernel(const uint32_t* __restrict__ bits,
                                                           uint64_t nwords,
                                                           const uint32_t* __restrict__ base,
                                                           uint64_t* __restrict__ out,
                                                           const uint64_t* out_base,
                                                           uint64_t cap) {
  const uint64_t i = blockIdx.x * (uint64_t)BLK + threadIdx.x;
  uint32_t word = i < nwords ? bits[i] : 0u, tot;
  uint64_t pos = (out_base ? *out_base : 0) + base[blockIdx.x] + block_excl_sum<BLK>(__popc(word), &tot);
  while (word) {
    const int b = __ffs(word) - 1;
    if (pos < cap) out[pos] = i * 32 + b;
    ++pos;
    word &= word - 1;
  }
}

// after minibatch k: offsets[k + 1] = offsets[k] + its member total
__global__ void advance_offset_kernel(const uint32_t* __restrict__ total, uint64_t* offsets,
                                      uint64_t k) {
  if (threadIdx.x == 0 && blockIdx.x == 0) offsets[k + 1] = offsets[k] + *total;
}

uint64_t host_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

}  // namespace tgb

using namespace tgb;

struct tg_sampler {
  tg_ctx* ctx = nullptr;
  SGraphView g;  // the graph the sampler reads (a plain device graph, or a tiered one)
  const tg_sgraph* sg = nullptr;          // the tiered graph, when there is one
  unsigned long long* reads = nullptr;    // device: ids read per tier (shared by the lanes)
  uint64_t n = 0;
  uint32_t* layer_mark = nullptr;   // n
  uint32_t* member_bits = nullptr;  // ceil(n / 32)
  uint64_t nwords = 0;
  uint32_t* buf[2] = {nullptr, nullptr};
  uint64_t buf_cap = 0;
  uint32_t* picks = nullptr;
  uint64_t picks_cap = 0;
  uint32_t* small = nullptr;  // counters
  uint32_t* blk = nullptr;    // compaction block counts
  uint32_t stamp = 0;
  // the stream this sampler state works on: the context's, or a lane's own
  cudaStream_t stream = nullptr;
  // tg_sample_batches lanes: independent sampler states (stamps, member
  // bits, frontiers) on their own streams, so consecutive minibatches expand
  // concurrently; lane 0 is this object. Created on first use.
  std::vector<tg_sampler*> lanes;
  bool is_lane = false;
  cudaEvent_t ev = nullptr;  // lane: its last batch's compaction is done
};

namespace {

void ensure(uint32_t** p, uint64_t* cap, uint64_t want) {
  if (*cap >= want) return;
  cudaFree(*p);
  *p = nullptr;
  want = std::max<uint64_t>(want, 1024);
  TGB_CUDA(tgb::dev_malloc(p, sizeof(uint32_t) * want));
  *cap = want;
}

uint32_t next_stamp(tg_sampler* s) {
  if (s->stamp >= 0xFFFFFFF0u) {  // wrap: forget every old stamp
    TGB_CUDA(cudaMemsetAsync(s->layer_mark, 0, 4 * s->n, s->stream));
    s->stamp = 0;
  }
  return ++s->stamp;
}

// Concurrent sampler states for tg_sample_batches (TIERGRAPH_SAMPLER_LANES,
// default 4).
uint32_t sampler_lanes() {
  const char* v = std::getenv("TIERGRAPH_SAMPLER_LANES");
  const int n = v ? std::atoi(v) : 4;
  return static_cast<uint32_t>(std::max(1, std::min(n, 16)));
}

// Per-state device buffers (layer stamps, member bits, counters).
void sampler_alloc(tg_sampler* s) {
  TGB_CUDA(tgb::dev_malloc(&s->layer_mark, 4 * std::max<uint64_t>(s->n, 1)));
  s->nwords = std::max<uint64_t>((s->n + 31) / 32, 1);
  TGB_CUDA(tgb::dev_malloc(&s->member_bits, 4 * s->nwords));
  TGB_CUDA(cudaMemsetAsync(s->layer_mark, 0, 4 * std::max<uint64_t>(s->n, 1), s->stream));
  TGB_CUDA(cudaMemsetAsync(s->member_bits, 0, 4 * s->nwords, s->stream));
  TGB_CUDA(tgb::dev_malloc(&s->small, 256));
  const uint64_t nblk = (s->nwords + kCompactBlock - 1) / kCompactBlock;
  TGB_CUDA(tgb::dev_malloc(&s->blk, 4 * std::max<uint64_t>(nblk, 1)));
}

}  // namespace

extern "C" {
int tg_sampler_destroy(tg_sampler* s);

int tg_sampler_create(tg_ctx* ctx, const tg_graph* gt, tg_sampler** out) {
  return guard([&] {
    if (!ctx || !gt || !out) domain_error("tg_sampler_create: null argument");
    DeviceGuard dg(ctx->device);
    auto* s = new tg_sampler;
    s->ctx = ctx;
    s->stream = ctx->stream;
    s->n = tg_graph_num_nodes(gt);
    // an untiered graph: every row "replicated" in this device's HBM
    s->g.off = tg_graph_offsets32(gt);
    s->g.rep = tg_graph_targets32(gt);
    s->g.lb = s->g.mb = s->g.n = static_cast<uint32_t>(s->n);
    try {
      sampler_alloc(s);
    } catch (...) {
      tg_sampler_destroy(s);
      throw;
    }
    *out = s;
  });
}

int tg_sampler_create_tiered(tg_ctx* ctx, const tg_sgraph* sg, tg_sampler** out) {
  return guard([&] {
    if (!ctx || !sg || !out) domain_error("tg_sampler_create_tiered: null argument");
    if (sg->ctx->device != ctx->device)
      domain_error("tg_sampler_create_tiered: the tiered graph lives on another device");
    DeviceGuard dg(ctx->device);
    auto* s = new tg_sampler;
    s->ctx = ctx;
    s->stream = ctx->stream;
    s->n = sg->n;
    s->sg = sg;
    try {
      TGB_CUDA(tgb::dev_malloc(&s->reads, 3 * sizeof(unsigned long long)));
      TGB_CUDA(cudaMemsetAsync(s->reads, 0, 3 * sizeof(unsigned long long), s->stream));
      s->g = sg->view();
      s->g.reads = s->reads;
      sampler_alloc(s);
    } catch (...) {
      tg_sampler_destroy(s);
      throw;
    }
    *out = s;
  });
}

int tg_sampler_structure_reads(tg_sampler* s, uint64_t* out, int reset) {
  return guard([&] {
    if (!s || !out) domain_error("tg_sampler_structure_reads: null argument");
    if (!s->reads) domain_error("tg_sampler_structure_reads: the sampler's graph is not tiered");
    DeviceGuard dg(s->ctx->device);
    TGB_CUDA(cudaMemcpyAsync(out, s->reads, 3 * 8, cudaMemcpyDeviceToHost, s->stream));
    if (reset) TGB_CUDA(cudaMemsetAsync(s->reads, 0, 3 * 8, s->stream));
    TGB_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int tg_sampler_destroy(tg_sampler* s) {
  if (!s) return TG_OK;
  DeviceGuard dg(s->ctx->device);
  cudaStreamSynchronize(s->stream);
  for (tg_sampler* l : s->lanes) tg_sampler_destroy(l);
  if (s->is_lane) cudaStreamDestroy(s->stream);
  if (s->ev) cudaEventDestroy(s->ev);
  cudaFree(s->layer_mark);
  cudaFree(s->member_bits);
  cudaFree(s->buf[0]);
  cudaFree(s->buf[1]);
  cudaFree(s->picks);
  cudaFree(s->small);
  cudaFree(s->blk);
  if (!s->is_lane) cudaFree(s->reads);
  delete s;
  return TG_OK;
}

}  // extern "C"

namespace {

struct ExpandOut {
  unsigned long long* counts = nullptr;  // device, n
  int count_raw = 0;
  uint64_t* raw = nullptr;  // device
  uint64_t raw_cap = 0;
};

void check_fanouts(const uint32_t* fanouts, uint32_t nf) {  // sampling.cpp:18-25
  if (nf == 0) domain_error("fanouts must be non-empty");
  if (nf > 5)
    domain_error("fanout depth " + std::to_string(nf) + " exceeds the supported maximum of 5");
  for (uint32_t l = 0; l < nf; ++l)
    if (fanouts[l] < 1) domain_error("every fanout must be >= 1");
}

// Small device counters: [0] seed frontier size, [1 + l] layer l's new
// frontier size, [8] member total; u64 [5] first bad seed index, u64 [6] raw
// draws (as u32 indices 10..13).
constexpr int kSmallBad = 10, kSmallRaw = 12, kSmallTotal = 8, kSmallOrderBad = 14;

// First out-of-range seed of a whole batch order (sticky over every batch of a
// tg_sample_batches call; expand()'s own slot is per batch).
__global__ void order_range_kernel(const uint64_t* __restrict__ order, uint64_t m, uint64_t n,
                                   unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (order[i] >= n) atomicMin(bad, (unsigned long long)i);
}

// build_minibatch (sampling.cpp:56-90) on the device, stream-ordered with no
// host round trip: every layer's grid covers an upper bound of its frontier
// and the kernel reads the actual size from the device. Returns an upper
// bound of the member count.
uint64_t expand(tg_sampler* s, const uint64_t* sd, uint64_t ns, const uint32_t* fanouts, uint32_t nf,
                uint64_t rng_seed, uint64_t epoch, uint64_t batch, const ExpandOut& o) {
  if (ns == 0) domain_error("build_minibatch: seeds must be non-empty");
  tg_ctx* ctx = s->ctx;
  const uint64_t n = s->n;
  if (s->sg) {  // peers may have been attached since the sampler was made
    s->g = s->sg->view();
    s->g.reads = s->reads;
  }
  uint64_t cap0 = s->buf_cap;
  ensure(&s->buf[0], &cap0, n + 1);
  uint64_t cap1 = s->buf_cap;
  ensure(&s->buf[1], &cap1, n + 1);
  s->buf_cap = std::min(cap0, cap1);
  uint32_t* cnt = s->small;
  auto* bad = reinterpret_cast<unsigned long long*>(s->small + kSmallBad);
  auto* raw_n = reinterpret_cast<unsigned long long*>(s->small + kSmallRaw);
  TGB_CUDA(cudaMemsetAsync(cnt, 0, 4 * 10, s->stream));
  TGB_CUDA(cudaMemsetAsync(bad, 0xff, 8, s->stream));
  TGB_CUDA(cudaMemsetAsync(raw_n, 0, 8, s->stream));
  TGB_CUDA(cudaMemsetAsync(s->member_bits, 0, 4 * s->nwords, s->stream));
  uint32_t lstamp = next_stamp(s);
  seed_kernel<<<grid_for(ns, 256), 256, 0, s->stream>>>(sd, ns, n, s->layer_mark, lstamp,
                                                         s->member_bits, s->buf[0], cnt, bad,
                                                         o.counts, o.count_raw, o.raw, raw_n,
                                                         o.raw_cap);
  TGB_LAUNCHED();
  uint64_t f = std::min<uint64_t>(ns, n);  // frontier bound
  uint64_t members = f;
  const uint64_t key0 = host_mix64(rng_seed ^ 0x6A09E667F3BCC908ull);  // rng.hpp:23-28
  int cur = 0;
  for (uint32_t layer = 0; layer < nf && f > 0; ++layer) {
    const uint32_t k = fanouts[layer];
    uint64_t key = key0;
    const uint64_t coords[4] = {0x534Dull, epoch, batch, layer};  // sampling.cpp:35-37
    for (uint64_t c : coords) key = host_mix64(key ^ host_mix64(c));
    if (f * k > (1ull << 28)) {
      // a huge bound (wide fanouts on a big graph): size the picks by the
      // actual frontier instead (one host round trip)
      uint32_t hf = 0;
      TGB_CUDA(cudaMemcpyAsync(&hf, cnt + layer, 4, cudaMemcpyDeviceToHost, s->stream));
      TGB_CUDA(cudaStreamSynchronize(s->stream));
      f = hf;
    }
    ensure(&s->picks, &s->picks_cap, std::max<uint64_t>(f * k, 1));
    lstamp = next_stamp(s);
    SampleArgs a{s->g, s->buf[cur], cnt + layer, k, key, s->picks, s->layer_mark, lstamp,
                 s->member_bits, s->buf[cur ^ 1], cnt + layer + 1, o.counts, o.count_raw, o.raw,
                 raw_n, o.raw_cap};
    sample_layer_kernel<<<grid_for(f, 256, ctx->num_sms * 16), 256, 0, s->stream>>>(a);
    TGB_LAUNCHED();
    f = std::min<uint64_t>(n, f * k);
    members += f;
    cur ^= 1;
  }
  return std::min<uint64_t>(members, n);
}

// The stamped members in id order into out_dev (device, >= bound entries);
// the total is left in s->small[kSmallTotal]. No host round trip.
// `wait` (optional) is a cudaEvent the write waits for: the member count and
// its block prefix do not depend on the output offset, only the write does.
void compact_members(tg_sampler* s, uint64_t* out_dev, const uint64_t* out_base = nullptr,
                     uint64_t cap = ~0ull, cudaEvent_t wait = nullptr) {
  const bool big = s->nwords > kCompactBigWords;
  const int blk = big ? kCompactBig : kCompactBlock;
  const uint64_t nblk = (s->nwords + blk - 1) / blk;
  if (big) member_count_kernel<kCompactBig><<<nblk, blk, 0, s->stream>>>(s->member_bits, s->nwords, s->blk);
  else member_count_kernel<kCompactBlock><<<nblk, blk, 0, s->stream>>>(s->member_bits, s->nwords, s->blk);
  TGB_LAUNCHED();
  count_prefix_kernel<<<1, 1024, 0, s->stream>>>(s->blk, static_cast<uint32_t>(nblk),
                                                   s->small + kSmallTotal);
  TGB_LAUNCHED();
  if (wait) TGB_CUDA(cudaStreamWaitEvent(s->stream, wait, 0));
  if (big)
    member_write_kernel<kCompactBig><<<nblk, blk, 0, s->stream>>>(s->member_bits, s->nwords, s->blk,
                                                                  out_dev, out_base, cap);
  else
    member_write_kernel<kCompactBlock><<<nblk, blk, 0, s->stream>>>(s->member_bits, s->nwords,
                                                                    s->blk, out_dev, out_base, cap);
  TGB_LAUNCHED();
}

struct SmallOut {
  uint32_t total;
  unsigned long long bad, raw_n;
};

SmallOut read_small(tg_sampler* s) {
  uint32_t h[16];
  TGB_CUDA(cudaMemcpyAsync(h, s->small, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
  TGB_CUDA(cudaStreamSynchronize(s->stream));
  SmallOut r;
  r.total = h[kSmallTotal];
  std::memcpy(&r.bad, h + kSmallBad, 8);
  std::memcpy(&r.raw_n, h + kSmallRaw, 8);
  return r;
}

void check_seeds(tg_sampler* s, const uint64_t* sd, const SmallOut& r) {
  if (r.bad != ~0ull) {
    uint64_t v = 0;
    TGB_CUDA(cudaMemcpy(&v, sd + r.bad, 8, cudaMemcpyDeviceToHost));
    domain_error("seed " + std::to_string(v) + " out of range");  // sampling.cpp:61-62
  }
}

}  // namespace

extern "C" {

int tg_sample_minibatch(tg_sampler* s, const uint64_t* seeds, uint64_t ns, const uint32_t* fanouts,
                        uint32_t nf, uint64_t rng_seed, uint64_t epoch, uint64_t batch,
                        uint64_t* out, uint64_t cap, uint64_t* out_n) {
  return guard([&] {
    check_fanouts(fanouts, nf);
    if (ns == 0) domain_error("build_minibatch: seeds must be non-empty");
    tg_ctx* ctx = s->ctx;
    DeviceGuard dg(ctx->device);
    const uint64_t* sd = dev_in(ctx, seeds, ns, kStageIn0);
    const uint64_t bound = expand(s, sd, ns, fanouts, nf, rng_seed, epoch, batch, ExpandOut{});
    uint64_t* md = ctx->scratch_t<uint64_t>(kStageOut1, std::max<uint64_t>(bound, 1));
    compact_members(s, md);
    const SmallOut r = read_small(s);  // the one host round trip
    check_seeds(s, sd, r);
    *out_n = r.total;
    if (r.total > cap)
      domain_error("tg_sample_minibatch: " + std::to_string(r.total) +
                   " members exceed the output capacity " + std::to_string(cap));
    if (r.total) {
      TGB_CUDA(cudaMemcpyAsync(out, md, 8ull * r.total, cudaMemcpyDefault, ctx->stream));
      ctx->sync();
    }
  });
}

int tg_sample_minibatch_raw(tg_sampler* s, const uint64_t* seeds, uint64_t ns,
                            const uint32_t* fanouts, uint32_t nf, uint64_t rng_seed,
                            uint64_t epoch, uint64_t batch, uint64_t* out, uint64_t cap,
                            uint64_t* out_n, uint64_t* raw, uint64_t raw_cap, uint64_t* raw_n) {
  return guard([&] {
    check_fanouts(fanouts, nf);
    if (ns == 0) domain_error("build_minibatch: seeds must be non-empty");
    tg_ctx* ctx = s->ctx;
    DeviceGuard dg(ctx->device);
    const uint64_t* sd = dev_in(ctx, seeds, ns, kStageIn0);
    uint64_t* rd = ctx->scratch_t<uint64_t>(kStageOut0, std::max<uint64_t>(raw_cap, 1));
    ExpandOut o;
    o.raw = rd;
    o.raw_cap = raw_cap;
    const uint64_t bound = expand(s, sd, ns, fanouts, nf, rng_seed, epoch, batch, o);
    uint64_t* md = ctx->scratch_t<uint64_t>(kStageOut1, std::max<uint64_t>(bound, 1));
    compact_members(s, md);
    const SmallOut r = read_small(s);
    check_seeds(s, sd, r);
    *raw_n = r.raw_n;
    *out_n = r.total;
    if (r.total > cap || r.raw_n > raw_cap)
      domain_error("tg_sample_minibatch_raw: output capacity exceeded");
    if (r.total) TGB_CUDA(cudaMemcpyAsync(out, md, 8ull * r.total, cudaMemcpyDefault, ctx->stream));
    if (r.raw_n) TGB_CUDA(cudaMemcpyAsync(raw, rd, 8ull * r.raw_n, cudaMemcpyDefault, ctx->stream));
    ctx->sync();
  });
}

int tg_sample_batches(tg_sampler* s, const uint64_t* order, uint64_t n_order, uint64_t batch_size,
                      uint64_t first_batch, uint64_t nbatches, const uint32_t* fanouts,
                      uint32_t nf, uint64_t rng_seed, uint64_t epoch, uint64_t* out_members,
                      uint64_t cap, uint64_t* out_offsets) {
  return guard([&] {
    // run_training_trace's batching (sampling.cpp:106-115): batch b's seeds are
    // order[b*B, (b+1)*B), expanded by build_minibatch with BatchRng{seed, epoch, b}
    check_fanouts(fanouts, nf);
    if (batch_size < 1) domain_error("batch_size must be >= 1");
    const uint64_t nb_all = (n_order + batch_size - 1) / batch_size;
    if (first_batch + nbatches > nb_all)
      domain_error("batches [" + std::to_string(first_batch) + ", " +
                   std::to_string(first_batch + nbatches) + ") exceed the " +
                   std::to_string(nb_all) + " batches of the order");
    tg_ctx* ctx = s->ctx;
    DeviceGuard dg(ctx->device);
    // only the called batches' seeds cross to the device (a host order of a
    // whole epoch -- 11M ids at C3 -- is not re-sent for every 32 batches);
    // od is indexed by order position either way
    const uint64_t beg0 = first_batch * batch_size;
    const uint64_t m = std::min(n_order, (first_batch + nbatches) * batch_size) - beg0;
    const uint64_t* od = dev_in(ctx, order + beg0, m, kStageIn1) - beg0;
    DevOut<uint64_t> offs(ctx, out_offsets, nbatches + 1, kStageOut0);
    TGB_CUDA(cudaMemsetAsync(offs.dev(), 0, 8, ctx->stream));
    uint64_t* md = out_members;
    const bool host_out = !is_device_ptr(out_members);
    if (host_out) md = ctx->scratch_t<uint64_t>(kScratchA, std::max<uint64_t>(cap, 1));
    // Lanes: batch k expands on lane k % L, each lane a sampler state on its
    // own stream, so L minibatches expand at once (one expansion is a chain
    // of small latency-bound kernels). The compactions stay in batch order:
    // batch k's waits for batch k-1's (its output offset is k-1's end).
    const uint32_t L = static_cast<uint32_t>(std::min<uint64_t>(sampler_lanes(), std::max<uint64_t>(nbatches, 1)));
    while (s->lanes.size() + 1 < L) {
      auto* l = new tg_sampler;
      l->ctx = ctx;
      l->n = s->n;
      l->g = s->g;
      l->sg = s->sg;
      l->reads = s->reads;
      l->is_lane = true;
      s->lanes.push_back(l);
      TGB_CUDA(cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking));
      TGB_CUDA(cudaEventCreateWithFlags(&l->ev, cudaEventDisableTiming));
      sampler_alloc(l);
    }
    if (!s->ev) TGB_CUDA(cudaEventCreateWithFlags(&s->ev, cudaEventDisableTiming));
    auto lane = [&](uint64_t k) { return k % L == 0 ? s : s->lanes[k % L - 1]; };
    // every seed of the called batches range-checked once (sampling.cpp:61-62);
    // the first offending position is read back with the output total
    auto* obad = reinterpret_cast<unsigned long long*>(s->small + kSmallOrderBad);
    TGB_CUDA(cudaMemsetAsync(obad, 0xff, 8, ctx->stream));
    if (m) {
      order_range_kernel<<<grid_for(m, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
          od + beg0, m, s->n, obad);
      TGB_LAUNCHED();
    }
    unsigned long long first_bad = ~0ull;
    TGB_CUDA(cudaMemcpyAsync(&first_bad, obad, 8, cudaMemcpyDeviceToHost, ctx->stream));
    // inputs ready (order, offsets[0]) before any lane starts
    TGB_CUDA(cudaEventRecord(s->ev, ctx->stream));
    for (uint32_t i = 1; i < L; ++i) TGB_CUDA(cudaStreamWaitEvent(s->lanes[i - 1]->stream, s->ev, 0));
    for (uint64_t k = 0; k < nbatches; ++k) {
      tg_sampler* ls = lane(k);
      const uint64_t b = first_batch + k;
      const uint64_t beg = b * batch_size, len = std::min(batch_size, n_order - beg);
      expand(ls, od + beg, len, fanouts, nf, rng_seed, epoch, b, ExpandOut{});
      compact_members(ls, md, offs.dev() + k, cap, k > 0 && L > 1 ? lane(k - 1)->ev : nullptr);
      advance_offset_kernel<<<1, 32, 0, ls->stream>>>(ls->small + kSmallTotal, offs.dev(), k);
      TGB_LAUNCHED();
      if (L > 1) TGB_CUDA(cudaEventRecord(ls->ev, ls->stream));
    }
    for (uint32_t i = 1; i < L; ++i) TGB_CUDA(cudaStreamWaitEvent(ctx->stream, s->lanes[i - 1]->ev, 0));
    uint64_t total = 0;
    TGB_CUDA(cudaMemcpyAsync(&total, offs.dev() + nbatches, 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (first_bad != ~0ull) {
      uint64_t v = 0;
      TGB_CUDA(cudaMemcpy(&v, od + beg0 + first_bad, 8, cudaMemcpyDeviceToHost));
      domain_error("seed " + std::to_string(v) + " out of range");  // sampling.cpp:61-62
    }
    if (total > cap)
      domain_error("tg_sample_batches: " + std::to_string(total) +
                   " members exceed the output capacity " + std::to_string(cap));
    if (host_out && total)
      TGB_CUDA(cudaMemcpyAsync(out_members, md, 8 * total, cudaMemcpyDeviceToHost, ctx->stream));
    offs.finish();
  });
}

int tg_sampler_trace(tg_sampler* s, const uint64_t* tid, uint64_t ntid, const uint32_t* fanouts,
                     uint32_t nf, uint64_t batch_size, uint64_t epochs, uint64_t rng_seed,
                     int dedup_per_batch, uint64_t* counts) {
  return guard([&] {
    // run_training_trace, sampling.cpp:92-140 (tid already validated by the caller's
    // TrainIdSet; ids are range-checked here)
    check_fanouts(fanouts, nf);
    if (ntid == 0) domain_error("run_training_trace: train id set is empty");
    if (batch_size < 1) domain_error("batch_size must be >= 1");
    if (epochs < 1) domain_error("epochs must be >= 1");
    tg_ctx* ctx = s->ctx;
    DeviceGuard dg(ctx->device);
    const uint64_t n = s->n;
    std::vector<uint64_t> order(ntid);
    if (is_device_ptr(tid)) {
      TGB_CUDA(cudaMemcpy(order.data(), tid, 8 * ntid, cudaMemcpyDeviceToHost));
    } else {
      std::memcpy(order.data(), tid, 8 * ntid);
    }
    for (uint64_t id : order)
      if (id >= n) domain_error("train id " + std::to_string(id) + " out of range");
    const std::vector<uint64_t> ids = order;
    DevOut<uint64_t> c(ctx, counts, n, kStageOut0);
    TGB_CUDA(cudaMemsetAsync(c.dev(), 0, 8 * std::max<uint64_t>(n, 1), ctx->stream));
    ExpandOut o;
    o.counts = reinterpret_cast<unsigned long long*>(c.dev());
    o.count_raw = dedup_per_batch ? 0 : 1;
    uint64_t* dorder = ctx->scratch_t<uint64_t>(kStageIn1, ntid);
    for (uint64_t epoch = 0; epoch < epochs; ++epoch) {
      tg_epoch_order(ids.data(), ntid, rng_seed, epoch, order.data());  // sampling.cpp:106-109
      TGB_CUDA(cudaMemcpyAsync(dorder, order.data(), 8 * ntid, cudaMemcpyHostToDevice,
                               ctx->stream));
      const uint64_t nb = (ntid + batch_size - 1) / batch_size;
      for (uint64_t b = 0; b < nb; ++b) {
        const uint64_t beg = b * batch_size, len = std::min(batch_size, ntid - beg);
        expand(s, dorder + beg, len, fanouts, nf, rng_seed, epoch, b, o);
      }
    }
    c.finish();
  });
}

}  // extern "C"
