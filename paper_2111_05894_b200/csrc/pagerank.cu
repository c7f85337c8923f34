// Hot path A, part 1: device CSR, in-degrees (K1), score init (K2) and the
// fused normalize + pull SpMV (K3) of the train-seeded reverse PageRank.
//
// Reference: proj/src/scoring.cpp:50-102 (run_iterations, reverse_pagerank,
// weighted_reverse_pagerank) and proj/src/csr_graph.cpp:89-93 (in_degrees).
//
// Bit-exactness contract (SURVEY §7 "hard parts"): every score equals the
// reference's double for double. Therefore
//   * normalized[j] = score[j] / (double)max(indeg[j],1) uses IEEE division;
//   * each row's pull is accumulated by ONE thread, left to right in CSR
//     storage order, starting from 0.0 (scoring.cpp:66-68);
//   * next = base + damp*pulled with separately rounded __dmul_rn/__dadd_rn
//     (never a DFMA; the reference build has no FMA).
// Parallelism comes from many rows per warp and from the loads: a warp owns a
// group of 32 consecutive rows, streams the group's targets window by window
// (coalesced), gathers the normalized values into shared memory, and each
// lane then sums its own row's slice of the window serially. A row that spans
// several windows keeps its partial sum in a register, so storage order is
// preserved exactly. Groups holding very long rows (a serial chain of
// DADDs) are scheduled first so their chains overlap the bulk of the work.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "internal.cuh"

struct tg_graph {
  tg_ctx* ctx = nullptr;
  uint64_t n = 0, e = 0;
  uint32_t* off = nullptr;     // n+1, u32
  uint32_t* tgt = nullptr;     // e, u32
  uint32_t* hub = nullptr;     // rows longer than kHubLen, longest first
  uint32_t n_hub = 0;
  uint32_t max_row = 0;
  uint32_t* indeg = nullptr;   // in_degrees (csr_graph.cpp:89-93), built with the device graph
};

namespace tgb {

constexpr int kGroupRows = 32;
constexpr uint32_t kHubLen = 2048;  // longer rows: one CTA each, warp-specialised
constexpr int kPrWin = 256;         // edges staged per warp per window (light path)
constexpr int kPrWarps = 8;         // warps per CTA
constexpr int kHubSlot = 512;       // doubles per ring slot (hub path)
constexpr int kHubSlots = 8;        // ring depth

// ------------------------------------------------------------ graph upload
__global__ void narrow_offsets_kernel(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                                      uint64_t n, uint64_t e, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = in[i];
    bool ok = v <= e;
    if (i == 0) ok = ok && v == 0;
    if (i == n) ok = ok && v == e;
    if (i > 0) ok = ok && in[i - 1] <= v;
    if (!ok) atomicMin(bad, (unsigned long long)i);
    out[i] = static_cast<uint32_t>(v);
  }
}

__global__ void narrow_targets_kernel(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                                      uint64_t count, uint64_t base, uint64_t n,
                                      unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = in[i];
    if (v >= n) atomicMin(bad, (unsigned long long)(base + i));
    out[i] = static_cast<uint32_t>(v);
  }
}

// Rows longer than kHubLen get a whole CTA each (hub path of K3).
__global__ void hub_rows_kernel(const uint32_t* __restrict__ off, uint64_t n,
                                uint32_t* __restrict__ hub, uint32_t* __restrict__ cnt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t len = off[i + 1] - off[i];
    if (len > kHubLen) hub[atomicAdd(cnt, 1u)] = static_cast<uint32_t>(i);
    if (len) atomicMax(cnt + 1, len);
  }
}

// ------------------------------------------------------------------ K1
// In-degree histogram. Low ids are privatised in shared memory: R-MAT hubs
// and score-reordered graphs both concentrate the heavy in-degrees there, so
// the hot counters never contend in L2.
constexpr uint32_t kPrivBins = 12288;
__global__ void __launch_bounds__(512) indeg_kernel(const uint32_t* __restrict__ tgt, uint64_t e,
                                                    uint32_t n, uint32_t* __restrict__ deg) {
  __shared__ uint32_t priv[kPrivBins];
  const uint32_t nb = n < kPrivBins ? n : kPrivBins;
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) priv[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 4; i < e; i += stride) {
    if (i + 3 < e && ((reinterpret_cast<uintptr_t>(tgt + i) & 15) == 0)) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(tgt + i));
      const uint32_t t[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (t[k] < nb) atomicAdd(&priv[t[k]], 1u);
        else atomicAdd(&deg[t[k]], 1u);
      }
    } else {
      for (uint64_t j = i; j < i + 4 && j < e; ++j) {
        const uint32_t t = tgt[j];
        if (t < nb) atomicAdd(&priv[t], 1u);
        else atomicAdd(&deg[t], 1u);
      }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x)
    if (priv[i]) atomicAdd(&deg[i], priv[i]);
}

__global__ void widen_u32_kernel(const uint32_t* __restrict__ in, uint64_t* __restrict__ out,
                                 uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

__global__ void degree_score_kernel(const uint32_t* __restrict__ off, uint64_t n,
                                    double* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<double>(off[i + 1] - off[i]);  // scoring.cpp:36
}

// ------------------------------------------------------------------ K2
// Train-id multiplicities (a TrainIdSet normally holds unique ids, but the
// reference multiplies once per listed id, scoring.cpp:97-100).
__global__ void train_mult_kernel(const uint64_t* __restrict__ tid, uint64_t ntid, uint64_t n,
                                  uint32_t* __restrict__ mult, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ntid;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t id = tid[i];
    if (id >= n) atomicMin(bad, (unsigned long long)i);
    else atomicAdd(&mult[id], 1u);
  }
}

// normalized0[j] = score0[j] / max(indeg[j],1), score0 = 1/N (* weight per
// train occurrence) — scoring.cpp:96-100 then :59-61 of the first iteration.
__global__ void pr_init_kernel(const uint32_t* __restrict__ deg, const uint32_t* __restrict__ mult,
                               uint64_t n, double init, double weight, double* __restrict__ norm0) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    double s = init;
    if (mult) {
      for (uint32_t k = mult[j]; k > 0; --k) s = __dmul_rn(s, weight);
    }
    const uint32_t d = deg[j];
    norm0[j] = __ddiv_rn(s, static_cast<double>(d > 1u ? d : 1u));
  }
}

// ------------------------------------------------------------------ K3
struct PrStepArgs {
  const uint32_t* off;
  const uint32_t* tgt;
  const uint32_t* deg;
  const double* norm_in;
  double* norm_out;
  double* score_out;
  const uint32_t* hub;
  uint32_t n_hub;
  uint32_t group_begin, group_end;  // 32-row groups overlapping [row_begin,row_end)
  uint64_t row_begin, row_end;
  double base, damp;
  int last;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void finish_row(const PrStepArgs& a, uint64_t r, double acc) {
  const double nx = __dadd_rn(a.base, __dmul_rn(a.damp, acc));  // scoring.cpp:69, no FMA
  if (a.last) {
    a.score_out[r] = nx;
  } else {
    const uint32_t d = a.deg[r];
    a.norm_out[r] = __ddiv_rn(nx, static_cast<double>(d > 1u ? d : 1u));  // scoring.cpp:61
  }
}

// Serial, in-order accumulation of v[0..cnt) into acc: loads run 8 ahead of
// the dependent DADD chain (the chain is the only serial part).
__device__ __forceinline__ double chain_add(double acc, const double* v, uint32_t cnt) {
  uint32_t i = 0;
  if (cnt >= 16) {
    double x[8], y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = v[k];
    for (; i + 16 <= cnt; i += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) y[k] = v[i + 8 + k];  // next 8 in flight
#pragma unroll
      for (int k = 0; k < 8; ++k) acc = __dadd_rn(acc, x[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = y[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = __dadd_rn(acc, x[k]);
    i += 8;
  }
  for (; i < cnt; ++i) acc = __dadd_rn(acc, v[i]);
  return acc;
}

// Hub path: one CTA per long row. Warps 1..7 stream the row's targets and
// gather the normalized values into a ring of shared-memory slots; lane 0 of
// warp 0 runs the single in-order DADD chain over the ring (mbarrier
// full/empty handshake per slot).
__device__ void hub_row(const PrStepArgs& a, uint32_t r, double* ring, uint64_t* full,
                        uint64_t* empty) {
  const uint32_t beg = a.off[r], len = a.off[r + 1] - beg;
  const uint32_t chunks = (len + kHubSlot - 1) / kHubSlot;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kHubSlots; ++s) {
      mbar_init(&full[s], kPrWarps * 32 - 32);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid < 32) {
    if (tid == 0) {
      double acc = 0.0;  // scoring.cpp:67
      for (uint32_t c = 0; c < chunks; ++c) {
        const uint32_t s = c % kHubSlots;
        mbar_wait(&full[s], (c / kHubSlots) & 1);
        const uint32_t cnt = min(kHubSlot, len - c * kHubSlot);
        acc = chain_add(acc, ring + s * kHubSlot, cnt);  // scoring.cpp:68, in order
        mbar_arrive(&empty[s]);
      }
      finish_row(a, r, acc);
    }
  } else {
    const int lt = tid - 32;
    constexpr int kLoaders = kPrWarps * 32 - 32;
    constexpr int kPer = (kHubSlot + kLoaders - 1) / kLoaders;
    for (uint32_t c = 0; c < chunks; ++c) {
      const uint32_t s = c % kHubSlots;
      if (c >= kHubSlots) mbar_wait(&empty[s], ((c / kHubSlots) - 1) & 1);
      const uint32_t base = beg + c * kHubSlot;
      const uint32_t cnt = min(kHubSlot, len - c * kHubSlot);
      uint32_t t[kPer];
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const uint32_t j = lt + k * kLoaders;
        t[k] = j < cnt ? __ldg(a.tgt + base + j) : 0u;
      }
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const uint32_t j = lt + k * kLoaders;
        if (j < cnt) ring[s * kHubSlot + j] = __ldg(a.norm_in + t[k]);
      }
      mbar_arrive(&full[s]);
    }
  }
}

// Light path: a warp owns 32 consecutive rows; rows are processed in runs of
// consecutive non-hub rows whose edges are contiguous. A run's edges stream
// through 256-edge windows: coalesced target loads and value gathers staged
// in shared memory (the next window's loads in flight while the lanes run the
// current window's chains), then each lane adds its own row's slice in order.
__device__ void light_group(const PrStepArgs& a, uint32_t group, double* buf) {
  const int lane = threadIdx.x & 31;
  const uint64_t r = (uint64_t)group * kGroupRows + lane;
  const bool in_range = r >= a.row_begin && r < a.row_end;
  uint32_t beg = 0, end = 0;
  if (in_range) {
    beg = a.off[r];
    end = a.off[r + 1];
  }
  const bool hub = in_range && end - beg > kHubLen;
  const bool mine = in_range && !hub;
  const uint32_t hub_mask = __ballot_sync(0xffffffffu, hub);
  const uint32_t mine_mask = __ballot_sync(0xffffffffu, mine);
  double acc = 0.0;  // scoring.cpp:67
  uint32_t todo = mine_mask;
  while (todo) {
    // run = lanes [first, stop) with no hub row in between
    const int first = __ffs(todo) - 1;
    const uint32_t later_hubs = hub_mask & ~((2u << first) - 1u);
    const int stop = later_hubs ? __ffs(later_hubs) - 1 : 32;
    const uint32_t run = todo & (stop == 32 ? ~0u : ((1u << stop) - 1u));
    todo &= ~run;
    const int last_lane = 31 - __clz(run);
    const uint32_t span_b = __shfl_sync(0xffffffffu, beg, first);
    const uint32_t span_e = __shfl_sync(0xffffffffu, end, last_lane);
    const bool in_run = (run >> lane) & 1u;
    constexpr int K = kPrWin / 32;
    uint32_t t1[K];
    double v[K];
    // prologue: window 0 values, window 1 targets
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint32_t e = span_b + k * 32 + lane;
      t1[k] = e < span_e ? __ldg(a.tgt + e) : 0xffffffffu;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = t1[k] != 0xffffffffu ? __ldg(a.norm_in + t1[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint32_t e = span_b + kPrWin + k * 32 + lane;
      t1[k] = e < span_e ? __ldg(a.tgt + e) : 0xffffffffu;
    }
    for (uint32_t wb = span_b; wb < span_e; wb += kPrWin) {
#pragma unroll
      for (int k = 0; k < K; ++k) buf[k * 32 + lane] = v[k];
      __syncwarp();
      // next window's gathers and the one after's targets go in flight now
      double vn[K];
#pragma unroll
      for (int k = 0; k < K; ++k) vn[k] = t1[k] != 0xffffffffu ? __ldg(a.norm_in + t1[k]) : 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t e = wb + 2 * kPrWin + k * 32 + lane;
        t1[k] = e < span_e ? __ldg(a.tgt + e) : 0xffffffffu;
      }
      if (in_run) {
        const uint32_t lo = beg > wb ? beg : wb;
        const uint32_t hi = end < wb + kPrWin ? end : wb + kPrWin;
        if (hi > lo) acc = chain_add(acc, buf + (lo - wb), hi - lo);  // in order
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < K; ++k) v[k] = vn[k];
    }
  }
  if (mine) finish_row(a, r, acc);
}

__global__ void __launch_bounds__(kPrWarps * 32) pr_step_kernel(const PrStepArgs a) {
  __shared__ __align__(16) double smem[kHubSlots * kHubSlot];  // 32 KB: hub ring / light windows
  __shared__ uint64_t bars[2 * kHubSlots];
  static_assert(kPrWarps * kPrWin <= kHubSlots * kHubSlot, "light windows must fit");
  if (blockIdx.x < a.n_hub) {  // hub CTAs first: their chains start earliest
    const uint32_t r = a.hub[blockIdx.x];
    if (r >= a.row_begin && r < a.row_end) hub_row(a, r, smem, bars, bars + kHubSlots);
    return;
  }
  const int w = threadIdx.x >> 5;
  const uint64_t g = a.group_begin + (uint64_t)(blockIdx.x - a.n_hub) * kPrWarps + w;
  if (g >= a.group_end) return;
  light_group(a, static_cast<uint32_t>(g), smem + w * kPrWin);
}

unsigned long long read_flag(tg_ctx* ctx, unsigned long long* dflag) {
  unsigned long long h = 0;
  TGB_CUDA(cudaMemcpyAsync(&h, dflag, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  return h;
}

void compute_indeg(tg_ctx* ctx, const tg_graph* g, uint32_t* deg) {
  TGB_CUDA(cudaMemsetAsync(deg, 0, sizeof(uint32_t) * std::max<uint64_t>(g->n, 1), ctx->stream));
  if (g->e == 0) return;
  const unsigned grid = grid_for(g->e / 4 + 1, 512, ctx->num_sms * 4);
  indeg_kernel<<<grid, 512, 0, ctx->stream>>>(g->tgt, g->e, static_cast<uint32_t>(g->n), deg);
  TGB_LAUNCHED();
}

// Prepares deg + norm0 for the weighted (tid != nullptr) or plain recurrence.
// Out-of-range train ids set *bad (min index) and are skipped; the caller
// checks it after the run (no synchronisation here).
void pagerank_prepare(tg_ctx* ctx, const tg_graph* g, const uint64_t* tid_dev, uint64_t ntid,
                      uint32_t* deg, double* norm0, unsigned long long* bad) {
  const uint64_t n = g->n;
  if (deg != g->indeg)
    TGB_CUDA(cudaMemcpyAsync(deg, g->indeg, 4 * n, cudaMemcpyDeviceToDevice, ctx->stream));
  const double init = 1.0 / static_cast<double>(n);  // scoring.cpp:96
  double weight = 1.0;
  uint32_t* mult = nullptr;
  if (tid_dev) {
    weight = static_cast<double>(n) / static_cast<double>(ntid);  // scoring.cpp:94-95
    mult = ctx->scratch_t<uint32_t>(kScratchF, n);
    TGB_CUDA(cudaMemsetAsync(mult, 0, sizeof(uint32_t) * n, ctx->stream));
    train_mult_kernel<<<grid_for(ntid, 256), 256, 0, ctx->stream>>>(tid_dev, ntid, n, mult, bad);
    TGB_LAUNCHED();
  }
  pr_init_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(deg, mult, n, init, weight, norm0);
  TGB_LAUNCHED();
}

void pagerank_step(tg_ctx* ctx, const tg_graph* g, const uint32_t* deg, double damp,
                   const double* nin, double* nout, double* sout, uint64_t rb, uint64_t re,
                   int last) {
  if (re <= rb) return;
  PrStepArgs a;
  a.off = g->off;
  a.tgt = g->tgt;
  a.deg = deg;
  a.norm_in = nin;
  a.norm_out = nout;
  a.score_out = sout;
  a.hub = g->hub;
  a.n_hub = g->n_hub;
  a.group_begin = static_cast<uint32_t>(rb / kGroupRows);
  a.group_end = static_cast<uint32_t>((re + kGroupRows - 1) / kGroupRows);
  a.row_begin = rb;
  a.row_end = re;
  a.base = (1.0 - damp) / static_cast<double>(g->n);  // scoring.cpp:53
  a.damp = damp;
  a.last = last;
  const uint64_t light = (a.group_end - a.group_begin + kPrWarps - 1) / kPrWarps;
  const unsigned grid = static_cast<unsigned>(a.n_hub + light);
  pr_step_kernel<<<grid, kPrWarps * 32, 0, ctx->stream>>>(a);
  TGB_LAUNCHED();
}

void check_config(uint32_t iterations, double damp) {  // scoring.cpp:42-47
  if (iterations < 1) domain_error("pagerank: iterations must be >= 1");
  if (!(damp > 0.0 && damp < 1.0))
    domain_error("pagerank: damp must lie in (0,1), got " + std::to_string(damp));
}

void run_pagerank(tg_ctx* ctx, const tg_graph* g, uint32_t iterations, double damp,
                  const uint64_t* tid, uint64_t ntid, bool weighted, double* out) {
  check_config(iterations, damp);
  if (weighted && ntid == 0)
    domain_error(
        "weighted reverse pagerank needs a non-empty train id set; "
        "use reverse_pagerank when no nodes are labeled");  // scoring.cpp:89-91
  const uint64_t n = g ? g->n : 0;
  if (n == 0) return;
  DeviceGuard dg(ctx->device);
  const uint64_t* tid_dev = weighted ? dev_in(ctx, tid, ntid, kStageIn0) : nullptr;
  uint32_t* deg = g->indeg;  // cached with the device graph
  double* na = ctx->scratch_t<double>(kScratchB, n);
  double* nb = ctx->scratch_t<double>(kScratchC, n);
  DevOut<double> o(ctx, out, n, kStageOut0);
  auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 1);
  if (weighted) TGB_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
  pagerank_prepare(ctx, g, tid_dev, ntid, deg, na, bad);
  for (uint32_t it = 0; it < iterations; ++it) {
    const bool last = it + 1 == iterations;
    pagerank_step(ctx, g, deg, damp, na, nb, o.dev(), 0, n, last ? 1 : 0);
    std::swap(na, nb);
  }
  unsigned long long hb = ~0ull;
  if (weighted) TGB_CUDA(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
  o.finish();
  if (hb != ~0ull) {
    uint64_t id = 0;
    TGB_CUDA(cudaMemcpy(&id, tid_dev + hb, sizeof(id), cudaMemcpyDeviceToHost));
    domain_error("train id " + std::to_string(id) + " out of range");  // scoring.cpp:98
  }
}

}  // namespace tgb

using namespace tgb;

extern "C" {

int tg_graph_create(tg_ctx* ctx, const uint64_t* offsets, const uint64_t* targets, uint64_t n,
                    uint64_t e, tg_graph** out) {
  return guard([&] {
    if (!ctx || !out) domain_error("tg_graph_create: null argument");
    if (n >= 0xffffffffull || e >= 0xffffffffull)
      domain_error("tg_graph_create: n and e must be < 2^32 for the u32 device layout");
    DeviceGuard dg(ctx->device);
    auto* g = new tg_graph;
    g->ctx = ctx;
    g->n = n;
    g->e = e;
    try {
      TGB_CUDA(cudaMalloc(&g->off, sizeof(uint32_t) * (n + 1)));
      TGB_CUDA(cudaMalloc(&g->tgt, sizeof(uint32_t) * std::max<uint64_t>(e, 1)));
      auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 2);
      TGB_CUDA(cudaMemsetAsync(bad, 0xff, 2 * sizeof(unsigned long long), ctx->stream));
      const uint64_t* doff = dev_in(ctx, offsets, n + 1, kStageIn0);
      narrow_offsets_kernel<<<grid_for(n + 1, 256), 256, 0, ctx->stream>>>(doff, g->off, n, e, bad);
      TGB_LAUNCHED();
      // targets: straight from device memory, or in 32M-entry chunks from the host
      const bool tdev = is_device_ptr(targets);
      const uint64_t chunk = tdev ? std::max<uint64_t>(e, 1) : (32ull << 20);
      for (uint64_t base = 0; base < e; base += chunk) {
        const uint64_t cnt = std::min(chunk, e - base);
        const uint64_t* src = targets + base;
        if (!tdev) {
          auto* st = ctx->scratch_t<uint64_t>(kStageIn1, cnt);
          TGB_CUDA(cudaMemcpyAsync(st, src, cnt * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                   ctx->stream));
          src = st;
        }
        narrow_targets_kernel<<<grid_for(cnt, 256), 256, 0, ctx->stream>>>(src, g->tgt + base, cnt,
                                                                           base, n, bad + 1);
        TGB_LAUNCHED();
      }
      unsigned long long hb[2];
      TGB_CUDA(cudaMemcpyAsync(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      if (hb[0] != ~0ull)
        format_error("csr: offsets invalid at index " + std::to_string(hb[0]) +
                     " (need offsets[0]==0, monotone, offsets[num_nodes]==num_edges)");
      if (hb[1] != ~0ull)
        format_error("csr: target out of range at edge " + std::to_string(hb[1]));
      // hub rows (one CTA each in K3), longest first
      TGB_CUDA(cudaMalloc(&g->hub, sizeof(uint32_t) * (std::max<uint64_t>(n, 1) + 2)));
      uint32_t* cnt = g->hub + std::max<uint64_t>(n, 1);
      TGB_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(uint32_t), ctx->stream));
      if (n) {
        hub_rows_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(g->off, n, g->hub, cnt);
        TGB_LAUNCHED();
      }
      uint32_t hc[2];
      TGB_CUDA(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      g->n_hub = hc[0];
      g->max_row = hc[1];
      if (g->n_hub) {
        std::vector<uint32_t> rows(g->n_hub), offs(n + 1);
        TGB_CUDA(cudaMemcpy(rows.data(), g->hub, 4 * rows.size(), cudaMemcpyDeviceToHost));
        std::vector<std::pair<uint32_t, uint32_t>> lens;
        for (uint32_t r : rows) {
          uint32_t o2[2];
          TGB_CUDA(cudaMemcpy(o2, g->off + r, 8, cudaMemcpyDeviceToHost));
          lens.push_back({o2[1] - o2[0], r});
        }
        std::sort(lens.begin(), lens.end(), [](auto x, auto y) {
          return x.first != y.first ? x.first > y.first : x.second < y.second;
        });
        for (size_t i = 0; i < lens.size(); ++i) rows[i] = lens[i].second;
        TGB_CUDA(cudaMemcpy(g->hub, rows.data(), 4 * rows.size(), cudaMemcpyHostToDevice));
      }
      TGB_CUDA(cudaMalloc(&g->indeg, sizeof(uint32_t) * std::max<uint64_t>(n, 1)));
      compute_indeg(ctx, g, g->indeg);
      ctx->sync();
    } catch (...) {
      tg_graph_destroy(g);
      throw;
    }
    *out = g;
  });
}

int tg_graph_destroy(tg_graph* g) {
  if (!g) return TG_OK;
  cudaFree(g->off);
  cudaFree(g->tgt);
  cudaFree(g->hub);
  cudaFree(g->indeg);
  delete g;
  return TG_OK;
}

uint64_t tg_graph_num_nodes(const tg_graph* g) { return g ? g->n : 0; }
uint64_t tg_graph_num_edges(const tg_graph* g) { return g ? g->e : 0; }
const uint32_t* tg_graph_offsets32(const tg_graph* g) { return g ? g->off : nullptr; }
const uint32_t* tg_graph_targets32(const tg_graph* g) { return g ? g->tgt : nullptr; }

int tg_degree_score(tg_ctx* ctx, const tg_graph* g, double* out) {
  return guard([&] {
    if (!g->n) return;
    DeviceGuard dg(ctx->device);
    DevOut<double> o(ctx, out, g->n, kStageOut0);
    degree_score_kernel<<<grid_for(g->n, 256), 256, 0, ctx->stream>>>(g->off, g->n, o.dev());
    TGB_LAUNCHED();
    o.finish();
  });
}

int tg_in_degrees(tg_ctx* ctx, const tg_graph* g, uint64_t* out) {
  return guard([&] {
    if (!g->n) return;
    DeviceGuard dg(ctx->device);
    uint32_t* deg = ctx->scratch_t<uint32_t>(kScratchA, g->n);
    compute_indeg(ctx, g, deg);  // recomputed on purpose: this is the in_degrees() API
    DevOut<uint64_t> o(ctx, out, g->n, kStageOut0);
    widen_u32_kernel<<<grid_for(g->n, 256), 256, 0, ctx->stream>>>(deg, o.dev(), g->n);
    TGB_LAUNCHED();
    o.finish();
  });
}

int tg_reverse_pagerank(tg_ctx* ctx, const tg_graph* g, uint32_t iterations, double damp,
                        double* out) {
  return guard([&] { run_pagerank(ctx, g, iterations, damp, nullptr, 0, false, out); });
}

int tg_weighted_reverse_pagerank(tg_ctx* ctx, const tg_graph* g, uint32_t iterations,
                                 double damp, const uint64_t* tid, uint64_t ntid, double* out) {
  return guard([&] { run_pagerank(ctx, g, iterations, damp, tid, ntid, true, out); });
}

int tg_pagerank_prepare_async(tg_ctx* ctx, const tg_graph* g, const uint64_t* tid_dev,
                              uint64_t ntid, uint32_t* indeg_dev, double* norm0_dev) {
  return guard([&] {
    if (tid_dev && ntid == 0) domain_error("weighted reverse pagerank needs a non-empty train id set");
    if (!g->n) return;
    DeviceGuard dg(ctx->device);
    // train ids must be in range here (the synchronous entry points check them)
    auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 1);
    pagerank_prepare(ctx, g, tid_dev, ntid, indeg_dev, norm0_dev, bad);
  });
}

int tg_pagerank_step_async(tg_ctx* ctx, const tg_graph* g, const uint32_t* indeg_dev,
                           double damp, const double* norm_in_dev, double* norm_out_dev,
                           double* score_out_dev, uint64_t row_begin, uint64_t row_end,
                           int last) {
  return guard([&] {
    if (row_end > g->n || row_begin > row_end) domain_error("pagerank step: bad row range");
    DeviceGuard dg(ctx->device);
    pagerank_step(ctx, g, indeg_dev, damp, norm_in_dev, norm_out_dev, score_out_dev, row_begin,
                  row_end, last);
  });
}

}  // extern "C"
