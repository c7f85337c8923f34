// Hot path A, part 2: hot-set selection — validate + key transform (K4), a
// stable LSD radix sort of (key, id) (K5), and the permutation scatter (K6).
//
// Reference: proj/src/scoring.cpp:104-115 (score_ordering: reject non-finite
// or negative scores, sort ids by score descending, ties by ascending id) and
// proj/src/reorder.cpp:23-29 (permutation_from_scores: new_id_of[order[r]]=r).
//
// Key = ~bits(score) with -0.0 canonicalised to +0.0: for non-negative finite
// doubles the IEEE bit pattern is monotone, so ascending keys = descending
// scores, and equal scores (including +-0) share a key. A stable sort over
// ids presented in ascending order reproduces the id tie-break exactly.
//
// Sort: 8-bit LSD digits, ONE kernel per pass (onesweep: stable block-local
// ranking via warp __match_any_sync, the earlier tiles' digit counts by
// decoupled look-back, a digit-ordered shared-memory tile written out in
// coalesced runs). One upfront pass builds all eight digit histograms (the
// digits' global bases); passes whose digit is
// constant over the whole input are skipped on the device (no host sync), with
// the ping-pong buffer choice planned on the device as well.
#include <cuda_runtime.h>

#include <string>

#include "internal.cuh"

namespace tgb {

constexpr int kRsWarps = 8;
constexpr int kRsIpt = 16;
constexpr int kRsTile = kRsWarps * 32 * kRsIpt;  // 4096 items per CTA

struct RadixPlan {
  int skip[8];
  int src[8];
  int final_src;
};

__device__ __forceinline__ uint64_t score_key(double s) {
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(s));
  if (b == 0x8000000000000000ull) b = 0;  // -0.0 == +0.0 (scoring.cpp:111)
  return ~b;
}

// K4a: the smallest key (kmin) and the largest. Sorting key - kmin orders
// and ties exactly like key, and digits above the top bit of (kmax - kmin)
// become constant zero, so the planner skips their passes. The largest key
// is the lowest score.
__global__ void __launch_bounds__(256) key_range_kernel(const double* __restrict__ s, uint64_t n,
                                                        unsigned long long* kmin,
                                                        unsigned long long* kmax) {
  unsigned long long lo = ~0ull, hi = 0ull;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = score_key(__ldcs(s + i));
    lo = min(lo, k);
    hi = max(hi, k);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(kmin, lo);
    atomicMax(kmax, hi);
  }
}

// The lowest score ties (key == kmax) go last in id order: reverse PageRank
// gives every node without out-edges exactly the teleport score (1-d)/N, the
// minimum (scoring.cpp:65-70 with an empty sum) -- 61 % of the C3 nodes. They
// are compacted out of the sort (K4b/K4c) and written behind its result.
constexpr int kKpIpt = 16;
constexpr int kKpTile = 256 * kKpIpt;
__global__ void __launch_bounds__(256) key_tile_count_kernel(const double* __restrict__ s,
                                                             uint64_t n,
                                                             const unsigned long long* kmax,
                                                             uint64_t* __restrict__ cnt) {
  __shared__ uint32_t c;
  const uint64_t nt = (n + kKpTile - 1) / kKpTile;
  const unsigned long long km = *kmax;
  for (uint64_t t = blockIdx.x; t < nt; t += gridDim.x) {
    if (threadIdx.x == 0) c = 0;
    __syncthreads();
    uint32_t mine = 0;
#pragma unroll
    for (int k = 0; k < kKpIpt; ++k) {
      const uint64_t i = t * kKpTile + k * 256 + threadIdx.x;
      if (i < n && score_key(__ldcs(s + i)) != km) ++mine;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&c, mine);
    __syncthreads();
    if (threadIdx.x == 0) cnt[t] = c;
    __syncthreads();
  }
}

// K4c: validate, compact the keys below kmax (key - kmin, id) in id order to
// [0, m) with all 8 digit histograms; the ids of the kmax ties in id order to
// [m, n) of both value buffers (the sort's result lands in either).
__global__ void __launch_bounds__(256) key_prep_compact_kernel(
    const double* __restrict__ s, uint64_t n, const unsigned long long* __restrict__ kmin,
    const unsigned long long* __restrict__ kmax, const uint64_t* __restrict__ off,
    uint64_t* __restrict__ keys, uint32_t* __restrict__ vals, uint32_t* __restrict__ vals_alt,
    uint32_t* __restrict__ hist, unsigned long long* bad) {
  __shared__ uint32_t h[8][256];
  __shared__ uint32_t wc[8];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
  const uint64_t nt = (n + kKpTile - 1) / kKpTile;
  const uint64_t m = off[nt];
  const unsigned long long km = *kmax, k0 = *kmin;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint64_t t = blockIdx.x; t < nt; t += gridDim.x) {
    const uint64_t base = off[t];
    uint32_t run = 0;  // low keys of this tile in the rounds so far (same in every thread)
    for (int k = 0; k < kKpIpt; ++k) {  // index order: round k, then thread
      const uint64_t i = t * kKpTile + k * 256 + threadIdx.x;
      bool ok = i < n, low = false;
      unsigned long long key = 0;
      if (ok) {
        const double v = s[i];
        if (!(isfinite(v) && v >= 0.0)) atomicMin(bad, (unsigned long long)i);
        key = score_key(v);
        low = key != km;
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, low);
      if (lane == 0) wc[w] = __popc(bal);
      __syncthreads();
      uint32_t before = run, total = 0;
      for (int q = 0; q < 8; ++q) {
        if (q < w) before += wc[q];
        total += wc[q];
      }
      run += total;
      before += __popc(bal & ((1u << lane) - 1u));  // low keys of this tile before i
      if (ok) {
        if (low) {
          const uint64_t p = base + before;
          const uint64_t kk = key - k0;
          keys[p] = kk;
          vals[p] = static_cast<uint32_t>(i);
#pragma unroll
          for (int q = 0; q < 8; ++q) atomicAdd(&h[q][(kk >> (8 * q)) & 0xff], 1u);
        } else {
          const uint64_t p = m + (i - base - before);
          vals[p] = static_cast<uint32_t>(i);
          vals_alt[p] = static_cast<uint32_t>(i);
        }
      }
      __syncthreads();  // wc is rewritten by the next round
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

// K4: validate (scoring.cpp:105-107), build keys (- kmin)/ids, and all 8 digit histograms.
__global__ void __launch_bounds__(256) key_prep_kernel(const double* __restrict__ s, uint64_t n,
                                                       const unsigned long long* __restrict__ kmin,
                                                       uint64_t* __restrict__ keys,
                                                       uint32_t* __restrict__ vals,
                                                       uint32_t* __restrict__ hist,
                                                       unsigned long long* bad) {
  __shared__ uint32_t h[8][256];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = s[i];
    if (!(isfinite(v) && v >= 0.0)) atomicMin(bad, (unsigned long long)i);
    const uint64_t k = score_key(v) - *kmin;
    keys[i] = k;
    vals[i] = static_cast<uint32_t>(i);
#pragma unroll
    for (int p = 0; p < 8; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

// One 256-thread CTA: thread d checks digit value d of every pass (a pass
// whose histogram holds all n keys in one bucket is skipped).
__global__ void __launch_bounds__(256) plan_kernel(const uint32_t* __restrict__ hist, uint64_t n,
                                                   RadixPlan* plan, int keep = -1) {
  __shared__ int trivial[8];
  for (int p = 0; p < 8; ++p) {
    const int t = __syncthreads_or(hist[p * 256 + threadIdx.x] == n);
    if (threadIdx.x == 0) trivial[p] = t;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int src = 0;
  for (int p = 0; p < 8; ++p) {
    plan->skip[p] = (trivial[p] && p != keep) ? 1 : 0;  // `keep` narrows the keys: always runs
    plan->src[p] = src;
    if (!plan->skip[p]) src ^= 1;
  }
  plan->final_src = src;
}

// One onesweep pass (a single kernel per digit: no separate count and scan
// kernels). Each CTA takes the next tile id from a counter (tiles are
// claimed in launch order, so every tile waits only on tiles already
// running), ranks its 4,096 keys stably (warp rounds in index order +
// per-warp digit counters, __match_any_sync), publishes its per-digit counts
// and finds the counts of all earlier tiles by DECOUPLED LOOK-BACK over their
// published status words (flag: 1 = this tile's count, 2 = inclusive prefix
// of tiles 0..t). The digit's global base comes from the all-pass histogram
// of the key-prep kernel. The tile is then reordered by digit in shared
// memory and written out in that order (coalesced runs).
// Keys are u64 (scores) or u32 (row lengths, in-degrees, edge targets); a
// u64 sort narrows to u32 at the pass that sorts bits 32..39 (after it only
// bits 32..63 still order anything): that pass writes k >> 32, the later
// passes move 4 B keys instead of 8 B.
template <typename KIn>
constexpr int rs_scatter_smem() { return kRsTile * static_cast<int>(sizeof(KIn) + 4); }
constexpr uint64_t kStAgg = 1ull << 62, kStInc = 2ull << 62, kStMask = (1ull << 62) - 1;
template <typename KIn, typename KOut>
__global__ void __launch_bounds__(kRsWarps * 32, 3) scatter_kernel(
    void* __restrict__ k0v, uint32_t* __restrict__ v0, void* __restrict__ k1v,
    uint32_t* __restrict__ v1, uint64_t n, int pass, int shift, const RadixPlan* __restrict__ plan,
    const uint32_t* __restrict__ hist, uint64_t* __restrict__ status, uint32_t* __restrict__ tile_ctr) {
  if (plan->skip[pass]) return;
  const bool from1 = plan->src[pass] != 0;
  const KIn* kin = reinterpret_cast<const KIn*>(from1 ? k1v : k0v);
  const uint32_t* vin = from1 ? v1 : v0;
  KOut* kout = reinterpret_cast<KOut*>(from1 ? k0v : k1v);
  uint32_t* vout = from1 ? v0 : v1;
  extern __shared__ __align__(16) uint8_t rs_smem[];
  KIn* skey = reinterpret_cast<KIn*>(rs_smem);
  uint32_t* sval = reinterpret_cast<uint32_t*>(rs_smem + kRsTile * sizeof(KIn));
  __shared__ uint32_t wcnt[kRsWarps][256];
  __shared__ uint32_t doff[256];
  __shared__ uint32_t tstart[256];
  __shared__ uint32_t tile_s;
  if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr + pass, 1u);
  for (int i = threadIdx.x; i < kRsWarps * 256; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = tile_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  // tile-local 32-bit offsets; a full tile (all but the last) needs no bound checks
  const uint64_t t0 = (uint64_t)tile * kRsTile;
  const uint32_t tn = static_cast<uint32_t>(n - t0 < (uint64_t)kRsTile ? n - t0 : kRsTile);
  const bool full = tn == kRsTile;
  const uint32_t o0 = w * (32 * kRsIpt) + lane;  // + k * 32
  const KIn* kin_t = kin + t0 + o0;
  const uint32_t* vin_t = vin + t0 + o0;
  KIn key[kRsIpt];
  uint32_t val[kRsIpt];
  uint32_t rank[kRsIpt];
#pragma unroll
  for (int k = 0; k < kRsIpt; ++k) {
    const bool ok = full || o0 + k * 32 < tn;
    key[k] = ok ? kin_t[k * 32] : 0;
    val[k] = ok ? vin_t[k * 32] : 0;
  }
#pragma unroll
  for (int k = 0; k < kRsIpt; ++k) {
    const bool ok = full || o0 + k * 32 < tn;
    const uint32_t d = ok ? static_cast<uint32_t>((key[k] >> shift) & 0xff) : 256u;
    // lanes with the same digit (256 = past the end). __match_any_sync: on the
    // real C3 scores (61 % of them equal) 9.2 ms per selection against 9.8 ms
    // for the data-independent 9-ballot form, which only wins on keys with
    // few equal digits (log-normal probe: 10.15 vs 10.56 ms; profiles/r02ab,
    // r02sel)
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t pre = d < 256 ? wcnt[w][d] : 0;
    __syncwarp();
    if (d < 256 && (peers & lt) == 0) wcnt[w][d] = pre + __popc(peers);
    __syncwarp();
    rank[k] = pre + __popc(peers & lt);
  }
  __syncthreads();
  {
    const int d = threadIdx.x;  // 256 threads: one digit each
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < kRsWarps; ++ww) {
      const uint32_t c = wcnt[ww][d];
      wcnt[ww][d] = run;
      run += c;
    }
    // publish this tile's count, then look back for the earlier tiles'
    volatile uint64_t* st = status;
    st[(uint64_t)tile * 256 + d] = (tile ? kStAgg : kStInc) | run;
    // Look back four tiles per round trip: the four status words are loaded
    // together (independent L2 loads), then consumed in order up to the first
    // inclusive prefix; an unpublished one is re-read from there (spin).
    uint64_t excl = 0;
    for (int64_t j = (int64_t)tile - 1; j >= 0;) {
      uint64_t v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = j - q >= 0 ? st[(uint64_t)(j - q) * 256 + d] : (2ull << 62);  // kStInc, 0
      int q = 0;
      bool done = false;
      for (; q < 4; ++q) {
        if (!(v[q] & (kStAgg | kStInc))) break;  // not published yet
        excl += v[q] & kStMask;
        if (v[q] & kStInc) {
          done = true;
          break;
        }
      }
      if (done) break;
      j -= q;
    }
    if (tile) st[(uint64_t)tile * 256 + d] = kStInc | (excl + run);
    // the digit's global base: exclusive scan of this pass's histogram
    const uint32_t t = hist[pass * 256 + d];
    uint32_t incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    // tile-local digit start: exclusive scan of `run`
    uint32_t incl2 = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl2, o);
      if (lane >= o) incl2 += y;
    }
    __shared__ uint32_t wt[kRsWarps], st2[kRsWarps];
    if (lane == 31) {
      wt[w] = incl;
      st2[w] = incl2;
    }
    __syncthreads();
    uint32_t before = 0, before2 = 0;
    for (int k = 0; k < w; ++k) {
      before += wt[k];
      before2 += st2[k];
    }
    doff[d] = before + incl - t + static_cast<uint32_t>(excl);
    tstart[d] = before2 + incl2 - run;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kRsIpt; ++k) {
    if (full || o0 + k * 32 < tn) {
      const uint32_t d = static_cast<uint32_t>((key[k] >> shift) & 0xff);
      const uint32_t lp = tstart[d] + wcnt[w][d] + rank[k];
      skey[lp] = key[k];
      sval[lp] = val[k];
    }
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < tn; j += blockDim.x) {
    const KIn kk = skey[j];
    const uint32_t d = static_cast<uint32_t>((kk >> shift) & 0xff);
    const uint32_t pos = doff[d] + (j - tstart[d]);
    if constexpr (sizeof(KOut) < sizeof(KIn))
      kout[pos] = static_cast<KOut>(static_cast<uint64_t>(kk) >> 32);
    else
      kout[pos] = kk;
    vout[pos] = sval[j];
  }
}

// The passes of one LSD sort (keys k0/v0 in, result where plan->final_src
// says): one onesweep kernel per digit that is not constant. key_bytes 8:
// u64 keys, narrowed to u32 at pass `narrow_at` (>= 4; the plan must keep
// that pass, plan_kernel's `keep`), or never (-1); key_bytes 4: u32 keys.
template <typename KIn, typename KOut>
static void launch_pass(tg_ctx* ctx, void* k0, uint32_t* v0, void* k1, uint32_t* v1, uint64_t n,
                        int pass, int shift, const RadixPlan* plan, const uint32_t* hist,
                        uint64_t* status, uint32_t* ctr, uint32_t nblk) {
  static bool attr[TG_MAX_DEVICES] = {};
  if (!attr[ctx->device % TG_MAX_DEVICES]) {
    TGB_CUDA(cudaFuncSetAttribute(scatter_kernel<KIn, KOut>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, rs_scatter_smem<KIn>()));
    attr[ctx->device % TG_MAX_DEVICES] = true;
  }
  scatter_kernel<KIn, KOut><<<nblk, kRsWarps * 32, rs_scatter_smem<KIn>(), ctx->stream>>>(
      k0, v0, k1, v1, n, pass, shift, plan, hist, status, ctr);
  TGB_LAUNCHED();
}

void radix_passes(tg_ctx* ctx, void* k0, uint32_t* v0, void* k1, uint32_t* v1, uint64_t n,
                  int passes, const RadixPlan* plan, const uint32_t* hist, int key_bytes,
                  int narrow_at) {
  const uint32_t nblk = static_cast<uint32_t>((n + kRsTile - 1) / kRsTile);
  uint64_t* status = nullptr;
  const size_t sbytes = 8ull * 256 * nblk;
  TGB_CUDA(tgb::dev_malloc_async(reinterpret_cast<void**>(&status), sbytes + 64, ctx->stream));
  auto* ctr = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(status) + sbytes);
  TGB_CUDA(cudaMemsetAsync(ctr, 0, 64, ctx->stream));
  for (int p = 0; p < passes; ++p) {
    TGB_CUDA(cudaMemsetAsync(status, 0, sbytes, ctx->stream));
    if (key_bytes == 4)
      launch_pass<uint32_t, uint32_t>(ctx, k0, v0, k1, v1, n, p, 8 * p, plan, hist, status, ctr, nblk);
    else if (narrow_at < 0 || p < narrow_at)
      launch_pass<uint64_t, uint64_t>(ctx, k0, v0, k1, v1, n, p, 8 * p, plan, hist, status, ctr, nblk);
    else if (p == narrow_at)
      launch_pass<uint64_t, uint32_t>(ctx, k0, v0, k1, v1, n, p, 8 * p, plan, hist, status, ctr, nblk);
    else
      launch_pass<uint32_t, uint32_t>(ctx, k0, v0, k1, v1, n, p, 8 * p - 32, plan, hist, status, ctr,
                                      nblk);
  }
  TGB_CUDA(cudaFreeAsync(status, ctx->stream));
}

// K6: order[r] = id, new_id_of[id] = r (reorder.cpp:27)
__global__ void perm_kernel(const uint32_t* __restrict__ v0, const uint32_t* __restrict__ v1,
                            const RadixPlan* __restrict__ plan, uint64_t n,
                            uint64_t* __restrict__ order, uint64_t* __restrict__ new_id_of) {
  const uint32_t* v = plan->final_src ? v1 : v0;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = v[r];
    if (order) order[r] = id;
    if (new_id_of) new_id_of[id] = r;
  }
}

// K3 schedule: keys = ~len (u32 in a u64 key) of rows [rb, rb+m), vals = the
// row's offset in the range. Ascending keys = descending lengths; the sort is
// stable, so equal lengths keep ascending ids.
// (`val` non-null: key = ~val[rb+i] instead -- ids by a u32 value, descending,
// ties by id: the K3 relabelling by in-degree.)
__global__ void __launch_bounds__(256) rowlen_key_kernel(const uint32_t* __restrict__ off,
                                                         const uint32_t* __restrict__ val,
                                                         uint64_t rb, uint64_t m,
                                                         uint32_t* __restrict__ keys,
                                                         uint32_t* __restrict__ vals,
                                                         uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[4][256];
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = val ? ~val[rb + i] : ~(off[rb + i + 1] - off[rb + i]);
    keys[i] = k;
    vals[i] = static_cast<uint32_t>(i);
#pragma unroll
    for (int p = 0; p < 4; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
  // digits 4..7 of every key are 0: one full bin each
  if (blockIdx.x == 0)
    for (int p = 4 + threadIdx.x; p < 8; p += blockDim.x) hist[p * 256] = static_cast<uint32_t>(m);
}

__global__ void order_out_kernel(const uint32_t* __restrict__ v0, const uint32_t* __restrict__ v1,
                                 const RadixPlan* __restrict__ plan, uint64_t rb, uint64_t m,
                                 uint32_t* __restrict__ order) {
  const uint32_t* v = plan->final_src ? v1 : v0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    order[i] = static_cast<uint32_t>(rb + v[i]);
}

static void sort_desc_u32(tg_ctx* ctx, const uint32_t* off, const uint32_t* val, uint64_t rb,
                          uint64_t re, uint32_t* order_dev);

void sort_rows_by_length(tg_ctx* ctx, const uint32_t* off, uint64_t rb, uint64_t re,
                         uint32_t* order_dev) {
  sort_desc_u32(ctx, off, nullptr, rb, re, order_dev);
}

void sort_ids_by_value_desc(tg_ctx* ctx, const uint32_t* val, uint64_t n, uint32_t* order_dev) {
  sort_desc_u32(ctx, nullptr, val, 0, n, order_dev);
}

static void sort_desc_u32(tg_ctx* ctx, const uint32_t* off, const uint32_t* val, uint64_t rb,
                          uint64_t re, uint32_t* order_dev) {
  const uint64_t m = re - rb;
  if (m == 0) return;
  // private temporaries (stream-ordered allocations): callers may hold the
  // context's scratch slots across this call
  const size_t bytes = 4 * 4 * m + 4 * 16 + sizeof(RadixPlan) + 8 * 256 * 4 + 256;
  char* base = nullptr;
  TGB_CUDA(tgb::dev_malloc_async(reinterpret_cast<void**>(&base), bytes, ctx->stream));
  auto align = [](char* p) { return reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15)); };
  char* p = base;
  uint32_t* k0 = reinterpret_cast<uint32_t*>(p); p = align(p + 4 * m);  // u32 keys
  uint32_t* k1 = reinterpret_cast<uint32_t*>(p); p = align(p + 4 * m);
  uint32_t* v0 = reinterpret_cast<uint32_t*>(p); p = align(p + 4 * m);
  uint32_t* v1 = reinterpret_cast<uint32_t*>(p); p = align(p + 4 * m);
  auto* plan = reinterpret_cast<RadixPlan*>(p); p = align(p + sizeof(RadixPlan));
  uint32_t* hist = reinterpret_cast<uint32_t*>(p);
  TGB_CUDA(cudaMemsetAsync(hist, 0, 8 * 256 * 4, ctx->stream));
  rowlen_key_kernel<<<grid_for(m, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(off, val, rb, m,
                                                                                k0, v0, hist);
  TGB_LAUNCHED();
  plan_kernel<<<1, 256, 0, ctx->stream>>>(hist, m, plan);
  TGB_LAUNCHED();
  radix_passes(ctx, k0, v0, k1, v1, m, 4, plan, hist, 4, -1);  // digits 4..7 are constant
  order_out_kernel<<<grid_for(m, 256), 256, 0, ctx->stream>>>(v0, v1, plan, rb, m, order_dev);
  TGB_LAUNCHED();
  TGB_CUDA(cudaFreeAsync(base, ctx->stream));
}

// K6 without the random 8 B scatter. new_id_of[order[r]] = r over N ids is a
// scatter of 8 B values into an 8N-byte array: at C3 (888 MB, far beyond L2)
// every store lands in a different sector, and a partial-sector store makes L2
// fill the sector from DRAM first: 4.9 ms for 8.3 GB of DRAM traffic. Replaying
// bucket-partitioned pairs with the whole grid (an 8 MB live window that L2
// holds) still cost 2.1 ms: the fills happen per partial store, not per
// eviction. So every store must write whole sectors: (1) the (id, rank) pairs
// are partitioned by id >> 20 with coalesced staged writes -- bucket b's region
// of the pair array is exactly [b << 20, ...) because every id occurs once, so
// no counting pass -- (2) again by id >> 12 inside each bucket, (3) one CTA
// per 4,096 ids assembles their new_id_of in shared memory and stores it in
// whole sectors. 52 B per id, all of it streamed.
constexpr int kPmShift = 20;
constexpr int kPmIpt = 16;
constexpr int kPmTile = 256 * kPmIpt;
constexpr uint32_t kPmMaxBuckets = 1024;

__global__ void __launch_bounds__(256) perm_part_kernel(const uint32_t* __restrict__ v0,
                                                        const uint32_t* __restrict__ v1,
                                                        const RadixPlan* __restrict__ plan,
                                                        uint64_t n, uint32_t nb,
                                                        uint64_t* __restrict__ order,
                                                        uint2* __restrict__ pairs,
                                                        uint32_t* __restrict__ bcur) {
  const uint32_t* v = plan->final_src ? v1 : v0;
  __shared__ uint2 st[kPmTile];
  __shared__ uint32_t tcnt[kPmMaxBuckets], tst[kPmMaxBuckets], tbase[kPmMaxBuckets];
  __shared__ uint32_t wsum[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint64_t t0 = (uint64_t)blockIdx.x * kPmTile; t0 < n; t0 += (uint64_t)gridDim.x * kPmTile) {
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) tcnt[b] = 0;
    __syncthreads();
    uint32_t id[kPmIpt], rk[kPmIpt];
#pragma unroll
    for (int k = 0; k < kPmIpt; ++k) {
      const uint64_t i = t0 + k * 256 + threadIdx.x;
      id[k] = i < n ? v[i] : 0xffffffffu;
      if (i < n) {
        if (order) order[i] = id[k];
        rk[k] = atomicAdd(&tcnt[id[k] >> kPmShift], 1u);
      }
    }
    __syncthreads();
    {  // exclusive scan of tcnt (nb <= 1024: 4 per thread) + global reservations
      const uint32_t per = (nb + 255) / 256;
      const uint32_t b0 = min(nb, threadIdx.x * per), b1 = min(nb, b0 + per);
      uint32_t run = 0;
      for (uint32_t b = b0; b < b1; ++b) run += tcnt[b];
      uint32_t incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wsum[w] = incl;
      __syncthreads();
      uint32_t x = incl - run;
      for (int k = 0; k < w; ++k) x += wsum[k];
      for (uint32_t b = b0; b < b1; ++b) {
        tst[b] = x;
        x += tcnt[b];
        if (tcnt[b]) tbase[b] = atomicAdd(&bcur[b], tcnt[b]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPmIpt; ++k) {
      const uint64_t i = t0 + k * 256 + threadIdx.x;
      if (i < n) st[tst[id[k] >> kPmShift] + rk[k]] = make_uint2(id[k], static_cast<uint32_t>(i));
    }
    __syncthreads();
    const uint32_t tn = static_cast<uint32_t>(n - t0 < (uint64_t)kPmTile ? n - t0 : kPmTile);
    for (uint32_t j = threadIdx.x; j < tn; j += blockDim.x) {
      const uint2 p = st[j];
      const uint32_t b = p.x >> kPmShift;
      pairs[tbase[b] + (j - tst[b])] = p;  // bcur starts at the bucket's region
    }
    __syncthreads();
  }
}

// (2) each bucket's pairs again, by sub-bucket id >> 12 (4,096 ids, 32 KB of
// new_id_of): a tile of pairs spans at most two buckets, so at most 512
// sub-buckets, staged in shared memory and written out in runs; sub-bucket
// sb's region is again exactly [sb << 12, ...).
constexpr int kPmSubShift = 12;
constexpr int kPmSubThreads = 512, kPmSubIpt = 16;
constexpr int kPmSubTile = kPmSubThreads * kPmSubIpt;  // 8,192 pairs
constexpr uint32_t kPmSubLocal = 2u << (kPmShift - kPmSubShift);  // 512: one per thread
__global__ void __launch_bounds__(kPmSubThreads) perm_sub_kernel(const uint2* __restrict__ in,
                                                                 uint64_t n,
                                                                 uint2* __restrict__ out,
                                                                 uint32_t* __restrict__ scur) {
  extern __shared__ __align__(16) uint2 sst[];  // kPmSubTile
  __shared__ uint32_t tcnt[kPmSubLocal], tst[kPmSubLocal], tbase[kPmSubLocal];
  __shared__ uint32_t wsum[kPmSubThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint64_t t0 = (uint64_t)blockIdx.x * kPmSubTile; t0 < n;
       t0 += (uint64_t)gridDim.x * kPmSubTile) {
    const uint32_t tn = static_cast<uint32_t>(n - t0 < (uint64_t)kPmSubTile ? n - t0 : kPmSubTile);
    // the window of sub-buckets: from the first one of the tile's first bucket
    // (a tile of full 1 Mi-id bucket regions spans at most two buckets; pairs
    // beyond the window -- small regions after tail compaction -- take one
    // slot each)
    const uint32_t sb0 = (__ldg(&in[t0].x) >> kPmShift) << (kPmShift - kPmSubShift);
    tcnt[threadIdx.x] = 0;
    __syncthreads();
    uint2 p[kPmSubIpt];
    uint32_t rk[kPmSubIpt];
#pragma unroll
    for (int k = 0; k < kPmSubIpt; ++k) {
      const uint32_t j = k * kPmSubThreads + threadIdx.x;
      p[k] = make_uint2(0xffffffffu, 0u);
      if (j < tn) {
        const uint2 q = __ldcs(in + t0 + j);
        const uint32_t lb = (q.x >> kPmSubShift) - sb0;
        if (lb < kPmSubLocal) {
          p[k] = q;
          rk[k] = atomicAdd(&tcnt[lb], 1u);
        } else {
          out[atomicAdd(&scur[q.x >> kPmSubShift], 1u)] = q;
        }
      }
    }
    __syncthreads();
    {  // exclusive scan of the 512 counters (one per thread) + global reservations
      const uint32_t c = tcnt[threadIdx.x];
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wsum[w] = incl;
      __syncthreads();
      uint32_t x = incl - c;
      for (int k = 0; k < w; ++k) x += wsum[k];
      tst[threadIdx.x] = x;
      if (c) tbase[threadIdx.x] = atomicAdd(&scur[sb0 + threadIdx.x], c);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPmSubIpt; ++k)
      if (p[k].x != 0xffffffffu) sst[tst[(p[k].x >> kPmSubShift) - sb0] + rk[k]] = p[k];
    __syncthreads();
    const uint32_t ns = tst[kPmSubLocal - 1] + tcnt[kPmSubLocal - 1];  // in-window pairs
    for (uint32_t j = threadIdx.x; j < ns; j += blockDim.x) {
      const uint2 q = sst[j];
      const uint32_t lb = (q.x >> kPmSubShift) - sb0;
      out[tbase[lb] + (j - tst[lb])] = q;  // scur starts at the sub-bucket's region
    }
    __syncthreads();
  }
}

// Region starts of the ranked (non-tail) pairs: bucket b of width 2^shift
// starts at x - T(x), x = min(b << shift, n), T(x) = tail ids below x (the
// tail is sorted); starts[count] = m.
__global__ void perm_bounds_kernel(const uint32_t* __restrict__ tail, uint64_t nt, uint64_t count,
                                   int shift, uint64_t n, uint32_t* __restrict__ starts,
                                   uint32_t* __restrict__ cursor) {
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b <= count;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = (b << shift) < n ? (b << shift) : n;
    uint64_t lo = 0, hi = nt;  // lower_bound(tail, x)
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if (tail[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    starts[b] = static_cast<uint32_t>(x - lo);
    if (cursor && b < count) cursor[b] = static_cast<uint32_t>(x - lo);
  }
}

// order[r] for the compacted tail: the ids in their (ascending) order
__global__ void order_tail_kernel(const uint32_t* __restrict__ tail, uint64_t nt, uint64_t m,
                                  uint64_t* __restrict__ order) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nt;
       t += (uint64_t)gridDim.x * blockDim.x)
    order[m + t] = tail[t];
}

// (3) one CTA per sub-bucket: new_id_of of its 4,096 ids assembled in shared
// memory, then stored as whole sectors
__global__ void __launch_bounds__(256) perm_fill_kernel(const uint2* __restrict__ in, uint64_t n,
                                                        uint64_t m,
                                                        const uint32_t* __restrict__ tail,
                                                        const uint32_t* __restrict__ sbstart,
                                                        uint64_t* __restrict__ new_id_of) {
  __shared__ uint32_t r[1u << kPmSubShift];
  const uint64_t nsb = (n + (1u << kPmSubShift) - 1) >> kPmSubShift;
  for (uint64_t sb = blockIdx.x; sb < nsb; sb += gridDim.x) {
    const uint64_t i0 = sb << kPmSubShift;
    const uint64_t i1 = n - i0 < (1u << kPmSubShift) ? n : i0 + (1u << kPmSubShift);
    const uint32_t cnt = static_cast<uint32_t>(i1 - i0);
    const uint32_t h0 = sbstart[sb], h1 = sbstart[sb + 1];  // this sub-bucket's ranked pairs
    for (uint32_t j = h0 + threadIdx.x; j < h1; j += blockDim.x) {
      const uint2 q = __ldcs(in + j);
      r[q.x & ((1u << kPmSubShift) - 1)] = q.y;
    }
    // its ids among the compacted lowest-score ties (tail[t] has rank m + t):
    // tail ids < x number x - sbstart(x)
    for (uint64_t t = (i0 - h0) + threadIdx.x; t < i1 - h1; t += blockDim.x)
      r[tail[t] & ((1u << kPmSubShift) - 1)] = static_cast<uint32_t>(m + t);
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) new_id_of[i0 + j] = r[j];
    __syncthreads();
  }
}

// Sorts scores -> (order, new_id_of). Either output may be null. Device pointers.
void sort_scores(tg_ctx* ctx, const double* scores_dev, uint64_t n, uint64_t* order_dev,
                 uint64_t* perm_dev) {
  if (n >= 0xffffffffull) domain_error("score_ordering: n must be < 2^32");
  uint64_t* k0 = ctx->scratch_t<uint64_t>(kScratchA, n);
  uint64_t* k1 = ctx->scratch_t<uint64_t>(kScratchB, n);
  uint32_t* v0 = ctx->scratch_t<uint32_t>(kScratchC, n);
  uint32_t* v1 = ctx->scratch_t<uint32_t>(kScratchD, n);
  // small slot layout: [bad u64][plan][hist 8x256 u32]
  char* small = static_cast<char*>(
      ctx->scratch(kSmall, 64 + sizeof(RadixPlan) + 8 * 256 * 4 + 256 * 4));
  auto* bad = reinterpret_cast<unsigned long long*>(small);
  auto* plan = reinterpret_cast<RadixPlan*>(small + 64);
  auto* hist = reinterpret_cast<uint32_t*>(small + 64 + sizeof(RadixPlan));
  TGB_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
  TGB_CUDA(cudaMemsetAsync(hist, 0, 8 * 256 * 4, ctx->stream));
  auto* kmin = reinterpret_cast<unsigned long long*>(small) + 1;
  auto* kmax = reinterpret_cast<unsigned long long*>(small) + 2;
  TGB_CUDA(cudaMemsetAsync(kmin, 0xff, 8, ctx->stream));
  TGB_CUDA(cudaMemsetAsync(kmax, 0, 8, ctx->stream));
  key_range_kernel<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(scores_dev, n, kmin,
                                                                                kmax);
  TGB_LAUNCHED();
  // the lowest-score ties: how many keys stay in the sort (m)
  const uint64_t nt = (n + kKpTile - 1) / kKpTile;
  uint64_t* toff = ctx->scratch_t<uint64_t>(kScratchF, nt + 1);
  TGB_CUDA(cudaMemsetAsync(toff + nt, 0, 8, ctx->stream));
  key_tile_count_kernel<<<grid_for(nt, 1, ctx->num_sms * 8), 256, 0, ctx->stream>>>(scores_dev, n,
                                                                                    kmax, toff);
  TGB_LAUNCHED();
  exclusive_scan_u64(ctx, toff, nt + 1);
  uint64_t m = n;
  TGB_CUDA(cudaMemcpyAsync(&m, toff + nt, 8, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  const bool compact = (n - m) * 8 >= n;  // worth it when >= 1/8 of the keys tie at the bottom
  if (compact) {
    key_prep_compact_kernel<<<grid_for(nt, 1, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
        scores_dev, n, kmin, kmax, toff, k0, v0, v1, hist, bad);
  } else {
    m = n;
    key_prep_kernel<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(scores_dev, n, kmin,
                                                                                 k0, v0, hist, bad);
  }
  TGB_LAUNCHED();
  plan_kernel<<<1, 256, 0, ctx->stream>>>(hist, m, plan, 4);  // pass 4 narrows to u32 keys
  TGB_LAUNCHED();
  if (m) radix_passes(ctx, k0, v0, k1, v1, m, 8, plan, hist, 8, 4);
  const uint64_t nb = (n + (1ull << kPmShift) - 1) >> kPmShift;
  if (perm_dev && nb <= kPmMaxBuckets) {
    // ranks [0, m) come from the sort; the compacted lowest-score ties (sorted
    // ids, ranks m..n-1) sit in v0[m, n) (and v1[m, n)): they skip the
    // partition and are merged in by perm_fill
    const uint32_t* tail = v0 + m;
    const uint64_t nt = n - m;
    const uint64_t nsb = (n + (1u << kPmSubShift) - 1) >> kPmSubShift;
    uint32_t* bstart = ctx->scratch_t<uint32_t>(kScratchE, 2 * (kPmMaxBuckets + 1) + 2 * (nsb + 1));
    uint32_t* bcur = bstart + kPmMaxBuckets + 1;
    uint32_t* sbstart = bcur + kPmMaxBuckets + 1;
    uint32_t* scur = sbstart + nsb + 1;
    perm_bounds_kernel<<<grid_for(nb + 1, 256), 256, 0, ctx->stream>>>(tail, nt, nb, kPmShift, n,
                                                                        bstart, bcur);
    TGB_LAUNCHED();
    perm_bounds_kernel<<<grid_for(nsb + 1, 256), 256, 0, ctx->stream>>>(tail, nt, nsb, kPmSubShift,
                                                                         n, sbstart, scur);
    TGB_LAUNCHED();
    // both key buffers are free after the sort; pairs (8m bytes) go in k0
    uint2* pairs = reinterpret_cast<uint2*>(k0);
    int pocc = 1;
    TGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pocc, perm_part_kernel, 256, 0));
    if (m)
      perm_part_kernel<<<grid_for(m, kPmTile, ctx->num_sms * std::max(pocc, 1)), 256, 0,
                         ctx->stream>>>(v0, v1, plan, m, static_cast<uint32_t>(nb), order_dev,
                                        pairs, bcur);
    TGB_LAUNCHED();
    if (order_dev && nt) {
      order_tail_kernel<<<grid_for(nt, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(tail, nt, m,
                                                                                      order_dev);
      TGB_LAUNCHED();
    }
    uint2* pairs2 = reinterpret_cast<uint2*>(k1);
    static bool sattr[TG_MAX_DEVICES] = {};
    if (!sattr[ctx->device % TG_MAX_DEVICES]) {
      TGB_CUDA(cudaFuncSetAttribute(perm_sub_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    8 * kPmSubTile));
      sattr[ctx->device % TG_MAX_DEVICES] = true;
    }
    int occ = 1;
    TGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, perm_sub_kernel, kPmSubThreads,
                                                           8 * kPmSubTile));
    if (m)
      perm_sub_kernel<<<grid_for(m, kPmSubTile, ctx->num_sms * std::max(occ, 1)), kPmSubThreads,
                        8 * kPmSubTile, ctx->stream>>>(pairs, m, pairs2, scur);
    TGB_LAUNCHED();
    perm_fill_kernel<<<grid_for(nsb, 1, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        pairs2, n, m, tail, sbstart, perm_dev);
    TGB_LAUNCHED();
  } else {
    perm_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(v0, v1, plan, n, order_dev, perm_dev);
    TGB_LAUNCHED();
  }
  unsigned long long hb = 0;
  TGB_CUDA(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  if (hb != ~0ull)
    domain_error("score " + std::to_string(hb) + " is not finite and >= 0");  // scoring.cpp:107
}

// ------------------------------------------------------------- transpose
// csr_graph.cpp:67-80: row v of the transpose lists the sources u of the
// edges (u, v), ascending ("walking sources in ascending order leaves every
// transposed row sorted"). On the device: a STABLE radix sort of the edges by
// target, presented in CSR (= ascending source) order, carrying the source
// as the value; the transposed offsets are the key boundaries.
__global__ void __launch_bounds__(256) edge_keys_kernel(const uint64_t* __restrict__ off,
                                                        const uint64_t* __restrict__ tgt,
                                                        uint64_t n, uint32_t* __restrict__ keys,
                                                        uint32_t* __restrict__ vals,
                                                        uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[4][256];
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  // one warp per source row: coalesced over the row's edges
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t u = warp; u < n; u += nw) {
    for (uint64_t i = off[u] + lane; i < off[u + 1]; i += 32) {
      const uint32_t k = static_cast<uint32_t>(tgt[i]);  // < n < 2^32 (range-checked first)
      keys[i] = k;
      vals[i] = static_cast<uint32_t>(u);
#pragma unroll
      for (int p = 0; p < 4; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xff], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

__global__ void key_range_check_kernel(const uint64_t* __restrict__ tgt, uint64_t e, uint64_t n,
                                       uint32_t* __restrict__ hist, unsigned long long* bad) {
  // targets < n < 2^32, so digits 4..7 are 0: one full bin each; range check
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (tgt[i] >= n) atomicMin(bad, (unsigned long long)i);
  if (blockIdx.x == 0)
    for (int p = 4 + threadIdx.x; p < 8; p += blockDim.x) hist[p * 256] = static_cast<uint32_t>(e);
}

// t_off[v] = first sorted position with key >= v; t_tgt[i] = source (u64)
__global__ void transpose_out_kernel(const uint32_t* __restrict__ k0, const uint32_t* __restrict__ k1,
                                     const uint32_t* __restrict__ v0, const uint32_t* __restrict__ v1,
                                     const RadixPlan* __restrict__ plan, uint64_t n, uint64_t e,
                                     uint64_t* __restrict__ t_off, uint64_t* __restrict__ t_tgt) {
  const uint32_t* k = plan->final_src ? k1 : k0;
  const uint32_t* v = plan->final_src ? v1 : v0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= e;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t hi = i < e ? k[i] : n;          // rows (prev, hi] start at i
    const uint64_t lo = i ? k[i - 1] + 1 : 0;
    for (uint64_t r = lo; r <= hi && r <= n; ++r) t_off[r] = i;
    if (i < e) t_tgt[i] = v[i];
  }
}

void transpose_device(tg_ctx* ctx, const uint64_t* off, const uint64_t* tgt, uint64_t n, uint64_t e,
                      uint64_t* t_off, uint64_t* t_tgt) {
  if (n >= 0xffffffffull || e >= 0xffffffffull)
    domain_error("transpose: n and e must be < 2^32 on the device");
  if (e == 0) {
    TGB_CUDA(cudaMemsetAsync(t_off, 0, 8 * (n + 1), ctx->stream));
    return;
  }
  const size_t bytes = 4 * 4 * e + 64 + 64 + sizeof(RadixPlan) + 8 * 256 * 4 + 256;
  char* base = nullptr;
  TGB_CUDA(tgb::dev_malloc_async(reinterpret_cast<void**>(&base), bytes, ctx->stream));
  auto align = [](char* p) { return reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15)); };
  char* p = base;
  uint32_t* k0 = reinterpret_cast<uint32_t*>(p); p = align(p + 4 * e);  // u32 keys (targets)
  uint32_t* k1 = reinterpret_cast<uint32_t*>(p); p = align(p + 4 * e);
  uint32_t* v0 = reinterpret_cast<uint32_t*>(p); p = align(p + 4 * e);
  uint32_t* v1 = reinterpret_cast<uint32_t*>(p); p = align(p + 4 * e);
  auto* bad = reinterpret_cast<unsigned long long*>(p); p = align(p + 64);
  auto* plan = reinterpret_cast<RadixPlan*>(p); p = align(p + sizeof(RadixPlan));
  uint32_t* hist = reinterpret_cast<uint32_t*>(p);
  TGB_CUDA(cudaMemsetAsync(hist, 0, 8 * 256 * 4, ctx->stream));
  TGB_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
  key_range_check_kernel<<<grid_for(e, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(tgt, e, n,
                                                                                      hist, bad);
  TGB_LAUNCHED();
  unsigned long long hb;
  TGB_CUDA(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  if (hb != ~0ull) {
    cudaFreeAsync(base, ctx->stream);
    format_error("csr: target out of range at edge " + std::to_string(hb));
  }
  edge_keys_kernel<<<grid_for(n * 32, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(off, tgt, n, k0,
                                                                                     v0, hist);
  TGB_LAUNCHED();
  plan_kernel<<<1, 256, 0, ctx->stream>>>(hist, e, plan);
  TGB_LAUNCHED();
  radix_passes(ctx, k0, v0, k1, v1, e, 4, plan, hist, 4, -1);  // digits 4..7 are constant
  transpose_out_kernel<<<grid_for(e + 1, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
      k0, k1, v0, v1, plan, n, e, t_off, t_tgt);
  TGB_LAUNCHED();
  TGB_CUDA(cudaFreeAsync(base, ctx->stream));
}

}  // namespace tgb

using namespace tgb;

extern "C" {

int tg_transpose(tg_ctx* ctx, const uint64_t* offsets, const uint64_t* targets, uint64_t n,
                 uint64_t e, uint64_t* out_offsets, uint64_t* out_targets) {
  return guard([&] {  // csr_graph.cpp:67-80
    DeviceGuard dg(ctx->device);
    const uint64_t* off = dev_in(ctx, offsets, n + 1, kStageIn0);
    const uint64_t* tgt = dev_in(ctx, targets, e, kStageIn1);
    DevOut<uint64_t> oo(ctx, out_offsets, n + 1, kStageOut0);
    DevOut<uint64_t> ot(ctx, out_targets, e, kStageOut1);
    transpose_device(ctx, off, tgt, n, e, oo.dev(), ot.dev());
    if (oo.host)
      TGB_CUDA(cudaMemcpyAsync(out_offsets, oo.dev(), 8 * (n + 1), cudaMemcpyDeviceToHost,
                               ctx->stream));
    ot.finish();
  });
}

int tg_score_ordering(tg_ctx* ctx, const double* scores, uint64_t n, uint64_t* out_order) {
  return guard([&] {
    if (n == 0) return;
    DeviceGuard dg(ctx->device);
    const double* s = dev_in(ctx, scores, n, kStageIn0);
    DevOut<uint64_t> o(ctx, out_order, n, kStageOut0);
    sort_scores(ctx, s, n, o.dev(), nullptr);
    o.finish();
  });
}

int tg_permutation_from_scores(tg_ctx* ctx, const double* scores, uint64_t n,
                               uint64_t* out_new_id_of, uint64_t* out_order) {
  return guard([&] {
    if (n == 0) return;
    DeviceGuard dg(ctx->device);
    const double* s = dev_in(ctx, scores, n, kStageIn0);
    DevOut<uint64_t> p(ctx, out_new_id_of, n, kStageOut0);
    uint64_t* od = nullptr;
    bool order_host = false;
    if (out_order) {
      order_host = !is_device_ptr(out_order);
      od = order_host ? ctx->scratch_t<uint64_t>(kStageOut1, n) : out_order;
    }
    sort_scores(ctx, s, n, od, p.dev());
    if (order_host)
      TGB_CUDA(cudaMemcpyAsync(out_order, od, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    p.finish();
  });
}

}  // extern "C"
