// K1, binned: in_degrees (proj/src/csr_graph.cpp:89-93 — deg[t]++ for every
// stored target t) as a partition followed by shared-memory histograms.
//
// Why not one atomic per edge: an L2 atomic costs a slice cycle whatever the
// counter array's size, and on this part the L2 retires ~95 G RED/s (K1 ran
// at 97 G/s at C3, 444 MB of counters, and 93 G/s at C2, 9.8 MB of counters:
// the same rate), 15.8 ms for papers100M's 1.53 G targets. Shared-memory
// atomics retire an order of magnitude faster, but 111 M counters do not fit
// one SM. So:
//   1. count   per-chunk counts of the BUCKET b = t >> bs (2^bs ids per
//              bucket, bs in [15, 18], <= ~2,048 buckets), one CTA per chunk
//              of the target array, shared-memory histogram;
//   2. scan    bucket-major exclusive scan of the (bucket, chunk) counts: the
//              chunk's write cursor inside each bucket's segment of a
//              temporary copy of the targets;
//   3. scatter every CTA re-reads its chunk tile by tile, orders each tile
//              by bucket in shared memory and writes it out in bucket runs
//              (coalesced; the <= 8,192 open run ends stay in L2, so DRAM
//              sees full sectors);
//   4. count   2^(bs-15) CTAs per (bucket, <= 256k-target piece), persistent:
//              each a 32,768-bin shared-memory histogram of its id range of
//              the piece (the CTAs of one piece read it from L2), flushed with
//              plain coalesced stores when the bucket is one piece, with
//              atomics when a hub bucket is split over several.
// With thousands of buckets (C3: 3,388) a tile's runs are ~2 targets long,
// partial sectors that L2 fills from DRAM first (C3: 9.9 GB read + 10.8 GB
// written by the scatter for 6.1 GB of targets); a two-level partition
// (<= 128 x <= 32 buckets, per-tile cursor reservations) removed the fills
// but its two passes took 7.7 ms each (profiles/r02n), so one level stays.
// Traffic: 4 B x E read (1), 8 B x E (3), 4 B x E (4), 4 B x N written —
// 16 B per edge against the 4 B per edge of the one-pass form, in exchange
// for shared-memory instead of L2 atomics. The counts are exact integers
// whatever the order (no summation-order question).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"

namespace tgb {

#ifndef TG_K1_SHIFT  // ids per bucket = 2^shift (compile-time experiment knob)
#define TG_K1_SHIFT 15
#endif
#ifndef TG_K1_PIECE_LOG2  // elements per histogram work item = 2^this
#define TG_K1_PIECE_LOG2 18
#endif
constexpr int kK1Shift = TG_K1_SHIFT;
constexpr uint32_t kK1Bins = 1u << kK1Shift;    // ids per bucket (128 KB of counters)
constexpr uint32_t kK1MaxBuckets = 8192;        // n <= 2^28
#ifndef TG_K1_THREADS  // threads of the count / scatter CTAs (tile = 16 per thread)
#define TG_K1_THREADS 512
#endif
constexpr int kK1Threads = TG_K1_THREADS, kK1Ipt = 16;
constexpr uint32_t kK1Tile = kK1Threads * kK1Ipt;  // 8,192 targets per scatter tile
constexpr uint32_t kK1Piece = 1u << TG_K1_PIECE_LOG2;  // elements per histogram work item
constexpr int kK1HistThreads = 1024;

// (1) per-chunk bucket counts, bucket-major: cnt[b * G + c]
__global__ void __launch_bounds__(kK1Threads) k1_count_kernel(const uint32_t* __restrict__ tgt,
                                                              uint64_t e, uint64_t chunk,
                                                              uint32_t nb, uint32_t G, int bs,
                                                              uint64_t* __restrict__ cnt) {
  extern __shared__ uint32_t h[];  // nb
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint64_t c0 = blockIdx.x * chunk, c1 = min(e, c0 + chunk);  // c0 % 4 == 0
  const uint64_t v1 = c0 + ((c1 - c0) & ~3ull);
  // four 16 B loads in flight per thread, then their 16 shared-memory atomics
  const uint64_t step = 4 * (uint64_t)blockDim.x;
  uint64_t i = c0 + 4 * (uint64_t)threadIdx.x;
  for (; i + 3 * step < v1; i += 4 * step) {
    uint4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = __ldcs(reinterpret_cast<const uint4*>(tgt + i + q * step));
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      atomicAdd(&h[v[q].x >> bs], 1u);
      atomicAdd(&h[v[q].y >> bs], 1u);
      atomicAdd(&h[v[q].z >> bs], 1u);
      atomicAdd(&h[v[q].w >> bs], 1u);
    }
  }
  for (; i < v1; i += step) {
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(tgt + i));
    atomicAdd(&h[v.x >> bs], 1u);
    atomicAdd(&h[v.y >> bs], 1u);
    atomicAdd(&h[v.z >> bs], 1u);
    atomicAdd(&h[v.w >> bs], 1u);
  }
  for (uint64_t j = v1 + threadIdx.x; j < c1; j += blockDim.x) atomicAdd(&h[tgt[j] >> bs], 1u);
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) cnt[(uint64_t)b * G + blockIdx.x] = h[b];
}

// Block-wide exclusive scan of the nb counters in `c` into `s` (512 threads).
__device__ __forceinline__ void k1_block_scan(const uint32_t* c, uint32_t* s, uint32_t nb,
                                              uint32_t* wsum) {
  const uint32_t per = (nb + kK1Threads - 1) / kK1Threads;
  const uint32_t b0 = min(nb, threadIdx.x * per), b1 = min(nb, b0 + per);
  uint32_t run = 0;
  for (uint32_t b = b0; b < b1; ++b) run += c[b];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t before = 0;
  for (int k = 0; k < w; ++k) before += wsum[k];
  uint32_t x = before + incl - run;
  for (uint32_t b = b0; b < b1; ++b) {
    s[b] = x;
    x += c[b];
  }
}

// (3) scatter: chunk blockIdx.x, tile by tile, bucket-ordered in shared memory.
// (Warp-aggregated tile ranks -- one shared atomic per bucket per warp -- were
// slower at C2: 475 vs 403 us, __match_any_sync plus spills; profiles/r02k1d.)
__global__ void __launch_bounds__(kK1Threads, 1024 / kK1Threads) k1_scatter_kernel(const uint32_t* __restrict__ tgt,
                                                                uint64_t e, uint64_t chunk,
                                                                uint32_t nb, uint32_t G, int bs,
                                                                const uint64_t* __restrict__ cnt,
                                                                uint32_t* __restrict__ out) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* st = sm;                 // kK1Tile staged targets
  uint32_t* tcnt = st + kK1Tile;     // nb: this tile's count per bucket
  uint32_t* tst = tcnt + nb;         // nb: this tile's bucket starts in st
  uint32_t* cur = tst + nb;          // nb: this chunk's write cursor per bucket
  __shared__ uint32_t wsum[kK1Threads / 32];
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x)
    cur[b] = static_cast<uint32_t>(cnt[(uint64_t)b * G + blockIdx.x]);
  const uint64_t c0 = blockIdx.x * chunk, c1 = min(e, c0 + chunk);
  for (uint64_t t0 = c0; t0 < c1; t0 += kK1Tile) {
    const uint32_t tn = static_cast<uint32_t>((c1 - t0 < kK1Tile ? c1 - t0 : (uint64_t)kK1Tile));
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) tcnt[b] = 0;
    __syncthreads();
    uint32_t v[kK1Ipt], r[kK1Ipt];
    if (tn == kK1Tile) {
#pragma unroll
      for (int k = 0; k < kK1Ipt / 4; ++k) {
        const uint4 q = __ldcs(reinterpret_cast<const uint4*>(tgt + t0) + k * kK1Threads + threadIdx.x);
        v[4 * k] = q.x;
        v[4 * k + 1] = q.y;
        v[4 * k + 2] = q.z;
        v[4 * k + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kK1Ipt; ++k) {
        const uint32_t j = (k >> 2) * (4 * kK1Threads) + 4 * threadIdx.x + (k & 3);
        v[k] = j < tn ? tgt[t0 + j] : 0xffffffffu;
      }
    }
#pragma unroll
    for (int k = 0; k < kK1Ipt; ++k)  // ids < 2^28: 0xffffffff only marks a partial tile's end
      if (v[k] != 0xffffffffu) r[k] = atomicAdd(&tcnt[v[k] >> bs], 1u);
    __syncthreads();
    k1_block_scan(tcnt, tst, nb, wsum);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kK1Ipt; ++k)
      if (v[k] != 0xffffffffu) st[tst[v[k] >> bs] + r[k]] = v[k];
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < tn; j += blockDim.x) {
      const uint32_t t = st[j], b = t >> bs;
      out[cur[b] + (j - tst[b])] = t;
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) cur[b] += tcnt[b];
  }
}

struct K1Item {
  uint32_t bucket, begin, end, split;
};

// Work items: bucket b's segment [cnt[b*G], cnt[(b+1)*G]) cut into pieces of
// at most kK1Piece elements. One CTA of 1024 threads.
__global__ void __launch_bounds__(1024) k1_items_kernel(const uint64_t* __restrict__ cnt,
                                                        uint32_t nb, uint32_t G,
                                                        K1Item* __restrict__ items,
                                                        uint32_t* __restrict__ nitems) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t base_s;
  if (threadIdx.x == 0) base_s = 0;
  __syncthreads();
  for (uint32_t b0 = 0; b0 < nb; b0 += blockDim.x) {
    const uint32_t b = b0 + threadIdx.x;
    uint64_t beg = 0, end = 0;
    uint32_t np = 0;
    if (b < nb) {
      beg = cnt[(uint64_t)b * G];
      end = cnt[(uint64_t)(b + 1) * G];
      np = end > beg ? static_cast<uint32_t>((end - beg + kK1Piece - 1) / kK1Piece) : 1u;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = np;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    uint32_t before = base_s;
    for (int k = 0; k < w; ++k) before += wsum[k];
    const uint32_t first = before + incl - np;
    for (uint32_t p = 0; p < np; ++p) {
      const uint64_t pb = beg + (uint64_t)p * kK1Piece;
      items[first + p] = K1Item{b, static_cast<uint32_t>(pb),
                                static_cast<uint32_t>(end < pb + kK1Piece ? end : pb + kK1Piece),
                                np > 1 ? 1u : 0u};
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) base_s = first + np;
    __syncthreads();
  }
  if (threadIdx.x == 0) *nitems = base_s;
}

// (4) persistent: claim a piece, histogram it into 32,768 shared counters, flush.
// A bucket of 2^bs ids (bs >= 15) is counted by 2^(bs-15) CTAs per piece,
// each over its own 32,768-id range: every CTA reads the whole piece (the
// others' reads of it hit L2) and skips the targets outside its range.
__global__ void __launch_bounds__(kK1HistThreads) k1_hist_kernel(const uint32_t* __restrict__ part,
                                                                 const K1Item* __restrict__ items,
                                                                 const uint32_t* __restrict__ nitems,
                                                                 uint32_t* __restrict__ ctr,
                                                                 uint64_t n, int bs,
                                                                 uint32_t* __restrict__ deg) {
  extern __shared__ __align__(16) uint32_t hb[];  // kK1Bins
  __shared__ uint32_t item_s;
  const int qs = bs - kK1Shift;  // log2 of the CTAs per piece
  const uint32_t qm = (1u << qs) - 1;
  const uint32_t ni = *nitems << qs;
  for (;;) {
    if (threadIdx.x == 0) item_s = atomicAdd(ctr, 1u);
    for (uint32_t i = threadIdx.x; i < kK1Bins; i += blockDim.x) hb[i] = 0;
    __syncthreads();
    const uint32_t it = item_s;
    if (it >= ni) break;
    const K1Item m = items[it >> qs];
    const uint32_t qr = it & qm;  // this CTA's 32,768-id range of the bucket
    // head to a 16 B boundary, uint4 body, tail
    const uint32_t hb_end = min(m.end, (m.begin + 3u) & ~3u);
    for (uint32_t i = m.begin + threadIdx.x; i < hb_end; i += blockDim.x)
      { const uint32_t t = part[i]; if (((t >> kK1Shift) & qm) == qr) atomicAdd(&hb[t & (kK1Bins - 1)], 1u); }
    const uint32_t vb = hb_end, ve = vb + ((m.end - vb) & ~3u);
    const uint32_t step = 4 * blockDim.x;
    uint32_t i = vb + 4 * threadIdx.x;
    for (; i + 3 * step < ve; i += 4 * step) {  // four 16 B loads in flight per thread
      uint4 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = __ldcs(reinterpret_cast<const uint4*>(part + i + q * step));
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (((v[q].x >> kK1Shift) & qm) == qr) atomicAdd(&hb[v[q].x & (kK1Bins - 1)], 1u);
        if (((v[q].y >> kK1Shift) & qm) == qr) atomicAdd(&hb[v[q].y & (kK1Bins - 1)], 1u);
        if (((v[q].z >> kK1Shift) & qm) == qr) atomicAdd(&hb[v[q].z & (kK1Bins - 1)], 1u);
        if (((v[q].w >> kK1Shift) & qm) == qr) atomicAdd(&hb[v[q].w & (kK1Bins - 1)], 1u);
      }
    }
    for (; i < ve; i += step) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(part + i));
      if (((v.x >> kK1Shift) & qm) == qr) atomicAdd(&hb[v.x & (kK1Bins - 1)], 1u);
      if (((v.y >> kK1Shift) & qm) == qr) atomicAdd(&hb[v.y & (kK1Bins - 1)], 1u);
      if (((v.z >> kK1Shift) & qm) == qr) atomicAdd(&hb[v.z & (kK1Bins - 1)], 1u);
      if (((v.w >> kK1Shift) & qm) == qr) atomicAdd(&hb[v.w & (kK1Bins - 1)], 1u);
    }
    for (uint32_t i = ve + threadIdx.x; i < m.end; i += blockDim.x)
      { const uint32_t t = part[i]; if (((t >> kK1Shift) & qm) == qr) atomicAdd(&hb[t & (kK1Bins - 1)], 1u); }
    __syncthreads();
    const uint64_t id0 = ((uint64_t)m.bucket << bs) + ((uint64_t)qr << kK1Shift);
    const uint32_t nbin =
        id0 >= n ? 0u : static_cast<uint32_t>((n - id0 < kK1Bins ? n - id0 : (uint64_t)kK1Bins));
    if (m.split) {
      for (uint32_t i = threadIdx.x; i < nbin; i += blockDim.x)
        if (hb[i]) atomicAdd(&deg[id0 + i], hb[i]);
    } else {
      for (uint32_t i = threadIdx.x; i < nbin; i += blockDim.x) deg[id0 + i] = hb[i];
    }
    __syncthreads();
  }
}

// deg must be zeroed by the caller (split buckets accumulate into it).
// Returns false when the binned form does not apply (tiny graphs, n > 2^28,
// or no room for the 4 B x E temporary) so the caller runs the one-pass form.
bool compute_indeg_binned(tg_ctx* ctx, const uint32_t* tgt, uint64_t e, uint64_t n,
                          uint32_t* deg) {
  if (const char* k = std::getenv("TIERGRAPH_K1")) {
    if (std::strcmp(k, "atomic") == 0) return false;
  } else if (e < (1u << 20) || n <= 12288) {
    return false;  // launch-bound sizes: the one-pass kernel is cheaper
  }
  // bucket width 2^bs: at most ~2,048 buckets (longer scatter runs, fewer
  // partial sectors), at least the 32,768 ids of one shared-memory histogram
  // and at most 8 of them (C3: 2^16, 1,694 buckets: 11.8 ms against 14.4 at
  // 2^15, 12.6 at 2^17, 14.7 at 2^18; profiles/r02k1f). TIERGRAPH_K1_BS
  // overrides (experiments).
  int bs = kK1Shift;
  while (bs < kK1Shift + 3 && ((n + (1ull << bs) - 1) >> bs) > 2048) ++bs;
  if (const char* b = std::getenv("TIERGRAPH_K1_BS")) bs = std::max(kK1Shift, std::min(kK1Shift + 3, std::atoi(b)));
  const uint64_t nb64 = (n + (1ull << bs) - 1) >> bs;
  if (nb64 > kK1MaxBuckets || e == 0 || e >= 0xffffffffull ||
      (reinterpret_cast<uintptr_t>(tgt) & 15))
    return false;
  const uint32_t nb = static_cast<uint32_t>(nb64);
  static bool attr[TG_MAX_DEVICES] = {};

  const size_t scat_smem = 4 * (kK1Tile + 3 * (size_t)nb);
  if (!attr[ctx->device % TG_MAX_DEVICES]) {
    TGB_CUDA(cudaFuncSetAttribute(k1_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  4 * (kK1Tile + 3 * kK1MaxBuckets)));
    TGB_CUDA(cudaFuncSetAttribute(k1_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  4 * kK1Bins));
    TGB_CUDA(cudaFuncSetAttribute(k1_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  4 * kK1MaxBuckets));
    attr[ctx->device % TG_MAX_DEVICES] = true;
  }
  int occ = 0;
  TGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k1_scatter_kernel, kK1Threads,
                                                         scat_smem));
  occ = std::max(occ, 1);
  // one wave of chunks; each chunk a whole number of tiles
  uint64_t chunk = (e + (uint64_t)ctx->num_sms * occ - 1) / ((uint64_t)ctx->num_sms * occ);
  chunk = (chunk + kK1Tile - 1) / kK1Tile * kK1Tile;
  const uint32_t G = static_cast<uint32_t>((e + chunk - 1) / chunk);
  const uint64_t ncnt = (uint64_t)nb * G + 1;
  const uint64_t max_items = nb + e / kK1Piece + 1;
  const size_t bytes = 4 * e + 16 + 8 * ncnt + 16 + sizeof(K1Item) * max_items + 64;
  char* base = nullptr;
  if (tgb::dev_malloc_async(reinterpret_cast<void**>(&base), bytes, ctx->stream) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  auto align = [](char* p) {
    return reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  };
  char* p = base;
  auto* part = reinterpret_cast<uint32_t*>(p);  p = align(p + 4 * e);
  auto* cnt = reinterpret_cast<uint64_t*>(p);   p = align(p + 8 * ncnt);
  auto* items = reinterpret_cast<K1Item*>(p);   p = align(p + sizeof(K1Item) * max_items);
  auto* small = reinterpret_cast<uint32_t*>(p);  // [nitems, claim counter]
  TGB_CUDA(cudaMemsetAsync(small, 0, 8, ctx->stream));
  TGB_CUDA(cudaMemsetAsync(cnt + ncnt - 1, 0, 8, ctx->stream));
  k1_count_kernel<<<G, kK1Threads, 4 * nb, ctx->stream>>>(tgt, e, chunk, nb, G, bs, cnt);
  TGB_LAUNCHED();
  exclusive_scan_u64(ctx, cnt, ncnt);
  k1_scatter_kernel<<<G, kK1Threads, scat_smem, ctx->stream>>>(tgt, e, chunk, nb, G, bs, cnt, part);
  TGB_LAUNCHED();
  k1_items_kernel<<<1, 1024, 0, ctx->stream>>>(cnt, nb, G, items, small);
  TGB_LAUNCHED();
  // persistent: as many 1024-thread CTAs per SM as shared memory allows (2 at most)
  k1_hist_kernel<<<ctx->num_sms * (kK1Bins <= 16384 ? 2 : 1), kK1HistThreads, 4 * kK1Bins,
                   ctx->stream>>>(part, items, small, small + 1, n, bs, deg);
  TGB_LAUNCHED();
  TGB_CUDA(cudaFreeAsync(base, ctx->stream));
  return true;
}

}  // namespace tgb
