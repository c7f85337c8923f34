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
#include <cstdlib>
#include <string>
#include <vector>

#include "internal.cuh"
#include "pagerank_internal.cuh"
#include "store_internal.cuh"

namespace tgb {

// K3 row classes (rows sorted by length at graph upload):
//   A  len > kLenA          one CTA per row, exact parallel evaluation of the chain
//   B  kLenB < len <= kLenA one warp per row: lanes stage 256-edge windows, lane 0 chains
//   C  len <= kLenB         one thread per row (a warp's rows have near-equal lengths)
// The class-A bound is adaptive: max(kLenA, min(E >> 14, kLenAMax)). A class-B
// row's serial chain costs ~8 cycles per edge, so rows up to E / 2^14 edges
// finish well inside a step that streams E edges (C3: rows up to 65,536 edges,
// chain <= 0.3 ms of an 11 ms step); only rows longer than that need class
// A's exact parallel evaluation, whose per-edge instruction count (~9 per
// lane) made the 20.8k C3 rows of 4-65k edges cost 4.2 ms on their own
// (profiles/r02h, r02i: C3 step 13.9 -> 11.0 ms; C2 keeps 4096).
constexpr uint32_t kLenA = 4096;
constexpr uint32_t kLenAMax = 65536;
constexpr uint32_t kLenB = 512;
constexpr uint32_t kLenBTwin = 256;
// K3's L2 persisting window over the first labels of the twin (see L2Persist)
constexpr long kPersistDefaultMB = 48;
// class-A CTAs: 256 threads x 8 addends (2,048 per tile); 512 x 8 for the
// rows longer than kHubLong and a quarter of the longest row (half the tiles
// on the critical path; 1024 x 4 was measured no faster for the 77k-edge C2
// row: 158 vs 151 us)
constexpr uint32_t kHubLong = 16384;
constexpr int kPrWin = 256;         // edges staged per warp per window (class B)
#ifndef TG_PR_WARPS
#define TG_PR_WARPS 8
#endif
constexpr int kPrWarps = TG_PR_WARPS;  // warps per CTA (classes B, C)

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

// Class boundaries of a length-sorted schedule (one thread; binary search).
__global__ void class_bounds_kernel(const uint32_t* __restrict__ off,
                                    const uint32_t* __restrict__ order, uint64_t m,
                                    uint32_t len_a, uint32_t len_b, uint32_t* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  // 512-thread class-A CTAs only for the few rows that set the critical
  // path: longer than kHubLong AND than a quarter of the longest row
  const uint32_t longest = m ? off[order[0] + 1] - off[order[0]] : 0u;
  const uint32_t lim[3] = {len_a, len_b, max(max(kHubLong, len_a), longest / 4)};
  for (int c = 0; c < 3; ++c) {  // first index whose length is <= lim[c]
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      const uint32_t r = order[mid];
      if (off[r + 1] - off[r] > lim[c]) lo = mid + 1;
      else hi = mid;
    }
    out[c] = static_cast<uint32_t>(lo);
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
                                  const uint32_t* __restrict__ relabel,
                                  uint32_t* __restrict__ mult, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ntid;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t id = tid[i];
    if (id >= n) atomicMin(bad, (unsigned long long)i);
    else atomicAdd(&mult[relabel ? relabel[id] : id], 1u);
  }
}

// ------------------------------------------------------- K3 relabel twin
__global__ void twin_labels_kernel(const uint32_t* __restrict__ old_of,
                                   const uint32_t* __restrict__ indeg, uint64_t n,
                                   uint32_t* __restrict__ new_of, uint32_t* __restrict__ indeg_lab) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = old_of[v];
    new_of[u] = static_cast<uint32_t>(v);
    indeg_lab[v] = indeg[u];
  }
}

// Hybrid twin order key (descending sort, ties by id): class A rows (more
// than kLenA edges) by length above everything else; every other row by its
// length bucket (0: empty, 1 + ceil(log2 len)) and then its in-degree.
__global__ void hybrid_key_kernel(const uint32_t* __restrict__ off,
                                  const uint32_t* __restrict__ indeg, uint64_t n,
                                  uint32_t* __restrict__ key) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t len = off[v + 1] - off[v];
    constexpr uint32_t kLow = (1u << 26) - 1;
    uint32_t k;
    if (len > kLenA) {
      k = (63u << 26) | min(len, kLow);
    } else {
      const uint32_t b = len ? 1u + (32u - __clz(len - 1u)) : 0u;  // <= 13
      k = (b << 26) | min(indeg[v], kLow);
    }
    key[v] = k;
  }
}

// storage row k of the twin = original row sigma[k] (K3's schedule order)
__global__ void twin_rows_meta_kernel(const uint32_t* __restrict__ off,
                                      const uint32_t* __restrict__ sigma,
                                      const uint32_t* __restrict__ new_of,
                                      const uint32_t* __restrict__ indeg, uint64_t n,
                                      uint64_t* __restrict__ lens, uint32_t* __restrict__ row_label,
                                      uint32_t* __restrict__ row_orig,
                                      uint32_t* __restrict__ deg_rows) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = sigma[k];
    lens[k] = off[u + 1] - off[u];
    row_label[k] = new_of[u];
    row_orig[k] = u;
    deg_rows[k] = indeg[u];
  }
}

__global__ void narrow_u64_kernel(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                                  uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<uint32_t>(in[i]);
}

// Twin targets: storage row k = original row sigma[k], every target w
// renamed new_of[w], same order. Rows of <= 8 edges (most of an R-MAT
// graph) one per thread; longer rows one per warp.
__global__ void twin_rows_kernel(const uint32_t* __restrict__ off, const uint32_t* __restrict__ tgt,
                                 const uint32_t* __restrict__ sigma,
                                 const uint32_t* __restrict__ new_of, uint64_t k_short, uint64_t n,
                                 const uint32_t* __restrict__ off_tw, uint32_t* __restrict__ tgt_tw) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  // long rows [0, k_short): a warp each
  for (uint64_t k = tid >> 5; k < k_short; k += nthreads >> 5) {
    const uint32_t u = sigma[k];
    const uint32_t b = off[u], len = off[u + 1] - b;
    uint32_t* dst = tgt_tw + off_tw[k];
    for (uint32_t i = lane; i < len; i += 32) dst[i] = new_of[__ldcs(tgt + b + i)];
  }
  // short rows [k_short, n): a thread each
  for (uint64_t k = k_short + tid; k < n; k += nthreads) {
    const uint32_t u = sigma[k];
    const uint32_t b = off[u], len = off[u + 1] - b;
    uint32_t* dst = tgt_tw + off_tw[k];
    for (uint32_t i = 0; i < len; ++i) dst[i] = new_of[__ldcs(tgt + b + i)];
  }
}

// first storage row whose length is <= lim (rows sorted by length, descending)
__global__ void first_short_kernel(const uint32_t* __restrict__ off_tw, uint64_t n, uint32_t lim,
                                   uint64_t* out) {
  if (threadIdx.x || blockIdx.x) return;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (off_tw[mid + 1] - off_tw[mid] > lim) lo = mid + 1;
    else hi = mid;
  }
  *out = lo;
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
  const uint32_t* order;   // the range's rows by length, descending
  uint32_t nA, nB, m;      // class boundaries in `order`, range size
  uint32_t b_ctas;         // CTAs of class B (then class C)
  uint64_t c_end;          // end (absolute row) of the class-C rows (twin: first empty row)
  int score_to_norm;       // last step on the twin: scores by label into norm_out (then gathered)
  uint64_t row_begin, row_end;
  double base, damp;
  int last;
  // relabelled twin (see tg_graph): row r is stored at position r in length
  // order; its vectors are indexed by label[r]; its score goes to
  // score_out[score_index[r]] (the original id). Both null otherwise.
  const uint32_t* label;
  const uint32_t* score_index;
  // fused exchange: the same row also goes to every peer's norm / score
  // vector (NVLink P2P stores), replacing the all-gather of a partitioned run
  uint32_t n_peers;
  double* peer_norm[TG_MAX_DEVICES];
  double* peer_score[TG_MAX_DEVICES];
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
  if (a.last && a.score_to_norm) {
    a.norm_out[a.label ? a.label[r] : r] = nx;  // by label; score_gather_kernel un-permutes
  } else if (a.last) {
    a.score_out[a.score_index ? a.score_index[r] : r] = nx;
    for (uint32_t p = 0; p < a.n_peers; ++p) a.peer_score[p][r] = nx;
  } else {
    const uint32_t d = a.deg[r];  // in storage order
    const double v = __ddiv_rn(nx, static_cast<double>(d > 1u ? d : 1u));  // scoring.cpp:61
    const uint64_t o = a.label ? a.label[r] : r;
    a.norm_out[o] = v;
    for (uint32_t p = 0; p < a.n_peers; ++p) a.peer_norm[p][o] = v;
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

// Hub path: one CTA per long row, with the row's strictly sequential sum
//   acc = 0; for w in row: acc = RN(acc + norm[w])          (scoring.cpp:66-68)
// evaluated EXACTLY, but in parallel, instead of as one serial DADD chain
// (the chain costs 8 cycles per edge: 450 us for the 77k-edge row at C2).
//
// Why this is exact: all addends are finite and >= 0, so acc never decreases.
// While acc stays inside one binade [2^E, 2^(E+1)) its grid step is
// u = 2^(E-52), acc = m*u with integer m in [2^52, 2^53), and
//   RN(m*u + x) = (m + X + t)*u,  X = floor(x/u),  f = x/u - X,
//   t = 1 if f > 1/2, or f == 1/2 and (m + X) is odd (ties to even), else 0,
// as long as the result stays below 2^(E+1) (m + X + t <= 2^53). So inside a
// binade each addend contributes an integer increment that depends on the
// running m only through its parity. An increment is a pair (d0, d1) — the
// increment for incoming parity 0 and 1 — and pairs compose associatively:
//   (F then G).d[p] = F.d[p] + G.d[p ^ (F.d[p] & 1)].
// A block-wide scan of these pairs gives m after every addend. The first
// addend that would leave the binade (m >= 2^53) is added with a real
// __dadd_rn; the pass then restarts from the next addend in the new binade.
// acc crosses a binade only O(log(sum / first)) times per row, mostly in its
// first elements, so a 2048-element tile takes one or two passes.
constexpr long long kTop = 1ll << 53;
constexpr int kHubSerial = 256;                   // serial prefix at a row start

struct QPair {
  long long d0, d1;
};

__device__ __forceinline__ QPair q_compose(const QPair f, const QPair g) {
  QPair c;  // saturate at 2^53: anything beyond only has to read as "crossed"
  c.d0 = f.d0 >= kTop ? kTop : min(kTop, f.d0 + ((f.d0 & 1) ? g.d1 : g.d0));
  c.d1 = f.d1 >= kTop ? kTop : min(kTop, f.d1 + ((f.d1 & 1) ? g.d0 : g.d1));
  return c;
}

__device__ __forceinline__ QPair q_shfl_up(const QPair v, int o) {
  QPair r;
  r.d0 = __shfl_up_sync(0xffffffffu, v.d0, o);
  r.d1 = __shfl_up_sync(0xffffffffu, v.d1, o);
  return r;
}

// x * 2^k exactly. Fast path: x normal and the result normal, so only the
// exponent field moves. Otherwise two multiplications by normal powers of two
// (an underflow only happens for x/u < 2^-1000, where "f < 1/2" is still
// decided correctly; an overflow saturates to "crossed").
__device__ __forceinline__ double scale_pow2(double x, int k) {
  const long long xb = __double_as_longlong(x);
  const int ex = static_cast<int>(xb >> 52);  // x >= 0
  if (ex != 0 && ex + k > 0 && ex + k < 2047)
    return __longlong_as_double(xb + (static_cast<long long>(k) << 52));
  const int k1 = k / 2, k2 = k - k1;
  const double f1 = __longlong_as_double(static_cast<long long>(k1 + 1023) << 52);
  const double f2 = __longlong_as_double(static_cast<long long>(k2 + 1023) << 52);
  return __dmul_rn(__dmul_rn(x, f1), f2);
}

// The increment pair of addend x in the binade with grid step 2^(E-52).
// X = floor(x/u) and f = x/u - X without int<->fp conversions: for
// 0 <= sc < 2^52, sc + 2^52 rounded toward zero is exactly 2^52 + floor(sc).
__device__ __forceinline__ QPair q_of(double x, int E) {
  const double sc = scale_pow2(x, 52 - E);
  constexpr double k2p52 = 4503599627370496.0;
  if (!(sc < 2.0 * k2p52)) return QPair{kTop, kTop};  // >= 2^53, inf or NaN
  long long X;
  double f;
  if (sc < k2p52) {
    const double y = __dadd_rz(sc, k2p52);
    X = __double_as_longlong(y) & ((1ll << 52) - 1);
    f = __dsub_rn(sc, __dsub_rn(y, k2p52));  // exact
  } else {
    X = (__double_as_longlong(sc) & ((1ll << 52) - 1)) | (1ll << 52);  // sc is an integer
    f = 0.0;
  }
  const bool up = f > 0.5, tie = f == 0.5;
  const long long odd = X & 1;
  return QPair{X + ((up || (tie && odd)) ? 1 : 0), X + ((up || (tie && !odd)) ? 1 : 0)};
}

// Tie-free fast path: the increment of x when no addend of the pass sits
// exactly on a half-step (then the parity of m never matters and the pairs
// collapse to one integer). *tie reports a half-step; kTop = "crossed".
__device__ __forceinline__ long long q_single(double x, int E, bool* tie) {
  const double sc = scale_pow2(x, 52 - E);
  constexpr double k2p52 = 4503599627370496.0;
  if (!(sc < 2.0 * k2p52)) return kTop;
  if (sc >= k2p52) return (__double_as_longlong(sc) & ((1ll << 52) - 1)) | (1ll << 52);
  const double y = __dadd_rz(sc, k2p52);
  const double f = __dsub_rn(sc, __dsub_rn(y, k2p52));
  *tie |= f == 0.5;
  return (__double_as_longlong(y) & ((1ll << 52) - 1)) + (f > 0.5 ? 1 : 0);
}

__device__ __forceinline__ long long sat_add(long long a, long long b) {
  return min(a + b, kTop);  // a, b <= 2^53: no overflow
}

template <int W>
struct HubShared {
  QPair wagg[W];  // per-warp totals, then their exclusive prefixes
  long long wsum[W];  // tie-free path: the same for plain increments
  long long wsum_tot;
  QPair wtot;             // block total
  int wfirst[W];  // per-warp first crossing
  double acc;
};

// Class A: one CTA per row longer than kLenA.
template <int W, int T>
// at most 80 registers: a 512-thread class-A CTA (16 warps x 2,560 registers)
// then leaves room on its SM for one class-B/C CTA (8 x 2,560), which 90
// registers (3,072 per warp) did not
__global__ void __maxnreg__(80) pr_hub_kernel(const PrStepArgs a, uint32_t row0) {
  constexpr int kHubWarps = W;
  constexpr int kHubThreads = W * 32;
  constexpr int kHubT = T;
  constexpr int kHubTile = kHubThreads * kHubT;
  extern __shared__ __align__(16) double xs[];  // [kHubTile]
  __shared__ HubShared<W> sh;
  const uint32_t r = a.order ? a.order[row0 + blockIdx.x]
                             : static_cast<uint32_t>(a.row_begin + row0 + blockIdx.x);  // class A
  const uint32_t beg = a.off[r], len = a.off[r + 1] - beg;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  double acc = 0.0;  // scoring.cpp:67 — identical in every thread
  // software pipeline: this thread's 8 addends of the next tile
  double x_next[kHubT];
  auto load_tile = [&](uint32_t base) {
    uint32_t t[kHubT];
#pragma unroll
    for (int k = 0; k < kHubT; ++k) {
      const uint32_t j = base + tid * kHubT + k;
      t[k] = j < len ? __ldg(a.tgt + beg + j) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kHubT; ++k) {
      const uint32_t j = base + tid * kHubT + k;
      x_next[k] = j < len ? __ldg(a.norm_in + t[k]) : 0.0;
    }
  };
  load_tile(0);
  for (uint32_t base = 0; base < len; base += kHubTile) {
    const int cnt = static_cast<int>(len - base < (uint32_t)kHubTile ? len - base : (uint32_t)kHubTile);
    double x[kHubT];
#pragma unroll
    for (int k = 0; k < kHubT; ++k) {
      x[k] = x_next[k];
      xs[tid * kHubT + k] = x[k];
    }
    if (base + kHubTile < len) load_tile(base + kHubTile);  // next tile in flight
    __syncthreads();
    int k0 = 0;  // first addend of this tile not yet in acc
    while (k0 < cnt) {
      if (acc == 0.0) {
        // Row start (or an all-zero prefix): acc crosses binades every few
        // addends here, so one thread runs the plain chain over the next 256.
        if (tid == 0) {
          const int stop = k0 + kHubSerial < cnt ? k0 + kHubSerial : cnt;
          double s0 = 0.0;
          for (int j = k0; j < stop; ++j) s0 = __dadd_rn(s0, xs[j]);  // scoring.cpp:68
          sh.acc = s0;
        }
        __syncthreads();
        acc = sh.acc;
        k0 = k0 + kHubSerial < cnt ? k0 + kHubSerial : cnt;
        __syncthreads();
        continue;
      }
      const long long bits = __double_as_longlong(acc);
      const int ef = static_cast<int>(bits >> 52);
      const int E = ef ? ef - 1023 : -1022;
      const long long m0 = (bits & ((1ll << 52) - 1)) | (ef ? (1ll << 52) : 0ll);
      const int p0 = static_cast<int>(m0 & 1);
      const long long room = kTop - m0;  // crossing when the increment reaches it
      int mine = kHubTile;
      long long before = 0;  // increment before this thread's first crossing
      int jc = kHubTile;
      long long total = 0;
      // ---- tie-free fast path: plain saturating int64 prefix sums
      bool tie = false;
      long long inc[kHubT];
      long long run1 = 0;
#pragma unroll
      for (int k = 0; k < kHubT; ++k) {
        const int j = tid * kHubT + k;
        if (j >= k0 && j < cnt) run1 = sat_add(run1, q_single(x[k], E, &tie));
        inc[k] = run1;
      }
      long long v1 = run1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, v1, o);
        if (lane >= o) v1 = sat_add(y, v1);
      }
      if (lane == 31) sh.wsum[w] = v1;
      const bool any_tie = __syncthreads_or(tie);
      if (!any_tie) {
        if (w == 0) {
          long long vi = lane < kHubWarps ? sh.wsum[lane] : 0;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, vi, o);
            if (lane >= o) vi = sat_add(y, vi);
          }
          long long ex = __shfl_up_sync(0xffffffffu, vi, 1);
          if (lane == 0) ex = 0;
          if (lane < kHubWarps) sh.wsum[lane] = ex;
          if (lane == kHubWarps - 1) sh.wsum_tot = vi;
        }
        __syncthreads();
        long long ex1 = __shfl_up_sync(0xffffffffu, v1, 1);
        if (lane == 0) ex1 = 0;
        const long long pre1 = sat_add(sh.wsum[w], ex1);
#pragma unroll
        for (int k = 0; k < kHubT; ++k) {
          const int j = tid * kHubT + k;
          const long long c = sat_add(pre1, inc[k]);
          if (mine == kHubTile && j >= k0 && j < cnt && c >= room) {
            mine = j;
            before = k ? sat_add(pre1, inc[k - 1]) : pre1;
          }
        }
        total = sh.wsum_tot;
      } else {
      // ---- general path: parity-dependent increment pairs (ties to even)
      QPair run{0, 0};
#pragma unroll
      for (int k = 0; k < kHubT; ++k) {
        const int j = tid * kHubT + k;
        if (j >= k0 && j < cnt) run = q_compose(run, q_of(x[k], E));
      }
      // warp inclusive scan, then warp 0 scans the warp totals
      QPair v = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const QPair y = q_shfl_up(v, o);
        if (lane >= o) v = q_compose(y, v);
      }
      if (lane == 31) sh.wagg[w] = v;
      __syncthreads();
      if (w == 0) {
        const QPair t = lane < kHubWarps ? sh.wagg[lane] : QPair{0, 0};
        QPair vi = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const QPair y = q_shfl_up(vi, o);
          if (lane >= o) vi = q_compose(y, vi);
        }
        QPair ex = q_shfl_up(vi, 1);
        if (lane == 0) ex = QPair{0, 0};
        if (lane < kHubWarps) sh.wagg[lane] = ex;
        if (lane == kHubWarps - 1) sh.wtot = vi;
      }
      __syncthreads();
      QPair excl = q_shfl_up(v, 1);
      if (lane == 0) excl = QPair{0, 0};
      const QPair pre = q_compose(sh.wagg[w], excl);
      // m after each addend; this thread's first addend that leaves the binade
      {
        QPair c = pre;
#pragma unroll
        for (int k = 0; k < kHubT; ++k) {
          const int j = tid * kHubT + k;
          if (mine == kHubTile && j >= k0 && j < cnt) {
            const long long b = p0 ? c.d1 : c.d0;
            c = q_compose(c, q_of(x[k], E));
            if ((p0 ? c.d1 : c.d0) >= room) {
              mine = j;
              before = b;
            }
          }
        }
      }
      total = p0 ? sh.wtot.d1 : sh.wtot.d0;
      }
      // first crossing: crossings are monotone in the addend index, so it is
      // the lowest crossing lane of the lowest warp that has one
      const unsigned cm = __ballot_sync(0xffffffffu, mine < kHubTile);
      const int first_mine = __shfl_sync(0xffffffffu, mine, cm ? __ffs(cm) - 1 : 0);
      if (lane == 0) sh.wfirst[w] = cm ? first_mine : kHubTile;
      __syncthreads();
#pragma unroll
      for (int ww = 0; ww < kHubWarps; ++ww) jc = min(jc, sh.wfirst[ww]);
      const double u = (E - 52) >= -1022
                           ? __longlong_as_double(static_cast<long long>(E - 52 + 1023) << 52)
                           : __longlong_as_double(1ll << (E - 52 + 1074));
      if (jc == kHubTile) {
        // no crossing: acc = (m0 + total) * u exactly; every thread computes it
        acc = __dmul_rn(static_cast<double>(m0 + total), u);
        k0 = cnt;
      } else {
        // the owner of addend jc: exact value before it, then one real DADD
        if (mine == jc) {
          const double prev = __dmul_rn(static_cast<double>(m0 + before), u);
          sh.acc = __dadd_rn(prev, xs[jc]);  // scoring.cpp:68
        }
        __syncthreads();
        acc = sh.acc;
        k0 = jc + 1;
      }
      __syncthreads();
    }
  }
  if (tid == 0) finish_row(a, r, acc);
}

// Class B: 8 lanes per row (4 rows per warp, near-equal lengths). The 8
// lanes stream their row's targets in 64-edge windows (32 B coalesced per
// row), gather the normalized values into shared memory with the next
// window's gathers and the window after's targets in flight, and the group's
// first lane adds each window in storage order — 4 chains per warp.
#ifndef TG_PR_BLANES  // lanes per class-B row (compile-time experiment knob)
#define TG_PR_BLANES 8
#endif
constexpr int kBLanes = TG_PR_BLANES;
constexpr int kBWin = kBLanes * 8;  // 64 edges per window
// a group's window buffer stride: one double of padding puts the four chain
// lanes of a warp (one per group) on different banks (ncu: 4-way conflicts)
constexpr int kBStride = kBWin + 1;
__device__ __forceinline__ void group_row(const PrStepArgs& a, int64_t i, double* buf) {
  const int lane = threadIdx.x & 31, sl = lane & (kBLanes - 1);
  const bool has = i < static_cast<int64_t>(a.nB);
  const uint32_t r = has ? (a.order ? a.order[i] : static_cast<uint32_t>(a.row_begin + i)) : 0u;
  const uint32_t beg = has ? a.off[r] : 0u;
  const uint32_t len = has ? a.off[r + 1] - beg : 0u;
  constexpr int K = kBWin / kBLanes;  // 8 per lane per window
  uint32_t t1[K];
  double v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint32_t e = k * kBLanes + sl;
    t1[k] = e < len ? __ldg(a.tgt + beg + e) : 0xffffffffu;
  }
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = t1[k] != 0xffffffffu ? __ldg(a.norm_in + t1[k]) : 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint32_t e = kBWin + k * kBLanes + sl;
    t1[k] = e < len ? __ldg(a.tgt + beg + e) : 0xffffffffu;
  }
  // the warp loops until its longest row is done (lengths are near-equal)
  uint32_t wmax = len;
#pragma unroll
  for (int o = 16; o; o >>= 1) wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
  double acc = 0.0;  // scoring.cpp:67
  for (uint32_t wb = 0; wb < wmax; wb += kBWin) {
#pragma unroll
    for (int k = 0; k < K; ++k) buf[k * kBLanes + sl] = v[k];
    __syncwarp();
    double vn[K];
#pragma unroll
    for (int k = 0; k < K; ++k) vn[k] = t1[k] != 0xffffffffu ? __ldg(a.norm_in + t1[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint32_t e = wb + 2 * kBWin + k * kBLanes + sl;
      t1[k] = e < len ? __ldg(a.tgt + beg + e) : 0xffffffffu;
    }
    if (sl == 0 && wb < len)
      acc = chain_add(acc, buf, len - wb < (uint32_t)kBWin ? len - wb : kBWin);  // in order
    __syncwarp();
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = vn[k];
  }
  if (has && sl == 0) finish_row(a, r, acc);
}

// Class C: one thread per row of at most kLenB edges, in storage order. A
// warp's 32 rows have near-equal lengths (length-sorted schedule), so the
// lanes stay converged; 8 gathers per lane are in flight per step.
__device__ __forceinline__ void thread_row(const PrStepArgs& a, uint32_t r) {
  const uint32_t beg = a.off[r], len = a.off[r + 1] - beg;
  const uint32_t* t = a.tgt + beg;
  double acc = 0.0;  // scoring.cpp:67
  uint32_t k = 0;
  // peel to a 16 B boundary (its loads independent of each other), then two
  // 16 B target loads per 8 edges, the next group's targets in flight
  const uint32_t peel = min(len, (4u - (beg & 3u)) & 3u);
  if (peel) {
    uint32_t ti[3];
    double v[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) ti[q] = q < (int)peel ? __ldg(t + q) : 0u;
#pragma unroll
    for (int q = 0; q < 3; ++q) v[q] = q < (int)peel ? __ldg(a.norm_in + ti[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < 3; ++q)
      if (q < (int)peel) acc = __dadd_rn(acc, v[q]);
    k = peel;
  }
  if (k + 8 <= len) {
    uint4 q0 = __ldg(reinterpret_cast<const uint4*>(t + k));
    uint4 q1 = __ldg(reinterpret_cast<const uint4*>(t + k + 4));
    for (; k + 8 <= len; k += 8) {
      const uint32_t ti[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
      if (k + 16 <= len) {
        q0 = __ldg(reinterpret_cast<const uint4*>(t + k + 8));
        q1 = __ldg(reinterpret_cast<const uint4*>(t + k + 12));
      }
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldg(a.norm_in + ti[q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, v[q]);
    }
  }
  if (k < len) {
    uint32_t ti[8];
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) ti[q] = k + q < len ? __ldg(t + k + q) : 0u;
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = k + q < len ? __ldg(a.norm_in + ti[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (k + q < len) acc = __dadd_rn(acc, v[q]);
  }
  finish_row(a, r, acc);
}

// Class C on the relabelled twin, whose rows are STORED in length order: a
// warp's 32 rows are consecutive in storage, so their concatenated targets
// are one contiguous range. The warp streams it in chunks of kCWin edges
// (coalesced 4 B target loads, the next chunk's targets in flight), gathers
// the normalized values into shared memory, and every lane then adds its own
// row's part of the chunk in storage order (scoring.cpp:66-68) -- the same
// left-to-right chain per row as thread_row, with coalesced target traffic.
#ifndef TG_PR_CWIN  // class-C chunk on the twin (compile-time experiment knob)
#define TG_PR_CWIN 256
#endif
constexpr int kCWin = TG_PR_CWIN;  // edges per chunk (8 per lane at 256)
__device__ __forceinline__ void warp_rows_staged(const PrStepArgs& a, uint64_t k0, double* buf) {
  const int lane = threadIdx.x & 31;
  const uint64_t kend = min(k0 + 32, a.c_end);
  const uint32_t nrows = static_cast<uint32_t>(kend > k0 ? kend - k0 : 0);
  if (nrows == 0) return;
  const uint32_t e0 = a.off[k0], e1 = a.off[k0 + nrows];
  const bool has = static_cast<uint32_t>(lane) < nrows;
  const uint32_t rb = has ? a.off[k0 + lane] - e0 : 0u, re = has ? a.off[k0 + lane + 1] - e0 : 0u;
  const uint32_t total = e1 - e0;
  const uint32_t* t = a.tgt + e0;
  constexpr int K = kCWin / 32;
  uint32_t tn[K];
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const uint32_t j = q * 32 + lane;
    tn[q] = j < total ? __ldcs(t + j) : 0xffffffffu;
  }
  double acc = 0.0;  // scoring.cpp:67
  for (uint32_t base = 0; base < total; base += kCWin) {
    double v[K];
#pragma unroll
    for (int q = 0; q < K; ++q) v[q] = tn[q] != 0xffffffffu ? __ldg(a.norm_in + tn[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < K; ++q) {  // next chunk's targets in flight
      const uint32_t j = base + kCWin + q * 32 + lane;
      tn[q] = j < total ? __ldcs(t + j) : 0xffffffffu;
    }
#pragma unroll
    for (int q = 0; q < K; ++q) buf[q * 32 + lane] = v[q];
    __syncwarp();
    const uint32_t lo = max(rb, base), hi = min(re, base + kCWin);
    for (uint32_t j = lo; j < hi; ++j) acc = __dadd_rn(acc, buf[j - base]);  // in order
    __syncwarp();
  }
  if (has) finish_row(a, k0 + lane, acc);
}

// Class C on the relabelled twin, streamed (TIERGRAPH_PR_CSTREAM=1; default
// off: at C3 a step takes 24.2 ms with it against 14.2 ms with the warp-staged
// class C of pr_step_kernel, profiles/r02g): one warp takes kCsRows consecutive rows (one contiguous edge range,
// rows stored in length order) and streams it in kCsChunk-edge chunks with
// the memory pipeline never drained: cp.async copies the targets three
// chunks ahead (16 B, coalesced) and gathers the normalized values one chunk
// ahead straight into shared memory (8 B cp.async, no registers held), while
// the lanes add the current chunk. Row j of the warp belongs to lane j % 32,
// which adds its part of every chunk the row spans in storage order
// (scoring.cpp:66-68: the same left-to-right chain as thread_row), carrying
// the accumulator across chunk boundaries.
constexpr int kCsWarps = 4, kCsRows = 256, kCsChunk = 256;
constexpr int kCsTRing = 3, kCsVRing = 2;
struct CsWarpSmem {
  uint32_t off[kCsRows + 4];
  uint32_t t[kCsTRing][kCsChunk];
  double v[kCsVRing][kCsChunk];
};
constexpr int kCsSmem = kCsWarps * static_cast<int>(sizeof(CsWarpSmem));

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(kCsWarps * 32) pr_cstream_kernel(const PrStepArgs a,
                                                                   uint64_t c_begin) {
  extern __shared__ __align__(16) uint8_t cs_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  CsWarpSmem& S = reinterpret_cast<CsWarpSmem*>(cs_smem)[w];
  const uint64_t k0 = c_begin + ((uint64_t)blockIdx.x * kCsWarps + w) * kCsRows;
  if (k0 >= a.c_end) return;
  const uint32_t nrows = static_cast<uint32_t>((a.c_end - k0 < (uint64_t)kCsRows ? a.c_end - k0 : (uint64_t)kCsRows));
  for (uint32_t j = lane; j <= nrows; j += 32) S.off[j] = a.off[k0 + j];
  __syncwarp();
  const uint32_t e0 = S.off[0], e1 = S.off[nrows];
  const uint32_t A = e0 & ~3u;  // chunks on a 16 B grid of the target array
  const uint32_t nch = (e1 - A + kCsChunk - 1) / kCsChunk;
  auto load_t = [&](uint32_t c) {  // targets of chunk c: 64 x 16 B, 2 per lane
    if (c < nch) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t i = q * 32 + lane;
        const uint32_t pos = A + c * kCsChunk + 4 * i;
        const uint32_t nb = pos < e1 ? min(16u, 4 * (e1 - pos)) : 0u;
        cp_async16(&S.t[c % kCsTRing][4 * i], a.tgt + (nb ? pos : A), nb);
      }
    }
    cp_async_commit();
  };
  auto gather = [&](uint32_t c) {  // normalized values of chunk c: 8 per lane
    if (c < nch) {
      const uint32_t* tt = S.t[c % kCsTRing];
#pragma unroll
      for (int q = 0; q < kCsChunk / 32; ++q) {
        const uint32_t p = q * 32 + lane;
        const uint32_t pos = A + c * kCsChunk + p;
        const bool ok = pos >= e0 && pos < e1;
        cp_async8(&S.v[c % kCsVRing][p], a.norm_in + (ok ? tt[p] : 0u), ok ? 8u : 0u);
      }
    }
    cp_async_commit();
  };
  load_t(0);
  load_t(1);
  cp_async_wait<1>();  // T0
  __syncwarp();
  gather(0);
  load_t(2);
  uint32_t j = lane;
  double acc = 0.0;  // scoring.cpp:67
  for (uint32_t c = 0; c < nch; ++c) {
    cp_async_wait<1>();  // everything but T(c+2): V(c) and T(c+1) have landed
    __syncwarp();
    gather(c + 1);
    load_t(c + 3);  // into T(c)'s slot: T(c) was last read by gather(c)
    const double* vv = S.v[c % kCsVRing];
    const uint32_t cb = A + c * kCsChunk, ce = cb + kCsChunk;
    while (j < nrows) {
      const uint32_t rs = S.off[j], re = S.off[j + 1];
      if (rs >= ce) break;  // starts after this chunk
      const uint32_t lo = max(rs, cb), hi = min(re, ce);
      for (uint32_t k = lo; k < hi; ++k) acc = __dadd_rn(acc, vv[k - cb]);  // in order
      if (re > ce) break;  // continues in the next chunk
      finish_row(a, k0 + j, acc);
      acc = 0.0;
      j += 32;
    }
    __syncwarp();  // V(c)'s slot is refilled by gather(c + 2)
  }
  cp_async_wait<0>();
  for (; j < nrows; j += 32) finish_row(a, k0 + j, 0.0);  // empty rows at the very end
}

// The twin's last step leaves the scores in label order (sequential stores);
// out[u] = scores[new_of[u]] puts them back in the graph's ids as a gather
// (whole-sector stores) instead of 111M scattered 8 B stores, each of which
// makes L2 fill its sector from DRAM first (C3 last step 10.3 vs 8.9 ms).
__global__ void __launch_bounds__(256) score_gather_kernel(const double* __restrict__ by_label,
                                                           const uint32_t* __restrict__ new_of,
                                                           uint64_t n, double* __restrict__ out) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x)
    out[u] = by_label[__ldcs(new_of + u)];
}

// Rows without edges on the relabelled twin (61 % of the C3 rows): their
// row sum is 0.0, so every step writes the same norm = base / max(deg, 1)
// (scoring.cpp:59-70 with an empty chain) and the last step the same score =
// base. A streaming epilogue instead of a warp per 32 rows; the caller skips
// it once both Jacobi buffers hold the value (steps 3 .. n-1).
__global__ void __launch_bounds__(256) pr_empty_kernel(const PrStepArgs a, uint64_t k_begin) {
  for (uint64_t k = k_begin + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < a.row_end;
       k += (uint64_t)gridDim.x * blockDim.x)
    finish_row(a, k, 0.0);
}

// MinB: CTAs per SM the register allocation must allow (1: no cap, 71
// registers, 3 CTAs fit; 4: <= 64 registers). TIERGRAPH_PR_MINB=1|4 overrides
// the default (4 on the relabelled twin, else 1).
template <int MinB>
__global__ void __launch_bounds__(kPrWarps * 32, MinB) pr_step_kernel(const PrStepArgs a) {
  // class B windows (16.6 KB) or, on the twin, class C chunks (16 KB)
  constexpr int kSmemB = kPrWarps * 32 / kBLanes * kBStride, kSmemC = kPrWarps * kCWin;
  __shared__ __align__(16) double smem[kSmemB > kSmemC ? kSmemB : kSmemC];
  if (blockIdx.x < a.b_ctas) {
    const int g = threadIdx.x / kBLanes;  // row group within the CTA
    const int64_t i = a.nA + (int64_t)blockIdx.x * (kPrWarps * 32 / kBLanes) + g;
    group_row(a, i, smem + g * kBStride);
  } else if (!a.order) {
    // storage-sorted twin: 32 consecutive rows per warp, staged chunks
    const int w = threadIdx.x >> 5;
    const uint64_t k0 = a.row_begin + a.nB + ((uint64_t)(blockIdx.x - a.b_ctas) * kPrWarps + w) * 32;
    warp_rows_staged(a, k0, smem + w * kCWin);
  } else {
    const uint64_t i = a.nB + (uint64_t)(blockIdx.x - a.b_ctas) * blockDim.x + threadIdx.x;
    if (i < a.m) thread_row(a, a.order[i]);
  }
}

// The memory-system floor of one K3 step on this graph: the same E gathers
// x[tgt[e]] streamed over the same u32 targets, summed with no ordering
// constraint (one partial per thread). K3 / this = distance to the floor.
__global__ void __launch_bounds__(256) gather_floor_kernel(const uint32_t* __restrict__ tgt,
                                                           uint64_t e, const double* __restrict__ x,
                                                           double* __restrict__ sink) {
  double acc = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < e; i += 4 * stride) {
    const uint32_t a = __ldg(tgt + i), b = __ldg(tgt + i + stride), c = __ldg(tgt + i + 2 * stride),
                   d = __ldg(tgt + i + 3 * stride);
    acc += __ldg(x + a) + __ldg(x + b) + __ldg(x + c) + __ldg(x + d);
  }
  for (; i < e; i += stride) acc += __ldg(x + __ldg(tgt + i));
  if (acc == -1.0) sink[0] = acc;  // never true: keeps the loads alive
}

// Cross-GPU barrier of the fused exchange: release this rank's P2P stores
// (everything earlier on the stream), bump every peer's arrival counter, then
// wait until this rank's counter reaches `target`. A wait longer than ~2 s
// sets *err and returns instead of hanging the device.
struct PeerFlags {
  unsigned* peer[TG_MAX_DEVICES];
};
__global__ void peer_barrier_kernel(unsigned* local, PeerFlags peers, uint32_t n, unsigned target,
                                    unsigned* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  __threadfence_system();
  for (uint32_t p = 0; p < n; ++p) atomicAdd_system(peers.peer[p], 1u);
  const long long t0 = clock64();
  while (true) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(local) : "memory");
    if (v >= target) break;
    if (clock64() - t0 > 4000000000ll) {
      atomicExch(err, 1u);
      break;
    }
    __nanosleep(200);
  }
  __threadfence_system();
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
  if (compute_indeg_binned(ctx, g->tgt, g->e, g->n, deg)) return;  // indegree.cu
  const unsigned grid = grid_for(g->e / 4 + 1, 512, ctx->num_sms * 4);
  indeg_kernel<<<grid, 512, 0, ctx->stream>>>(g->tgt, g->e, static_cast<uint32_t>(g->n), deg);
  TGB_LAUNCHED();
}

// Prepares deg + norm0 for the weighted (tid != nullptr) or plain recurrence.
// Out-of-range train ids set *bad (min index) and are skipped; the caller
// checks it after the run (no synchronisation here).
// norm0[j] = score0[j] / max(deg[j],1) from final in-degrees `deg` (K2).
// Out-of-range train ids set *bad (min index) and are skipped; the caller
// checks it after the run (no synchronisation here). `relabel` maps train ids
// into a relabelled twin's ids.
void pagerank_init(tg_ctx* ctx, uint64_t n, const uint64_t* tid_dev, uint64_t ntid,
                   const uint32_t* deg, double* norm0, unsigned long long* bad,
                   const uint32_t* relabel) {
  const double init = 1.0 / static_cast<double>(n);  // scoring.cpp:96
  double weight = 1.0;
  uint32_t* mult = nullptr;
  if (tid_dev) {
    weight = static_cast<double>(n) / static_cast<double>(ntid);  // scoring.cpp:94-95
    mult = ctx->scratch_t<uint32_t>(kScratchF, n);
    TGB_CUDA(cudaMemsetAsync(mult, 0, sizeof(uint32_t) * n, ctx->stream));
    train_mult_kernel<<<grid_for(ntid, 256), 256, 0, ctx->stream>>>(tid_dev, ntid, n, relabel,
                                                                     mult, bad);
    TGB_LAUNCHED();
  }
  pr_init_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(deg, mult, n, init, weight, norm0);
  TGB_LAUNCHED();
}

// The same from a whole graph's cached in-degrees (copied into deg when deg
// is not the graph's own array).
void pagerank_prepare(tg_ctx* ctx, const tg_graph* g, const uint64_t* tid_dev, uint64_t ntid,
                      uint32_t* deg, double* norm0, unsigned long long* bad,
                      const uint32_t* relabel = nullptr) {
  if (!whole_graph(g))
    domain_error("pagerank prepare: a row-block graph holds partial in-degrees; sum them "
                 "over the blocks and use tg_pagerank_init_async");
  if (deg != g->indeg)
    TGB_CUDA(cudaMemcpyAsync(deg, g->indeg, 4 * g->n, cudaMemcpyDeviceToDevice, ctx->stream));
  pagerank_init(ctx, g->n, tid_dev, ntid, deg, norm0, bad, relabel);
}

bool relabel_wanted(const tg_ctx* ctx, const tg_graph* g);

const tg_graph::Sched& schedule(tg_ctx* ctx, const tg_graph* g, uint64_t rb, uint64_t re) {
  auto& v = const_cast<tg_graph*>(g)->scheds;
  for (const auto& sc : v)
    if (sc.rb == rb && sc.re == re) return sc;
  tg_graph::Sched sc{rb, re, nullptr, 0, 0, 0};
  TGB_CUDA(tgb::dev_malloc(&sc.order, sizeof(uint32_t) * std::max<uint64_t>(re - rb, 1) + 16));
  sort_rows_by_length(ctx, g->off, rb, re, sc.order);
  uint32_t* bounds = sc.order + std::max<uint64_t>(re - rb, 1);
  // TIERGRAPH_PR_LENA / _LENB override the class boundaries (experiments)
  const char* ea = std::getenv("TIERGRAPH_PR_LENA");
  const char* eb = std::getenv("TIERGRAPH_PR_LENB");
  const uint32_t la = ea ? static_cast<uint32_t>(std::atoi(ea))
                         : static_cast<uint32_t>(std::max<uint64_t>(
                               kLenA, std::min<uint64_t>(g->e >> 14, kLenAMax)));
  // class B/C bound: 512, or 256 when K3 will run on the relabelled twin
  // (warp-staged class C over storage-consecutive rows; C3 10.1 -> 9.9 ms,
  // profiles/r02k)
  const uint32_t lbn = eb ? static_cast<uint32_t>(std::atoi(eb))
                          : (whole_graph(g) && relabel_wanted(ctx, g) ? kLenBTwin : kLenB);
  class_bounds_kernel<<<1, 32, 0, ctx->stream>>>(g->off, sc.order, re - rb, la, std::min(lbn, la),
                                                 bounds);
  TGB_LAUNCHED();
  uint32_t hb[3];
  TGB_CUDA(cudaMemcpyAsync(hb, bounds, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();  // once per (graph, range)
  sc.nA = hb[0];
  sc.nB = hb[1];
  sc.nLong = hb[2];
  v.push_back(sc);
  return v.back();
}

void pagerank_step(tg_ctx* ctx, const tg_graph* g, const uint32_t* deg, double damp,
                   const double* nin, double* nout, double* sout, uint64_t rb, uint64_t re,
                   int last, uint32_t n_peers, double* const* peer_norm,
                   double* const* peer_score, const uint32_t* score_index, int skip_empty,
                   int score_to_norm) {
  if (re <= rb) return;
  if (rb < g->rb || re > g->re)
    domain_error("pagerank step: rows [" + std::to_string(rb) + ", " + std::to_string(re) +
                 ") are not held by this graph (rows [" + std::to_string(g->rb) + ", " +
                 std::to_string(g->re) + "))");
  const tg_graph::Sched& sc = schedule(ctx, g, rb, re);
  PrStepArgs a;
  a.off = g->off;
  a.tgt = g->tgt;
  a.deg = g->deg_rows ? g->deg_rows : deg;  // the twin's in-degrees in storage order
  a.norm_in = nin;
  a.norm_out = nout;
  a.score_out = sout;
  a.order = sc.order;
  a.nA = sc.nA;
  a.nB = sc.nB;
  a.m = static_cast<uint32_t>(re - rb);
  constexpr uint32_t kRowsPerCta = kPrWarps * 32 / kBLanes;
  a.b_ctas = (sc.nB - sc.nA + kRowsPerCta - 1) / kRowsPerCta;
  a.row_begin = rb;
  a.row_end = re;
  a.base = (1.0 - damp) / static_cast<double>(g->n);  // scoring.cpp:53
  a.damp = damp;
  a.last = last;
  a.label = g->row_label;
  a.score_index = g->row_orig ? g->row_orig : score_index;
  a.n_peers = n_peers;
  for (uint32_t p = 0; p < TG_MAX_DEVICES; ++p) {
    a.peer_norm[p] = p < n_peers ? peer_norm[p] : nullptr;
    a.peer_score[p] = p < n_peers ? peer_score[p] : nullptr;
  }
  // twin: class C ends at the first empty row; the empty rows get their own epilogue
  const uint64_t mC = (!sc.order && sc.nE < a.m) ? sc.nE : a.m;
  a.c_end = rb + mC;
  a.score_to_norm = score_to_norm;
  uint64_t c_ctas = (mC - sc.nB + kPrWarps * 32 - 1) / (kPrWarps * 32);
  // class C streamed on its own stream (relabelled twin: rows in storage order)
  const char* csv = std::getenv("TIERGRAPH_PR_CSTREAM");
  const bool cstream = csv && csv[0] == '1';
  const bool cs = cstream && !sc.order && mC > sc.nB;
  if (cs) c_ctas = 0;
  if (sc.nA || cs) ctx->fork();
  if (cs) {
    static bool cattr[TG_MAX_DEVICES] = {};
    if (!cattr[ctx->device % TG_MAX_DEVICES]) {
      TGB_CUDA(cudaFuncSetAttribute(pr_cstream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kCsSmem));
      cattr[ctx->device % TG_MAX_DEVICES] = true;
    }
    const uint64_t warps = (mC - sc.nB + kCsRows - 1) / kCsRows;
    pr_cstream_kernel<<<static_cast<unsigned>((warps + kCsWarps - 1) / kCsWarps), kCsWarps * 32,
                        kCsSmem, ctx->aux3>>>(a, rb + sc.nB);
    TGB_LAUNCHED();
  }
  if (sc.nA) {
    // class A on the side streams, concurrently with classes B and C: the
    // longest rows (> kHubLong) with 512-thread CTAs, the rest with 256
    static bool attr[TG_MAX_DEVICES] = {};  // a function attribute is per device
    if (!attr[ctx->device % TG_MAX_DEVICES]) {
      TGB_CUDA(cudaFuncSetAttribute(pr_hub_kernel<16, 8>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 32 * 8 * 8));
      TGB_CUDA(cudaFuncSetAttribute(pr_hub_kernel<8, 8>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 32 * 8 * 8));
      attr[ctx->device % TG_MAX_DEVICES] = true;
    }
    const uint32_t nl = sc.nLong;
    if (nl) {
      pr_hub_kernel<16, 8><<<nl, 16 * 32, 16 * 32 * 8 * 8, ctx->aux>>>(a, 0);
      TGB_LAUNCHED();
    }
    if (sc.nA > nl) {
      pr_hub_kernel<8, 8><<<sc.nA - nl, 8 * 32, 8 * 32 * 8 * 8, ctx->aux2>>>(a, nl);
      TGB_LAUNCHED();
    }
  }
  const unsigned grid = static_cast<unsigned>(a.b_ctas + c_ctas);
  if (grid) {
    // classes B (first CTAs: long chains start early) and C in one grid
    // 4 CTAs per SM (<= 64 registers) on the relabelled twin, where the
    // classes B/C are latency-bound on L2-missing gathers (C3 step 10.8 ->
    // 10.2 ms, profiles/r02j); 3 (71 registers) otherwise
    const char* mb = std::getenv("TIERGRAPH_PR_MINB");
    const bool four = mb ? mb[0] == '4' : !a.order;
    if (four)
      pr_step_kernel<4><<<grid, kPrWarps * 32, 0, ctx->stream>>>(a);
    else
      pr_step_kernel<1><<<grid, kPrWarps * 32, 0, ctx->stream>>>(a);
    TGB_LAUNCHED();
  }
  if (sc.nA || cs) ctx->join();
  if (mC < a.m && !(skip_empty && !last)) {
    pr_empty_kernel<<<grid_for(a.m - mC, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(a,
                                                                                      rb + mC);
    TGB_LAUNCHED();
  }
}

// TIERGRAPH_PR_RELABEL: "0" never, "1" always, default: when the norm vector
// (8 B per node) is larger than half of L2, i.e. when K3's random gathers
// miss L2 (C3/C4), not at C1/C2 where the whole vector stays resident.
bool relabel_wanted(const tg_ctx* ctx, const tg_graph* g) {
  if (!whole_graph(g)) return false;
  if (const char* e = std::getenv("TIERGRAPH_PR_RELABEL")) return e[0] == '1';
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device);
  return g->n > 1 && 8.0 * static_cast<double>(g->n) > 0.5 * static_cast<double>(l2);
}

// Builds g->twin (see tg_graph). One-time per graph: a radix sort of N
// keys, two passes over N, a scan and one pass over the targets.
const tg_graph* relabel_twin(tg_ctx* ctx, const tg_graph* gc) {
  auto* g = const_cast<tg_graph*>(gc);
  if (g->twin || g->twin_tried) return g->twin;
  g->twin_tried = true;
  if (!relabel_wanted(ctx, g)) return nullptr;
  const uint64_t n = g->n, e = g->e;
  const tg_graph::Sched sg = schedule(ctx, g, 0, n);  // sigma: K3's row order
  auto* t = new tg_graph;
  t->ctx = ctx;
  t->n = n;
  t->e = e;
  t->rb = 0;
  t->re = n;
  uint64_t* lens = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  try {
    TGB_CUDA(tgb::dev_malloc(&g->old_of, 4 * n));
    TGB_CUDA(tgb::dev_malloc(&g->new_of, 4 * n));
    TGB_CUDA(tgb::dev_malloc(&t->off, 4 * (n + 1)));
    TGB_CUDA(tgb::dev_malloc(&t->tgt, 4 * std::max<uint64_t>(e, 1) + 16));  // +16: K3 reads 16 B target groups
    TGB_CUDA(tgb::dev_malloc(&t->indeg, 4 * n));
    TGB_CUDA(tgb::dev_malloc(&t->row_label, 4 * n));
    TGB_CUDA(tgb::dev_malloc(&t->row_orig, 4 * n));
    TGB_CUDA(tgb::dev_malloc(&t->deg_rows, 4 * n));
    TGB_CUDA(tgb::dev_malloc(&lens, 8 * (n + 1) + 16));
    TGB_CUDA(cudaEventCreate(&ev0));
    TGB_CUDA(cudaEventCreate(&ev1));
    TGB_CUDA(cudaEventRecord(ev0, ctx->stream));
    // Labels (TIERGRAPH_PR_LABEL):
    //   indeg  label = in-degree rank; rows stored in K3's length order, so
    //          a row's norm write goes to a scattered label;
    //   rows   label = storage row (length order): sequential norm writes,
    //          hub norms packed by out-degree;
    //   hybrid (default) rows stored by (class A: length; else length
    //          bucket 2^k, then in-degree), label = storage row: sequential
    //          writes AND, inside every length bucket, the most-gathered
    //          norms first. Class boundaries (4096, 512) are bucket edges, so
    //          the class A/B/C row sets are those of the length order.
    const char* lab = std::getenv("TIERGRAPH_PR_LABEL");
    const std::string mode = lab && lab[0] ? lab : "hybrid";
    uint32_t* sigma = sg.order;
    if (mode == "rows") {
      TGB_CUDA(cudaMemcpyAsync(g->old_of, sg.order, 4 * n, cudaMemcpyDeviceToDevice, ctx->stream));
    } else if (mode == "indeg") {
      sort_ids_by_value_desc(ctx, g->indeg, n, g->old_of);
    } else {
      uint32_t* key = reinterpret_cast<uint32_t*>(lens);  // lens is filled later
      hybrid_key_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(g->off, g->indeg, n, key);
      TGB_LAUNCHED();
      sort_ids_by_value_desc(ctx, key, n, g->old_of);
      sigma = g->old_of;
    }
    twin_labels_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(g->old_of, g->indeg, n,
                                                                  g->new_of, t->indeg);
    TGB_LAUNCHED();
    twin_rows_meta_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
        g->off, sigma, g->new_of, g->indeg, n, lens, t->row_label, t->row_orig, t->deg_rows);
    TGB_LAUNCHED();
    TGB_CUDA(cudaMemsetAsync(lens + n, 0, 8, ctx->stream));
    exclusive_scan_u64(ctx, lens, n + 1);
    narrow_u64_kernel<<<grid_for(n + 1, 256), 256, 0, ctx->stream>>>(lens, t->off, n + 1);
    TGB_LAUNCHED();
    if (e) {
      uint64_t* k_short = lens;  // reuse: lens is consumed
      first_short_kernel<<<1, 32, 0, ctx->stream>>>(t->off, n, 8, k_short);
      TGB_LAUNCHED();
      uint64_t ks = 0;
      TGB_CUDA(cudaMemcpyAsync(&ks, k_short, 8, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      twin_rows_kernel<<<ctx->num_sms * 16, 256, 0, ctx->stream>>>(
          g->off, g->tgt, sigma, g->new_of, ks, n, t->off, t->tgt);
      TGB_LAUNCHED();
    }
    TGB_CUDA(cudaEventRecord(ev1, ctx->stream));
    TGB_CUDA(cudaEventSynchronize(ev1));
    TGB_CUDA(cudaEventElapsedTime(&g->twin_ms, ev0, ev1));
    if (mode != "indeg") {  // label = storage row: K3 indexes by the row itself
      TGB_CUDA(cudaFree(t->row_label));
      t->row_label = nullptr;
    }
    // storage order IS the schedule: identity order, the same class bounds
    tg_graph::Sched tsc{0, n, nullptr, sg.nA, sg.nB, sg.nLong};
    tsc.nE = n;
    if (e) {  // first storage row without edges (empty rows are stored last)
      uint64_t* k_e = lens;
      first_short_kernel<<<1, 32, 0, ctx->stream>>>(t->off, n, 0, k_e);
      TGB_LAUNCHED();
      TGB_CUDA(cudaMemcpyAsync(&tsc.nE, k_e, 8, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
    }
    t->scheds.push_back(tsc);
  } catch (...) {
    cudaFree(lens);
    tg_graph_destroy(t);
    cudaFree(g->old_of);
    cudaFree(g->new_of);
    g->old_of = g->new_of = nullptr;
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    throw;
  }
  cudaFree(lens);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  g->twin = t;
  return t;
}

void check_config(uint32_t iterations, double damp) {  // scoring.cpp:42-47
  if (iterations < 1) domain_error("pagerank: iterations must be >= 1");
  if (!(damp > 0.0 && damp < 1.0))
    domain_error("pagerank: damp must lie in (0,1), got " + std::to_string(damp));
}

// L2 residency of the hot norm values (C3/C4, where the vector exceeds L2):
// on the relabelled twin the most-gathered nodes have the lowest labels, so
// the first bytes of norm_in are the hottest. They are marked persisting for
// every K3 launch of the run (an access-policy window on the three K3
// streams) so the streamed targets (4 B per edge, read once) cannot evict
// them; the lines are released when the run ends.
// TIERGRAPH_PR_PERSIST_MB: window size in MB (0 = off); default: 48 MB
// (within the device's window and persisting limits) whenever the relabelled
// twin runs.
struct L2Persist {
  tg_ctx* ctx = nullptr;
  size_t bytes = 0;
  L2Persist(tg_ctx* c, bool twin, uint64_t n) : ctx(c) {
    long want = -1;
    if (const char* e = std::getenv("TIERGRAPH_PR_PERSIST_MB")) want = std::atol(e);
    if (want == 0 || (want < 0 && !twin)) return;
    int maxwin = 0, maxpers = 0;
    cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device);
    cudaDeviceGetAttribute(&maxpers, cudaDevAttrMaxPersistingL2CacheSize, ctx->device);
    size_t b = std::min<size_t>(static_cast<size_t>(maxwin), static_cast<size_t>(maxpers));
    // default 48 MB: the hottest 6M norm values (~88 % of the C3 gathers);
    // 48 MB measured better than the device maximum (10.80 vs 10.99 ms per
    // C3 step, profiles/r02i), which leaves too little L2 for the rest
    if (want < 0) want = kPersistDefaultMB;
    b = std::min<size_t>(b, static_cast<size_t>(want) << 20);
    b = std::min<size_t>(b, 8 * n);
    if (b == 0) return;
    TGB_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, b));
    if (!ctx->aux) {  // the side streams of K3's class A
      ctx->fork();
      ctx->join();
    }
    bytes = b;
  }
  void window(const void* base) {
    if (!bytes) return;
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    v.accessPolicyWindow.num_bytes = bytes;
    v.accessPolicyWindow.hitRatio = 1.0f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    for (cudaStream_t s : {ctx->stream, ctx->aux, ctx->aux2, ctx->aux3})
      TGB_CUDA(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
  }
  ~L2Persist() {
    if (!bytes) return;
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.num_bytes = 0;
    for (cudaStream_t s : {ctx->stream, ctx->aux, ctx->aux2, ctx->aux3})
      cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaCtxResetPersistingL2Cache();  // the run's end synchronised the stream (DevOut::finish)
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
  }
};

void run_pagerank(tg_ctx* ctx, const tg_graph* g, uint32_t iterations, double damp,
                  const uint64_t* tid, uint64_t ntid, bool weighted, double* out,
                  double* phase_ms = nullptr) {
  check_config(iterations, damp);
  if (weighted && ntid == 0)
    domain_error(
        "weighted reverse pagerank needs a non-empty train id set; "
        "use reverse_pagerank when no nodes are labeled");  // scoring.cpp:89-91
  const uint64_t n = g ? g->n : 0;
  if (n == 0) return;
  if (!whole_graph(g))
    domain_error("pagerank: this graph holds only rows [" + std::to_string(g->rb) + ", " +
                 std::to_string(g->re) + "); run the partitioned entry points");
  DeviceGuard dg(ctx->device);
  const uint64_t* tid_dev = weighted ? dev_in(ctx, tid, ntid, kStageIn0) : nullptr;
  // the relabelled twin when enabled (bit-identical results; scores are
  // written back to the original ids by the last step's epilogue)
  const tg_graph* tw = relabel_twin(ctx, g);
  const tg_graph* run = tw ? tw : g;
  uint32_t* deg = run->indeg;  // cached with the device graph
  double* na = ctx->scratch_t<double>(kScratchB, n);
  double* nb = ctx->scratch_t<double>(kScratchC, n);
  DevOut<double> o(ctx, out, n, kStageOut0);
  auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 1);
  if (weighted) TGB_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
  // phase_ms (optional, [iterations + 1]): device time of the prepare and of
  // every step, CUDA events on the stream
  std::vector<cudaEvent_t> ev;
  if (phase_ms) {
    ev.resize(iterations + 2);
    for (auto& x : ev) TGB_CUDA(cudaEventCreate(&x));
    TGB_CUDA(cudaEventRecord(ev[0], ctx->stream));
  }
  pagerank_prepare(ctx, run, tid_dev, ntid, deg, na, bad, tw ? g->new_of : nullptr);
  if (phase_ms) TGB_CUDA(cudaEventRecord(ev[1], ctx->stream));
  L2Persist persist(ctx, tw != nullptr, n);
  for (uint32_t it = 0; it < iterations; ++it) {
    const bool last = it + 1 == iterations;
    persist.window(na);
    // steps 3.. (it >= 2) find both buffers already holding the empty rows' norm
    pagerank_step(ctx, run, deg, damp, na, nb, o.dev(), 0, n, last ? 1 : 0, 0, nullptr, nullptr,
                  nullptr, tw && it >= 2 ? 1 : 0, tw ? 1 : 0);
    if (last && tw) {  // scores by label (in nb) -> the graph's ids
      score_gather_kernel<<<grid_for(n, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
          nb, g->new_of, n, o.dev());
      TGB_LAUNCHED();
    }
    if (phase_ms) TGB_CUDA(cudaEventRecord(ev[it + 2], ctx->stream));
    std::swap(na, nb);
  }
  if (phase_ms) {
    TGB_CUDA(cudaEventSynchronize(ev.back()));
    for (uint32_t i = 0; i <= iterations; ++i) {
      float ms = 0;
      TGB_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      phase_ms[i] = ms;
    }
    for (auto& x : ev) cudaEventDestroy(x);
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

namespace tgb {
void graph_from_device(tg_ctx* ctx, const uint64_t* doff, uint32_t* tgt, uint64_t n, uint64_t e,
                       tg_graph** out) {
  auto* g = new tg_graph;
  g->ctx = ctx;
  g->n = n;
  g->e = e;
  g->rb = 0;
  g->re = n;
  g->tgt = tgt;  // owned from here on
  try {
    TGB_CUDA(tgb::dev_malloc(&g->off, sizeof(uint32_t) * (n + 1)));
    auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 2);
    TGB_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), ctx->stream));
    narrow_offsets_kernel<<<grid_for(n + 1, 256), 256, 0, ctx->stream>>>(doff, g->off, n, e, bad);
    TGB_LAUNCHED();
    unsigned long long hb;
    TGB_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (hb != ~0ull)
      format_error("csr: offsets invalid at index " + std::to_string(hb) +
                   " (need offsets[0]==0, monotone, offsets[num_nodes]==num_edges)");
    if (n) schedule(ctx, g, 0, n);  // K3 schedule of the whole graph
    TGB_CUDA(tgb::dev_malloc(&g->indeg, sizeof(uint32_t) * std::max<uint64_t>(n, 1)));
    compute_indeg(ctx, g, g->indeg);
    ctx->sync();
  } catch (...) {
    tg_graph_destroy(g);
    throw;
  }
  *out = g;
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
    uint32_t* tgt = nullptr;
    TGB_CUDA(tgb::dev_malloc(&tgt, sizeof(uint32_t) * std::max<uint64_t>(e, 1) + 16));  // +16: K3 reads 16 B target groups
    try {
      auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 2);
      TGB_CUDA(cudaMemsetAsync(bad + 1, 0xff, sizeof(unsigned long long), ctx->stream));
      // targets: straight from device memory, or in 32M-entry chunks from the host
      const bool tdev = is_device_ptr(targets);
      const bool tpinned = !tdev && is_pinned_host(targets);
      const uint64_t chunk = tdev ? std::max<uint64_t>(e, 1) : (32ull << 20);
      uint64_t host_bad = ~0ull;  // first out-of-range target seen by host-side narrowing
      static const bool host_narrow = [] {  // TIERGRAPH_UPLOAD_NARROW=0: u64 over PCIe (A/B)
        const char* v = std::getenv("TIERGRAPH_UPLOAD_NARROW");
        return !(v && v[0] == '0');
      }();
      for (uint64_t base = 0; base < e; base += chunk) {
        const uint64_t cnt = std::min(chunk, e - base);
        const uint64_t* src = targets + base;
        if (!tdev && !tpinned && cnt * sizeof(uint64_t) >= kPipeMin && host_narrow) {
          // large pageable targets: narrowed to u32 by the host cores on their
          // way into the pinned pipeline (half the PCIe bytes, no u64 staging)
          const uint64_t f = copy_h2d_narrow(ctx, tgt + base, src, cnt, n);
          if (host_bad == ~0ull && f != ~0ull) host_bad = base + f;
          continue;
        }
        if (!tdev) {
          // pinned, small (or TIERGRAPH_UPLOAD_NARROW=0): DMA the u64 values,
          // narrow on the device; two staging slots, so chunk k+1 crosses
          // PCIe while chunk k narrows
          auto* st = ctx->scratch_t<uint64_t>((base / chunk) & 1 ? kStageIn2 : kStageIn1, cnt);
          if (cnt * sizeof(uint64_t) >= kPipeMin && !tpinned)
            copy_h2d(ctx, st, src, cnt * sizeof(uint64_t), /*sync_end=*/false);
          else
            TGB_CUDA(cudaMemcpyAsync(st, src, cnt * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                     ctx->stream));
          src = st;
        }
        narrow_targets_kernel<<<grid_for(cnt, 256), 256, 0, ctx->stream>>>(src, tgt + base, cnt,
                                                                           base, n, bad + 1);
        TGB_LAUNCHED();
      }
      unsigned long long hb;
      TGB_CUDA(cudaMemcpyAsync(&hb, bad + 1, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      hb = std::min<unsigned long long>(hb, host_bad);
      if (hb != ~0ull) format_error("csr: target out of range at edge " + std::to_string(hb));
    } catch (...) {
      cudaFree(tgt);
      throw;
    }
    const uint64_t* doff = dev_in(ctx, offsets, n + 1, kStageIn0);
    graph_from_device(ctx, doff, tgt, n, e, out);
  });
}

int tg_pagerank_relabel_info(tg_ctx* ctx, const tg_graph* g, int* relabelled, double* build_ms) {
  return guard([&] {
    DeviceGuard dg(ctx->device);
    const tg_graph* tw = g->n ? relabel_twin(ctx, g) : nullptr;
    if (relabelled) *relabelled = tw ? 1 : 0;
    if (build_ms) *build_ms = tw ? g->twin_ms : 0.0;
  });
}

// A row-block graph: rows [row_begin, row_end) of the CSR only (SURVEY §8e,
// the shard of one rank of a partitioned PageRank). Offsets are the whole
// graph's (n+1, host or device u64); targets the whole array (host or
// device), of which only this block's edges are read and uploaded.
int tg_graph_create_rows(tg_ctx* ctx, const uint64_t* offsets, const uint64_t* targets,
                         uint64_t n, uint64_t e, uint64_t row_begin, uint64_t row_end,
                         tg_graph** out) {
  return guard([&] {
    if (!ctx || !out) domain_error("tg_graph_create_rows: null argument");
    if (n >= 0xffffffffull || e >= 0xffffffffull)
      domain_error("tg_graph_create_rows: n and e must be < 2^32 for the u32 device layout");
    if (row_begin > row_end || row_end > n)
      domain_error("tg_graph_create_rows: bad row range [" + std::to_string(row_begin) + ", " +
                   std::to_string(row_end) + ") of " + std::to_string(n) + " rows");
    DeviceGuard dg(ctx->device);
    const uint64_t m = row_end - row_begin;
    // this block's offsets (m + 1 values) and its edge range
    std::vector<uint64_t> ho(m + 1);
    if (is_device_ptr(offsets)) {
      TGB_CUDA(cudaMemcpy(ho.data(), offsets + row_begin, 8 * (m + 1), cudaMemcpyDeviceToHost));
    } else {
      std::memcpy(ho.data(), offsets + row_begin, 8 * (m + 1));
    }
    const uint64_t e0 = ho[0], e1 = ho[m];
    for (uint64_t i = 0; i <= m; ++i)
      if (ho[i] > e || (i && ho[i] < ho[i - 1]))
        format_error("csr: offsets invalid at index " + std::to_string(row_begin + i) +
                     " (need offsets[0]==0, monotone, offsets[num_nodes]==num_edges)");
    if ((row_begin == 0 && e0 != 0) || (row_end == n && e1 != e))
      format_error("csr: offsets invalid at index " + std::to_string(row_begin == 0 && e0 ? 0 : n) +
                   " (need offsets[0]==0, monotone, offsets[num_nodes]==num_edges)");
    auto* g = new tg_graph;
    g->ctx = ctx;
    g->n = n;
    g->e = e1 - e0;
    g->rb = row_begin;
    g->re = row_end;
    try {
      std::vector<uint32_t> o32(m + 1);
      for (uint64_t i = 0; i <= m; ++i) o32[i] = static_cast<uint32_t>(ho[i] - e0);
      TGB_CUDA(tgb::dev_malloc(&g->off_alloc, 4 * (m + 1)));
      TGB_CUDA(cudaMemcpy(g->off_alloc, o32.data(), 4 * (m + 1), cudaMemcpyHostToDevice));
      g->off = g->off_alloc - row_begin;  // off[r] for r in [row_begin, row_end]
      TGB_CUDA(tgb::dev_malloc(&g->tgt, 4 * std::max<uint64_t>(g->e, 1) + 16));  // +16: K3 reads 16 B target groups
      auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 2);
      TGB_CUDA(cudaMemsetAsync(bad + 1, 0xff, 8, ctx->stream));
      const bool tdev = is_device_ptr(targets);
      const bool tpinned = !tdev && is_pinned_host(targets);
      const uint64_t chunk = tdev ? std::max<uint64_t>(g->e, 1) : (32ull << 20);
      for (uint64_t base = 0; base < g->e; base += chunk) {
        const uint64_t cnt = std::min(chunk, g->e - base);
        const uint64_t* src = targets + e0 + base;
        if (!tdev) {
          auto* st = ctx->scratch_t<uint64_t>(kStageIn1, cnt);
          TGB_CUDA(cudaMemcpyAsync(st, src, cnt * 8, cudaMemcpyHostToDevice, ctx->stream));
          src = st;
        }
        narrow_targets_kernel<<<grid_for(cnt, 256), 256, 0, ctx->stream>>>(src, g->tgt + base, cnt,
                                                                           e0 + base, n, bad + 1);
        TGB_LAUNCHED();
      }
      unsigned long long hb;
      TGB_CUDA(cudaMemcpyAsync(&hb, bad + 1, 8, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      if (hb != ~0ull) format_error("csr: target out of range at edge " + std::to_string(hb));
      if (m) schedule(ctx, g, row_begin, row_end);
      TGB_CUDA(tgb::dev_malloc(&g->indeg, 4 * std::max<uint64_t>(n, 1)));
      compute_indeg(ctx, g, g->indeg);  // partial: this block's edges only
      ctx->sync();
    } catch (...) {
      tg_graph_destroy(g);
      throw;
    }
    *out = g;
  });
}

int tg_in_degrees_u32_async(tg_ctx* ctx, const tg_graph* g, uint32_t* out_dev) {
  return guard([&] {
    if (!g->n) return;
    DeviceGuard dg(ctx->device);
    TGB_CUDA(cudaMemcpyAsync(out_dev, g->indeg, 4 * g->n, cudaMemcpyDeviceToDevice, ctx->stream));
  });
}

int tg_pagerank_init_async(tg_ctx* ctx, uint64_t n, const uint64_t* tid_dev, uint64_t ntid,
                           const uint32_t* indeg_dev, double* norm0_dev) {
  return guard([&] {
    if (tid_dev && ntid == 0) domain_error("weighted reverse pagerank needs a non-empty train id set");
    if (!n) return;
    DeviceGuard dg(ctx->device);
    auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 1);
    if (tid_dev) TGB_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
    pagerank_init(ctx, n, tid_dev, ntid, indeg_dev, norm0_dev, bad);
    if (!tid_dev) return;
    unsigned long long hb = ~0ull;
    TGB_CUDA(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (hb != ~0ull) {
      uint64_t id = 0;
      TGB_CUDA(cudaMemcpy(&id, tid_dev + hb, sizeof(id), cudaMemcpyDeviceToHost));
      domain_error("train id " + std::to_string(id) + " out of range");  // scoring.cpp:98
    }
  });
}

int tg_measure_gather_floor_us(tg_ctx* ctx, const tg_graph* g, int reps, double* us) {
  return guard([&] {
    DeviceGuard dg(ctx->device);
    // K3's labelling (the twin when enabled); reps < 0: g's own labelling
    if (reps >= 0)
      if (const tg_graph* tw = g->n ? relabel_twin(ctx, g) : nullptr) g = tw;
    reps = std::abs(reps);
    double* x = ctx->scratch_t<double>(kScratchA, std::max<uint64_t>(g->n, 1) + 1);
    TGB_CUDA(cudaMemsetAsync(x, 0, 8 * (g->n + 1), ctx->stream));
    cudaEvent_t a, b;
    TGB_CUDA(cudaEventCreate(&a));
    TGB_CUDA(cudaEventCreate(&b));
    float best = 1e30f;
    for (int r = 0; r <= std::max(reps, 1); ++r) {
      TGB_CUDA(cudaEventRecord(a, ctx->stream));
      gather_floor_kernel<<<ctx->num_sms * 16, 256, 0, ctx->stream>>>(g->tgt, g->e, x, x + g->n);
      TGB_LAUNCHED();
      TGB_CUDA(cudaEventRecord(b, ctx->stream));
      TGB_CUDA(cudaEventSynchronize(b));
      float ms = 0;
      TGB_CUDA(cudaEventElapsedTime(&ms, a, b));
      if (r && ms < best) best = ms;  // first run warms
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *us = best * 1e3;
  });
}

int tg_graph_destroy(tg_graph* g) {
  if (!g) return TG_OK;
  tg_graph_destroy(g->twin);
  cudaFree(g->old_of);
  cudaFree(g->new_of);
  cudaFree(g->row_label);
  cudaFree(g->row_orig);
  cudaFree(g->deg_rows);
  cudaFree(g->off_alloc ? g->off_alloc : g->off);
  cudaFree(g->tgt);
  for (auto& sc : g->scheds)
    if (sc.order) cudaFree(sc.order);
  cudaFree(g->indeg);
  delete g;
  return TG_OK;
}

uint64_t tg_graph_num_nodes(const tg_graph* g) { return g ? g->n : 0; }
uint64_t tg_graph_num_edges(const tg_graph* g) { return g ? g->e : 0; }
// whole graphs only (a row block's arrays are not indexable by node id)
const uint32_t* tg_graph_offsets32(const tg_graph* g) {
  return g && whole_graph(g) ? g->off : nullptr;
}
const uint32_t* tg_graph_targets32(const tg_graph* g) {
  return g && whole_graph(g) ? g->tgt : nullptr;
}
int tg_graph_row_range(const tg_graph* g, uint64_t* row_begin, uint64_t* row_end) {
  return guard([&] {
    if (!g) domain_error("tg_graph_row_range: null graph");
    if (row_begin) *row_begin = g->rb;
    if (row_end) *row_end = g->re;
  });
}

int tg_degree_score(tg_ctx* ctx, const tg_graph* g, double* out) {
  return guard([&] {
    if (!g->n) return;
    if (!whole_graph(g)) domain_error("degree_score: needs a whole graph, not a row block");
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

int tg_weighted_reverse_pagerank_timed(tg_ctx* ctx, const tg_graph* g, uint32_t iterations,
                                       double damp, const uint64_t* tid, uint64_t ntid,
                                       double* out, double* phase_ms) {
  return guard([&] { run_pagerank(ctx, g, iterations, damp, tid, ntid, true, out, phase_ms); });
}

int tg_pagerank_prepare_async(tg_ctx* ctx, const tg_graph* g, const uint64_t* tid_dev,
                              uint64_t ntid, uint32_t* indeg_dev, double* norm0_dev) {
  return guard([&] {
    if (tid_dev && ntid == 0) domain_error("weighted reverse pagerank needs a non-empty train id set");
    if (!g->n) return;
    DeviceGuard dg(ctx->device);
    // out-of-range train ids are a DomainError as in the reference
    // (scoring.cpp:98): the one 8 B read-back of the first offending index is
    // this call's only synchronisation
    auto* bad = ctx->scratch_t<unsigned long long>(kSmall, 1);
    if (tid_dev) TGB_CUDA(cudaMemsetAsync(bad, 0xff, 8, ctx->stream));
    pagerank_prepare(ctx, g, tid_dev, ntid, indeg_dev, norm0_dev, bad);
    if (!tid_dev) return;
    unsigned long long hb = ~0ull;
    TGB_CUDA(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (hb != ~0ull) {
      uint64_t id = 0;
      TGB_CUDA(cudaMemcpy(&id, tid_dev + hb, sizeof(id), cudaMemcpyDeviceToHost));
      domain_error("train id " + std::to_string(id) + " out of range");  // scoring.cpp:98
    }
  });
}

int tg_pagerank_step_peers_async(tg_ctx* ctx, const tg_graph* g, const uint32_t* indeg_dev,
                                 double damp, const double* norm_in_dev, double* norm_out_dev,
                                 double* score_out_dev, uint64_t row_begin, uint64_t row_end,
                                 int last, double* const* peer_norm_out,
                                 double* const* peer_score_out, uint32_t n_peers) {
  return guard([&] {
    if (row_end > g->n || row_begin > row_end) domain_error("pagerank step: bad row range");
    if (n_peers >= TG_MAX_DEVICES) domain_error("pagerank step: too many peers");
    DeviceGuard dg(ctx->device);
    pagerank_step(ctx, g, indeg_dev, damp, norm_in_dev, norm_out_dev, score_out_dev, row_begin,
                  row_end, last, n_peers, peer_norm_out, peer_score_out);
  });
}

int tg_peer_barrier_async(tg_ctx* ctx, uint32_t* local_flag, uint32_t* const* peer_flags,
                          uint32_t n_peers, uint32_t target, uint32_t* err_dev) {
  return guard([&] {
    if (n_peers >= TG_MAX_DEVICES) domain_error("peer barrier: too many peers");
    DeviceGuard dg(ctx->device);
    PeerFlags pf{};
    for (uint32_t p = 0; p < n_peers; ++p) pf.peer[p] = peer_flags[p];
    peer_barrier_kernel<<<1, 32, 0, ctx->stream>>>(local_flag, pf, n_peers, target, err_dev);
    TGB_LAUNCHED();
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
