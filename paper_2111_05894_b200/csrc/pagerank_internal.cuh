// The device graph (tg_graph) and the K1-K3 entry points shared by
// pagerank.cu (single device) and multigpu.cu (partitioned, several devices).
#pragma once
#include <cstdint>
#include <vector>

#include "internal.cuh"

struct tg_graph {
  tg_ctx* ctx = nullptr;
  uint64_t n = 0, e = 0;       // e: edges held (a row block's own edges)
  // Rows held: [rb, re). A whole graph holds [0, n); a ROW-BLOCK graph
  // (tg_graph_create_rows, one shard of a partitioned PageRank) holds only
  // its block: off is then a shifted view (off[r] valid for r in [rb, re],
  // rebased so off[rb] == 0) of off_alloc, tgt holds the block's edges, and
  // indeg counts only those edges (the partial K1 a multi-GPU run sums).
  uint64_t rb = 0, re = 0;
  uint32_t* off_alloc = nullptr;
  uint32_t* off = nullptr;     // n+1, u32
  uint32_t* tgt = nullptr;     // e, u32
  uint32_t* indeg = nullptr;   // in_degrees (csr_graph.cpp:89-93), built with the device graph
  // K3 schedules: rows of [rb, re) by length descending (ties by id), split
  // into the three row classes. [0, n) is built with the graph; row ranges
  // of a partitioned (multi-GPU) run are built on first use.
  struct Sched {
    uint64_t rb, re;
    uint32_t* order;
    uint32_t nA, nB;  // order[0,nA): len > kLenA; [nA,nB): kLenB < len <= kLenA
    uint32_t nLong;   // order[0,nLong): len > kHubLong (512-thread class-A CTAs)
    // relabelled twin only (storage order = schedule): rows [nE, re-rb) have
    // no edges; their step is a streaming epilogue, skipped once both norm
    // buffers hold its constant value. Otherwise nE = re - rb.
    uint64_t nE = ~0ull;
  };
  std::vector<Sched> scheds;
  // K3 relabelling ("K3 relabel"): a twin of this graph with node
  // ids renumbered by in-degree, descending (ties by id), built on the first
  // PageRank call when enabled. Row v of the twin is row old_of[v] of this
  // graph with every target w stored as new_of[w], in the SAME storage order,
  // so every row sum is the reference's chain over the same values (bit-exact)
  // while the gathered norm values of the most-referenced nodes share sectors
  // and stay L2-resident.
  //
  // The twin also STORES its rows in K3's schedule order (length descending,
  // ties by id), so its schedule is the identity and a warp's class-C rows
  // are contiguous in memory (coalesced target streaming). Its vectors are
  // indexed by label: row k writes norm[row_label[k]]; its in-degrees are
  // kept by label (indeg, for the init) and by storage row (deg_rows); the
  // last step writes the score of row k to out[row_orig[k]].
  tg_graph* twin = nullptr;
  uint32_t* old_of = nullptr;  // label -> this graph's id
  uint32_t* new_of = nullptr;  // this graph's id -> label
  bool twin_tried = false;
  float twin_ms = 0.0f;        // one-time build time (device, allocations excluded)
  // (twin only)
  uint32_t* row_label = nullptr;
  uint32_t* row_orig = nullptr;
  uint32_t* deg_rows = nullptr;
};

namespace tgb {
inline bool whole_graph(const tg_graph* g) { return g->rb == 0 && g->re == g->n; }
void compute_indeg(tg_ctx* ctx, const tg_graph* g, uint32_t* deg);
// K1 as partition + shared-memory histograms (indegree.cu); false = not applicable
bool compute_indeg_binned(tg_ctx* ctx, const uint32_t* tgt, uint64_t e, uint64_t n, uint32_t* deg);
const tg_graph::Sched& schedule(tg_ctx* ctx, const tg_graph* g, uint64_t rb, uint64_t re);
void check_config(uint32_t iterations, double damp);
// deg + norm0 (full length) from in-degrees `deg` (already final).
void pagerank_init(tg_ctx* ctx, uint64_t n, const uint64_t* tid_dev, uint64_t ntid,
                   const uint32_t* deg, double* norm0, unsigned long long* bad,
                   const uint32_t* relabel = nullptr);
void pagerank_step(tg_ctx* ctx, const tg_graph* g, const uint32_t* deg, double damp,
                   const double* nin, double* nout, double* sout, uint64_t rb, uint64_t re,
                   int last, uint32_t n_peers = 0, double* const* peer_norm = nullptr,
                   double* const* peer_score = nullptr, const uint32_t* score_index = nullptr,
                   int skip_empty = 0, int score_to_norm = 0);
}  // namespace tgb
