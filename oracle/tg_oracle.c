/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the tiergraph hot path.
 *
 * A plain-C restatement of the reference algorithms on the data-tiering hot
 * path (reference = /root/reference/proj, C++20 + OpenMP). Each function cites
 * the reference file:line it follows. It is pinned against the reference
 * itself (oracle/_ref/libtgref.so, built from the unmodified sources by
 * oracle/Makefile) and against the reference tests' known answers by
 * tests/test_oracle.py.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker. The product (libtiergraph_b200)
 * never links or calls it.
 *
 * Conventions: return 0 on success, 2 on a reference DomainError
 * (tools/tiergraph_cli.cpp:589-601 exit-code mapping). u64 everywhere, like
 * types.hpp:9-10. Built with -ffp-contract=off so no FMA can appear.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;

/* ------------------------------------------------------------------ rng */

/* rng.hpp:13-18 splitmix64 finalizer */
u64 tgo_mix64(u64 x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* rng.hpp:23-28 derive_stream_key */
u64 tgo_derive_stream_key(u64 seed, const u64* coords, uint32_t n) {
  u64 h = tgo_mix64(seed ^ 0x6A09E667F3BCC908ull);
  for (uint32_t i = 0; i < n; ++i) h = tgo_mix64(h ^ tgo_mix64(coords[i]));
  return h;
}

/* rng.hpp:36 next_u64 : splitmix64 of an incrementing counter */
static inline u64 rng_next(u64* state) { return tgo_mix64((*state)++); }

/* rng.hpp:39-52 next_below : Lemire multiply-shift with rejection */
static u64 rng_below(u64* state, u64 bound) {
  u64 x = rng_next(state);
  unsigned __int128 m = (unsigned __int128)x * bound;
  u64 lo = (u64)m;
  if (lo < bound) {
    const u64 threshold = (0 - bound) % bound;
    while (lo < threshold) {
      x = rng_next(state);
      m = (unsigned __int128)x * bound;
      lo = (u64)m;
    }
  }
  return (u64)(m >> 64);
}
u64 tgo_rng_below(u64* state, u64 bound) { return rng_below(state, bound); }

/* rng.cpp:8-40 Floyd k-subset, insertion order. The reference switches from a
 * linear scan (k <= 64) to a hash set; both test membership in the set of
 * values already emitted, so one membership structure suffices here. */
static int contains_linear(const u64* a, u64 n, u64 v) {
  for (u64 i = 0; i < n; ++i)
    if (a[i] == v) return 1;
  return 0;
}
typedef struct {
  u64* keys;
  u64 cap;
} hset;
static int hset_insert(hset* s, u64 v) { /* returns 1 if newly inserted */
  u64 h = tgo_mix64(v) & (s->cap - 1);
  while (s->keys[h] != ~0ull) {
    if (s->keys[h] == v) return 0;
    h = (h + 1) & (s->cap - 1);
  }
  s->keys[h] = v;
  return 1;
}
/* out must hold min(k, population) entries; returns count */
u64 tgo_sample_index_subset(u64* state, u64 population, u64 k, u64* out) {
  if (k >= population) {
    for (u64 i = 0; i < population; ++i) out[i] = i;
    return population;
  }
  u64 n = 0;
  if (k <= 64) {
    for (u64 j = population - k; j < population; ++j) {
      const u64 t = rng_below(state, j + 1);
      out[n++] = contains_linear(out, n, t) ? j : t;
    }
  } else {
    hset s;
    s.cap = 1;
    while (s.cap < 4 * k) s.cap <<= 1;
    s.keys = (u64*)malloc(sizeof(u64) * s.cap);
    memset(s.keys, 0xff, sizeof(u64) * s.cap);
    for (u64 j = population - k; j < population; ++j) {
      const u64 t = rng_below(state, j + 1);
      if (hset_insert(&s, t)) {
        out[n++] = t;
      } else {
        hset_insert(&s, j);
        out[n++] = j;
      }
    }
    free(s.keys);
  }
  return n;
}

/* rng.hpp:67-73 Fisher-Yates */
void tgo_shuffle(u64* state, u64* items, u64 n) {
  for (u64 i = n; i > 1; --i) {
    const u64 j = rng_below(state, i);
    const u64 t = items[i - 1];
    items[i - 1] = items[j];
    items[j] = t;
  }
}

/* -------------------------------------------------------------- graph core */

static int cmp_u64(const void* a, const void* b) {
  const u64 x = *(const u64*)a, y = *(const u64*)b;
  return (x > y) - (x < y);
}

/* csr_graph.cpp:89-93 in_degrees */
void tgo_in_degrees(const u64* offsets, const u64* targets, u64 n, u64* deg) {
  memset(deg, 0, sizeof(u64) * n);
  const u64 e = offsets[n];
  for (u64 i = 0; i < e; ++i) ++deg[targets[i]];
}

/* csr_graph.cpp:67-80 transpose ; out_offsets n+1, out_targets e */
void tgo_transpose(const u64* offsets, const u64* targets, u64 n, u64* t_off, u64* t_tgt) {
  memset(t_off, 0, sizeof(u64) * (n + 1));
  const u64 e = offsets[n];
  for (u64 i = 0; i < e; ++i) ++t_off[targets[i] + 1];
  for (u64 u = 0; u < n; ++u) t_off[u + 1] += t_off[u];
  u64* cursor = (u64*)malloc(sizeof(u64) * (n ? n : 1));
  memcpy(cursor, t_off, sizeof(u64) * n);
  for (u64 u = 0; u < n; ++u)
    for (u64 k = offsets[u]; k < offsets[u + 1]; ++k) t_tgt[cursor[targets[k]]++] = u;
  free(cursor);
}

/* csr_graph.cpp:36-65 from_edge_list: rows sorted ascending, duplicates dropped,
 * self-loops kept. out_offsets n+1; *out_targets malloc'ed; returns 2 when an id
 * is out of range. */
int tgo_from_edge_list(u64 n, const u64* src, const u64* dst, u64 m, u64* out_offsets,
                       u64** out_targets, u64* out_e) {
  for (u64 i = 0; i < m; ++i)
    if (src[i] >= n || dst[i] >= n) return 2;
  u64* raw = (u64*)calloc(n + 1, sizeof(u64));
  for (u64 i = 0; i < m; ++i) ++raw[src[i] + 1];
  for (u64 u = 0; u < n; ++u) raw[u + 1] += raw[u];
  u64* flat = (u64*)malloc(sizeof(u64) * (m ? m : 1));
  u64* cursor = (u64*)malloc(sizeof(u64) * (n ? n : 1));
  memcpy(cursor, raw, sizeof(u64) * n);
  for (u64 i = 0; i < m; ++i) flat[cursor[src[i]]++] = dst[i];
  u64* tg = (u64*)malloc(sizeof(u64) * (m ? m : 1));
  u64 e = 0;
  out_offsets[0] = 0;
  for (u64 u = 0; u < n; ++u) {
    qsort(flat + raw[u], raw[u + 1] - raw[u], sizeof(u64), cmp_u64);
    for (u64 i = raw[u]; i < raw[u + 1]; ++i)
      if (i == raw[u] || flat[i] != flat[i - 1]) tg[e++] = flat[i];
    out_offsets[u + 1] = e;
  }
  free(raw);
  free(flat);
  free(cursor);
  *out_targets = tg;
  *out_e = e;
  return 0;
}

/* feature_matrix.cpp:16-28 make_test_features: f32 value(r,c) = float(mix64(r)>>40) + c */
void tgo_make_test_features(u64 rows, u64 dim, float* out) {
  for (u64 r = 0; r < rows; ++r) {
    const float base = (float)(tgo_mix64(r) >> 40);
    for (u64 c = 0; c < dim; ++c) out[r * dim + c] = base + (float)c;
  }
}

/* ----------------------------------------------------------------- scoring */

/* scoring.cpp:22-31 draw_random_train_ids ; out has `count` sorted ids */
int tgo_draw_random_train_ids(u64 num_nodes, u64 count, u64 seed, u64* out) {
  if (count < 1 || count > num_nodes) return 2;
  const u64 tag = 0x6C61ull;
  u64 st = tgo_derive_stream_key(seed, &tag, 1);
  tgo_sample_index_subset(&st, num_nodes, count, out);
  qsort(out, count, sizeof(u64), cmp_u64);
  return 0;
}

/* scoring.cpp:50-74 run_iterations + scoring.cpp:78-102 initialisation.
 * tid == NULL -> reverse_pagerank (scoring.cpp:78-84); else the weighted
 * variant with weight N/|tid| applied as score[id] *= weight (:94-100).
 * Row sums run left to right in storage order (:65-70); no FMA. */
int tgo_reverse_pagerank(const u64* offsets, const u64* targets, u64 n, const u64* tid,
                         u64 ntid, uint32_t iterations, double damp, double* out) {
  if (iterations < 1) return 2;                 /* :43-44 */
  if (!(damp > 0.0 && damp < 1.0)) return 2;    /* :45-46 */
  if (tid && ntid == 0) return 2;               /* :89-91 */
  if (n == 0) return 0;
  double* score = out;
  for (u64 i = 0; i < n; ++i) score[i] = 1.0 / (double)n;
  if (tid) {
    const double weight = (double)n / (double)ntid;
    for (u64 i = 0; i < ntid; ++i) {
      if (tid[i] >= n) return 2;
      score[tid[i]] *= weight;
    }
  }
  const double base = (1.0 - damp) / (double)n;
  u64* indeg = (u64*)malloc(sizeof(u64) * n);
  tgo_in_degrees(offsets, targets, n, indeg);
  double* normalized = (double*)malloc(sizeof(double) * n);
  for (uint32_t it = 0; it < iterations; ++it) {
#pragma omp parallel for schedule(static)
    for (long long j = 0; j < (long long)n; ++j)
      normalized[j] = score[j] / (double)(indeg[j] > 1 ? indeg[j] : 1);
#pragma omp parallel for schedule(dynamic, 4096)
    for (long long j = 0; j < (long long)n; ++j) {
      double pulled = 0.0;
      for (u64 k = offsets[j]; k < offsets[j + 1]; ++k) pulled += normalized[targets[k]];
      score[j] = base + damp * pulled; /* reads only `normalized`: in-place is Jacobi */
    }
  }
  free(indeg);
  free(normalized);
  return 0;
}

/* scoring.cpp:33-38 degree_score */
void tgo_degree_score(const u64* offsets, u64 n, double* out) {
  for (u64 u = 0; u < n; ++u) out[u] = (double)(offsets[u + 1] - offsets[u]);
}

static const double* g_sort_scores;
static int cmp_score_desc_id_asc(const void* a, const void* b) {
  const u64 x = *(const u64*)a, y = *(const u64*)b;
  const double sx = g_sort_scores[x], sy = g_sort_scores[y];
  if (sx != sy) return sx > sy ? -1 : 1; /* scoring.cpp:111 (-0.0 == +0.0) */
  return (x > y) - (x < y);              /* scoring.cpp:112 */
}

/* scoring.cpp:104-115 score_ordering */
int tgo_score_ordering(const double* scores, u64 n, u64* out) {
  for (u64 i = 0; i < n; ++i)
    if (!isfinite(scores[i]) || scores[i] < 0.0) return 2; /* :105-107 */
  for (u64 i = 0; i < n; ++i) out[i] = i;
  g_sort_scores = scores;
  qsort(out, n, sizeof(u64), cmp_score_desc_id_asc);
  return 0;
}

/* ----------------------------------------------------------------- reorder */

/* reorder.cpp:10-21 validate_permutation */
int tgo_validate_permutation(const u64* perm, u64 n) {
  unsigned char* seen = (unsigned char*)calloc(n ? n : 1, 1);
  for (u64 u = 0; u < n; ++u) {
    if (perm[u] >= n || seen[perm[u]]) {
      free(seen);
      return 2;
    }
    seen[perm[u]] = 1;
  }
  free(seen);
  return 0;
}

/* reorder.cpp:23-29 permutation_from_scores */
int tgo_permutation_from_scores(const double* scores, u64 n, u64* out) {
  u64* order = (u64*)malloc(sizeof(u64) * (n ? n : 1));
  const int rc = tgo_score_ordering(scores, n, order);
  if (rc == 0)
    for (u64 r = 0; r < n; ++r) out[order[r]] = r;
  free(order);
  return rc;
}

/* reorder.cpp:31-37 invert */
int tgo_invert(const u64* perm, u64 n, u64* out) {
  if (tgo_validate_permutation(perm, n)) return 2;
  for (u64 u = 0; u < n; ++u) out[perm[u]] = u;
  return 0;
}

/* reorder.cpp:68-95 sequential_reorder_oracle (== reorder_graph :39-66) */
int tgo_reorder_graph(const u64* offsets, const u64* targets, u64 n, const u64* perm,
                      u64* out_offsets, u64* out_targets) {
  if (tgo_validate_permutation(perm, n)) return 2;
  memset(out_offsets, 0, sizeof(u64) * (n + 1));
  for (u64 u = 0; u < n; ++u) out_offsets[perm[u] + 1] = offsets[u + 1] - offsets[u];
  for (u64 u = 0; u < n; ++u) out_offsets[u + 1] += out_offsets[u];
  for (u64 u = 0; u < n; ++u) {
    u64* dst = out_targets + out_offsets[perm[u]];
    for (u64 k = offsets[u]; k < offsets[u + 1]; ++k) dst[k - offsets[u]] = perm[targets[k]];
  }
  return 0;
}

/* reorder.cpp:97-117 reorder_features: new row perm[u] = old row u */
int tgo_reorder_features(const uint8_t* data, u64 rows, u64 row_bytes, const u64* perm,
                         uint8_t* out) {
  if (tgo_validate_permutation(perm, rows)) return 2;
  for (u64 u = 0; u < rows; ++u) memcpy(out + perm[u] * row_bytes, data + u * row_bytes, row_bytes);
  return 0;
}

/* ----------------------------------------------------------------- tiering */
/* layout6 = {num_rows, local_boundary, multi_boundary, num_devices, feature_dim,
 * elem_bytes} (tiering.hpp:16-25); report6 = {local_acc, peer_acc, host_acc,
 * local_bytes, peer_bytes, host_bytes} (tiering.hpp:51-58). */

/* tiering.cpp:10-18 validate_layout */
int tgo_validate_layout(const u64* l) {
  if (l[3] < 1) return 2;
  if (l[1] > l[2] || l[2] > l[0]) return 2;
  return 0;
}

/* tiering.cpp:48-65 resolve ; out3 = {tier(0 local,1 interleaved,2 cold), device, row} */
int tgo_resolve(const u64* l, u64 row, uint32_t dev, u64* out3) {
  if (row >= l[0]) return 2;
  if (dev >= l[3]) return 2;
  if (row < l[1]) {
    out3[0] = 0, out3[1] = 0, out3[2] = row;
  } else if (row < l[2]) {
    const u64 off = row - l[1];
    out3[0] = 1, out3[1] = off % l[3], out3[2] = off / l[3];
  } else {
    out3[0] = 2, out3[1] = 0, out3[2] = row - l[2];
  }
  return 0;
}

/* tiering.cpp:67-98 plan_layout (llround = round half away from zero) */
int tgo_plan_layout(u64 num_rows, double hot, double rep, uint32_t devices, u64 dim,
                    uint32_t elem_bytes, u64 budget, u64* out6) {
  if (!(rep >= 0.0 && rep <= hot && hot <= 1.0)) return 2;
  if (devices < 1) return 2;
  out6[0] = num_rows;
  out6[1] = (u64)llround(rep * (double)num_rows);
  out6[2] = (u64)llround(hot * (double)num_rows);
  out6[3] = devices;
  out6[4] = dim;
  out6[5] = elem_bytes;
  if (tgo_validate_layout(out6)) return 2;
  if (budget > 0) {
    const u64 inter = out6[2] - out6[1];
    const u64 per_dev_rows = out6[1] + (inter + devices - 1) / devices;
    if (per_dev_rows * (dim * elem_bytes) > budget) return 2;
  }
  return 0;
}

/* tiering.cpp:100-125 gather (accounting only). Accumulates into report6;
 * stops at the first invalid id leaving the prefix accounted, like the
 * reference's throwing loop. */
int tgo_gather(const u64* l, const u64* ids, u64 n, uint32_t dev, u64* r) {
  const u64 rb = l[4] * l[5];
  for (u64 i = 0; i < n; ++i) {
    u64 loc[3];
    if (tgo_resolve(l, ids[i], dev, loc)) return 2;
    if (loc[0] == 0 || (loc[0] == 1 && loc[1] == dev)) {
      r[0] += 1, r[3] += rb;
    } else if (loc[0] == 1) {
      r[1] += 1, r[4] += rb;
    } else {
      r[2] += 1, r[5] += rb;
    }
  }
  return 0;
}

/* tiering.cpp:127-162 simulate_trace */
int tgo_simulate_trace(const u64* counts, u64 n, const u64* l, u64* r) {
  if (tgo_validate_layout(l)) return 2;
  if (n != l[0]) return 2;
  u64 total = 0;
  for (u64 i = 0; i < n; ++i) total += counts[i];
  if (total == 0) return 2;
  memset(r, 0, sizeof(u64) * 6);
  const u64 D = l[3];
  for (u64 row = 0; row < n; ++row) {
    const u64 c = counts[row];
    if (!c) continue;
    if (row < l[1]) {
      r[0] += c;
    } else if (row < l[2]) {
      const u64 owner = (row - l[1]) % D;
      const u64 local = c / D + (owner < c % D ? 1 : 0); /* :148 */
      r[0] += local;
      r[1] += c - local;
    } else {
      r[2] += c;
    }
  }
  const u64 rb = l[4] * l[5];
  r[3] = r[0] * rb, r[4] = r[1] * rb, r[5] = r[2] * rb;
  return 0;
}

/* tiering.cpp:164-175 counts_in_row_order */
int tgo_counts_in_row_order(const u64* counts, u64 n, const u64* ordering, u64 m, u64* out) {
  if (m != n) return 2;
  for (u64 k = 0; k < m; ++k) {
    if (ordering[k] >= n) return 2;
    out[k] = counts[ordering[k]];
  }
  return 0;
}

/* tiering.cpp:177-202 hot_fraction_sweep */
int tgo_hot_fraction_sweep(const u64* counts, u64 n, const u64* ordering, const double* fr,
                           u64 nf, double replicated, uint32_t devices, u64 dim,
                           uint32_t elem_bytes, u64 budget, u64* out_layouts, u64* out_reports,
                           double* out_rep) {
  for (u64 i = 1; i < nf; ++i)
    if (fr[i] < fr[i - 1]) return 2;
  u64* rc = (u64*)malloc(sizeof(u64) * (n ? n : 1));
  int err = tgo_counts_in_row_order(counts, n, ordering, n, rc);
  for (u64 i = 0; !err && i < nf; ++i) {
    const double rep = replicated < fr[i] ? replicated : fr[i];
    out_rep[i] = rep;
    err = tgo_plan_layout(n, fr[i], rep, devices, dim, elem_bytes, budget, out_layouts + 6 * i);
    if (!err) err = tgo_simulate_trace(rc, n, out_layouts + 6 * i, out_reports + 6 * i);
  }
  free(rc);
  return err;
}

/* ---------------------------------------------------------------- sampling */

/* sampling.cpp:35-37 BatchRng::stream key {0x534D, epoch, batch, layer, node} */
static u64 batch_stream_key(u64 seed, u64 epoch, u64 batch, u64 layer, u64 node) {
  const u64 c[5] = {0x534Dull, epoch, batch, layer, node};
  return tgo_derive_stream_key(seed, c, 5);
}

static u64 sort_unique(u64* a, u64 n) {
  if (!n) return 0;
  qsort(a, n, sizeof(u64), cmp_u64);
  u64 m = 1;
  for (u64 i = 1; i < n; ++i)
    if (a[i] != a[m - 1]) a[m++] = a[i];
  return m;
}

/* sampling.cpp:56-90 build_minibatch over the transposed graph (gt) with
 * sampling.cpp:39-54 sample_in_neighbors. Returns a malloc'ed sorted unique id
 * list and its length; 2 on a bad argument (:59-62, sampling.cpp:18-25). */
/* Graph-structure tiering: the neighbour ids a sampler
 * reads per tier when row v of gt lives where resolve(v) puts it
 * (tiering.cpp:48-65; lay = {lb, mb, D}): min(deg(v), fanout) ids per
 * frontier node, counted local (v < lb, or interleaved on `dev`), peer or
 * host (v >= mb). Not in the reference (it only sizes pseudo-rows,
 * tiergraph_cli.cpp:389-406); the GPU sampler's counters are checked
 * against it. */
static void count_tier_reads(u64 v, u64 c, const u64* lay, uint32_t dev, u64* reads) {
  if (!reads) return;
  int t = 2;
  if (v < lay[0]) t = 0;
  else if (v < lay[1]) t = ((v - lay[0]) % lay[2]) == dev ? 0 : 1;
  reads[t] += c;
}

static int build_minibatch_impl(const u64* gt_off, const u64* gt_tgt, u64 n, const u64* seeds,
                                u64 nseeds, const uint32_t* fanouts, uint32_t nf, u64 rng_seed,
                                u64 epoch, u64 batch, u64** out, u64* out_n, const u64* lay,
                                uint32_t dev, u64* reads);

int tgo_build_minibatch(const u64* gt_off, const u64* gt_tgt, u64 n, const u64* seeds,
                        u64 nseeds, const uint32_t* fanouts, uint32_t nf, u64 rng_seed,
                        u64 epoch, u64 batch, u64** out, u64* out_n) {
  return build_minibatch_impl(gt_off, gt_tgt, n, seeds, nseeds, fanouts, nf, rng_seed, epoch,
                              batch, out, out_n, NULL, 0, NULL);
}

int tgo_build_minibatch_tier_reads(const u64* gt_off, const u64* gt_tgt, u64 n, const u64* seeds,
                                   u64 nseeds, const uint32_t* fanouts, uint32_t nf,
                                   u64 rng_seed, u64 epoch, u64 batch, const u64* lay,
                                   uint32_t dev, u64* reads) {
  u64* m = NULL;
  u64 nm = 0;
  reads[0] = reads[1] = reads[2] = 0;
  const int rc = build_minibatch_impl(gt_off, gt_tgt, n, seeds, nseeds, fanouts, nf, rng_seed,
                                      epoch, batch, &m, &nm, lay, dev, reads);
  free(m);
  return rc;
}

static int build_minibatch_impl(const u64* gt_off, const u64* gt_tgt, u64 n, const u64* seeds,
                                u64 nseeds, const uint32_t* fanouts, uint32_t nf, u64 rng_seed,
                                u64 epoch, u64 batch, u64** out, u64* out_n, const u64* lay,
                                uint32_t dev, u64* reads) {
  if (nf == 0 || nf > 5) return 2;
  for (uint32_t i = 0; i < nf; ++i)
    if (fanouts[i] < 1) return 2;
  if (nseeds == 0) return 2;
  for (u64 i = 0; i < nseeds; ++i)
    if (seeds[i] >= n) return 2;

  u64 cap = nseeds, fcap = nseeds;
  for (uint32_t l = 0; l < nf; ++l) fcap *= fanouts[l], cap += fcap;
  u64* members = (u64*)malloc(sizeof(u64) * cap);
  u64* frontier = (u64*)malloc(sizeof(u64) * (fcap > nseeds ? fcap : nseeds));
  u64* next = (u64*)malloc(sizeof(u64) * (fcap > nseeds ? fcap : nseeds));
  u64 picks[4096];
  memcpy(frontier, seeds, sizeof(u64) * nseeds);
  u64 nfr = sort_unique(frontier, nseeds);
  memcpy(members, frontier, sizeof(u64) * nfr);
  u64 nm = nfr;
  for (uint32_t layer = 0; layer < nf; ++layer) {
    u64 nn = 0;
    for (u64 i = 0; i < nfr; ++i) {
      const u64 v = frontier[i];
      const u64 b = gt_off[v], deg = gt_off[v + 1] - b;
      count_tier_reads(v, deg < fanouts[layer] ? deg : fanouts[layer], lay, dev, reads);
      if (deg <= fanouts[layer]) {
        for (u64 k = 0; k < deg; ++k) next[nn++] = gt_tgt[b + k];
      } else {
        u64 st = batch_stream_key(rng_seed, epoch, batch, layer, v);
        u64* pk = fanouts[layer] <= 4096 ? picks : (u64*)malloc(sizeof(u64) * fanouts[layer]);
        const u64 got = tgo_sample_index_subset(&st, deg, fanouts[layer], pk);
        for (u64 k = 0; k < got; ++k) next[nn++] = gt_tgt[b + pk[k]];
        if (pk != picks) free(pk);
      }
    }
    nn = sort_unique(next, nn);
    u64* t = frontier;
    frontier = next;
    next = t;
    nfr = nn;
    memcpy(members + nm, frontier, sizeof(u64) * nfr);
    nm += nfr;
    if (nfr == 0) break;
  }
  nm = sort_unique(members, nm);
  free(frontier);
  free(next);
  *out = members;
  *out_n = nm;
  return 0;
}

void tgo_free(void* p) { free(p); }
