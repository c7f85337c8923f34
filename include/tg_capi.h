/*
 * tg_capi.h — the C-ABI drop-in boundary of the B200 tiergraph hot path.
 *
 * Plain pointers and sizes only (no torch, no STL). Every entry point names the
 * reference interface it replaces (reference = arXiv 2111.05894 `tiergraph`,
 * files under proj/include/tiergraph and proj/src). The C++ drop-in headers in
 * include/tiergraph/tiergraph.hpp is implemented on top of these calls, and the
 * Python host mirror (paper_2111_05894_b200/tiergraph.py) binds them with
 * ctypes; INTEGRATION.md shows the bindings.
 *
 * Pointer arguments marked "host|device" may be either: the library inspects
 * them (cudaPointerGetAttributes) and stages host memory through the context's
 * stream. All calls are stream-ordered on the context's stream; calls that
 * return results in host memory synchronise that stream before returning.
 * Calls with an `_async` suffix never synchronise and take device pointers.
 *
 * Errors: every int-returning call returns TG_OK or one of the codes below,
 * which mirror the reference CLI's exit codes for its exception classes
 * (tools/tiergraph_cli.cpp:589-601; types.hpp:13-29). The thread-local
 * message of the last failure is available from tg_last_error().
 */
#ifndef TG_CAPI_H_
#define TG_CAPI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TG_OK 0
#define TG_ERR_DOMAIN 2   /* reference DomainError (types.hpp:26-29) */
#define TG_ERR_FORMAT 3   /* reference FormatError (types.hpp:20-23) */
#define TG_ERR_IO 4       /* reference IoError     (types.hpp:13-16) */
#define TG_ERR_INTERNAL 5 /* CUDA / allocation failures (CLI exit 5)  */

#define TG_MAX_DEVICES 16

/* Message of the last failing call on this thread. */
const char* tg_last_error(void);
/* Library / kernel build identification, e.g. "tiergraph_b200 sm_100a". */
const char* tg_version(void);

/* ------------------------------------------------------------------ POD views
 * Layout-identical to the reference structs so a C++ caller can pass them
 * straight through. */

/* tiering.hpp:16-25 TierLayout */
typedef struct tg_layout {
  uint64_t num_rows;
  uint64_t local_boundary;
  uint64_t multi_boundary;
  uint32_t num_devices;
  uint64_t feature_dim;
  uint32_t elem_bytes;
} tg_layout;

/* tiering.hpp:51-58 TrafficReport (counters only) */
typedef struct tg_report {
  uint64_t local_accesses;
  uint64_t peer_accesses;
  uint64_t host_accesses;
  uint64_t local_bytes;
  uint64_t peer_bytes;
  uint64_t host_bytes;
} tg_report;

/* tiering.hpp:29-37 Tier / Location */
#define TG_TIER_LOCAL_HOT 0
#define TG_TIER_INTERLEAVED 1
#define TG_TIER_COLD_HOST 2
typedef struct tg_location {
  uint8_t tier;
  uint32_t device;
  uint64_t row_within_tier;
} tg_location;

/* ---------------------------------------------------------------- context
 * One device + one CUDA stream + scratch memory. Mirrors the reference's
 * process-global worker count (parallel.hpp:5-9): the device is chosen per
 * context; tg_default_device() resolves TIERGRAPH_DEVICES like
 * TIERGRAPH_THREADS (parallel.cpp:13-19). */
typedef struct tg_ctx tg_ctx;
int tg_ctx_create(int device, tg_ctx** out);
/* Run on a caller-owned stream (e.g. torch.cuda.current_stream()). */
int tg_ctx_create_on_stream(int device, void* cuda_stream, tg_ctx** out);
int tg_ctx_destroy(tg_ctx* ctx);
/* Stream-ordered copy of `bytes` between any two UVA addresses (device, peer
 * or CUDA-IPC mapped, pinned host): the contiguous block push of a
 * partitioned PageRank exchange (copy engines over NVLink). */
int tg_memcpy_async(tg_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int tg_ctx_sync(tg_ctx* ctx);
/* Synchronises the context, frees its grow-only scratch (staging buffers and
 * sort temporaries) and returns the device pool's cached free memory to the
 * driver: for a caller about to make one very large allocation (no
 * reference counterpart; the reference holds no device memory). */
int tg_ctx_trim(tg_ctx* ctx);
void* tg_ctx_stream(tg_ctx* ctx);
int tg_ctx_device(tg_ctx* ctx);
/* First entry of TIERGRAPH_DEVICES ("0,1,..."), else 0. */
int tg_default_device(void);
/* Number of devices listed in TIERGRAPH_DEVICES (>=1), or the visible count. */
int tg_device_count(void);
/* The devices TIERGRAPH_DEVICES lists ("0,1,2"; entries may repeat: virtual
 * devices on one GPU), else {0}. Writes min(count, cap) ids; returns count.
 * The C++ drop-in partitions PageRank over them when there are several. */
int tg_device_list(int* out, int cap);
/* Launches of this library's kernels since process start (all contexts). */
uint64_t tg_kernel_launches(void);

/* ------------------------------------------------------------------ graph
 * Device copy of a reference CsrGraph (csr_graph.hpp:22-35): offsets
 * (n+1 x u64) and targets (e x u64), host|device. Stored narrowed to u32
 * (requires n, e < 2^32); targets are range-checked (TG_ERR_FORMAT, message
 * as validate_csr csr_graph.cpp:21-25). Also builds the row-group schedule
 * used by the SpMV. */
typedef struct tg_graph tg_graph;
int tg_graph_create(tg_ctx* ctx, const uint64_t* offsets, const uint64_t* targets, uint64_t n,
                    uint64_t e, tg_graph** out);
int tg_graph_destroy(tg_graph* g);
uint64_t tg_graph_num_nodes(const tg_graph* g);
uint64_t tg_graph_num_edges(const tg_graph* g);
/* Device pointers of the narrowed CSR (u32) — for peer kernels and tests. */
const uint32_t* tg_graph_offsets32(const tg_graph* g);
const uint32_t* tg_graph_targets32(const tg_graph* g);

/* --------------------------------------------------------------- scoring
 * scoring.hpp:32 degree_score -> out (n x f64, host|device) */
int tg_degree_score(tg_ctx* ctx, const tg_graph* g, double* out);
/* csr_graph.cpp:89-93 in_degrees -> out (n x u64, host|device) */
int tg_in_degrees(tg_ctx* ctx, const tg_graph* g, uint64_t* out);
/* scoring.hpp:40 reverse_pagerank (scoring.cpp:78-84). Bit-exact fp64. */
int tg_reverse_pagerank(tg_ctx* ctx, const tg_graph* g, uint32_t iterations, double damp,
                        double* out);
/* scoring.hpp:45-46 weighted_reverse_pagerank (scoring.cpp:86-102).
 * tid = TrainIdSet::ids (host|device), ntid >= 1 else TG_ERR_DOMAIN. */
int tg_weighted_reverse_pagerank(tg_ctx* ctx, const tg_graph* g, uint32_t iterations,
                                 double damp, const uint64_t* tid, uint64_t ntid, double* out);

/* The same, with phase_ms[0] = the device time of the prepare (K2) and
 * phase_ms[1 + i] = that of step i (K3), CUDA events on the context stream
 * (measurement entry point; phase_ms has iterations + 1 entries). */
int tg_weighted_reverse_pagerank_timed(tg_ctx* ctx, const tg_graph* g, uint32_t iterations,
                                       double damp, const uint64_t* tid, uint64_t ntid,
                                       double* out, double* phase_ms);

/* Row-partitioned iteration for multi-GPU: the caller owns the
 * exchange (NCCL all-gather of `norm`). norm_in/norm_out/score_out are device
 * vectors of length n; only rows [row_begin,row_end) are written.
 *   tg_pagerank_prepare: in-degrees (u32, device, length n) and the initial
 *     normalized vector for the weighted (tid!=NULL) or plain recurrence.
 *     A train id >= n is TG_ERR_DOMAIN "train id X out of range"
 *     (scoring.cpp:98); checking it synchronises the stream once.
 *   tg_pagerank_step: one Jacobi step over the rows; `last` writes scores
 *     instead of the next normalized vector. */
int tg_pagerank_prepare_async(tg_ctx* ctx, const tg_graph* g, const uint64_t* tid_dev,
                              uint64_t ntid, uint32_t* indeg_dev, double* norm0_dev);
int tg_pagerank_step_async(tg_ctx* ctx, const tg_graph* g, const uint32_t* indeg_dev,
                           double damp, const double* norm_in_dev, double* norm_out_dev,
                           double* score_out_dev, uint64_t row_begin, uint64_t row_end,
                           int last);

/* ----------------------------------------------- partitioned (multi-GPU) K1/K3
 * SURVEY §8e. Edge-balanced contiguous row blocks: bounds[0..parts] with
 * bounds[r] = the first row whose offset reaches ceil(r*E/parts) (host
 * offsets, n+1 values). */
int tg_row_blocks(const uint64_t* offsets, uint64_t n, uint32_t parts, uint64_t* bounds);
/* A ROW-BLOCK graph: rows [row_begin, row_end) only (one rank's shard).
 * offsets: the whole graph's n+1 (host|device); targets: the whole array
 * (host|device), of which only the block's edges are uploaded. Its in-degrees
 * count the block's edges only (the K1 shard; sum them over the ranks).
 * Valid with tg_pagerank_step_async over sub-ranges of the block,
 * tg_in_degrees_u32_async and tg_measure_gather_floor_us; whole-graph calls
 * (PageRank, degree_score, sampler, transpose) return TG_ERR_DOMAIN. */
int tg_graph_create_rows(tg_ctx* ctx, const uint64_t* offsets, const uint64_t* targets,
                         uint64_t n, uint64_t e, uint64_t row_begin, uint64_t row_end,
                         tg_graph** out);
int tg_graph_row_range(const tg_graph* g, uint64_t* row_begin, uint64_t* row_end);
/* In-degrees over the edges g holds (u32, device, length n), stream-ordered. */
int tg_in_degrees_u32_async(tg_ctx* ctx, const tg_graph* g, uint32_t* out_dev);
/* norm0 (device, length n) from FINAL in-degrees indeg_dev (e.g. the summed
 * shards); tid_dev NULL = unweighted. Train ids >= n: TG_ERR_DOMAIN (one
 * synchronisation). */
int tg_pagerank_init_async(tg_ctx* ctx, uint64_t n, const uint64_t* tid_dev, uint64_t ntid,
                           const uint32_t* indeg_dev, double* norm0_dev);

/* Partitioned PageRank over several devices of ONE process (what the C++
 * drop-in runs when TIERGRAPH_DEVICES lists several devices). Each device
 * holds one edge-balanced row block; K1 is sharded and summed over the devices
 * once; each K3 step pushes every device's block of the next vector to the
 * others as one contiguous peer copy per peer (copy engines over NVLink).
 * Bit-identical to one device for any device count. ctxs: distinct contexts
 * (devices may repeat: virtual devices on one GPU). */
typedef struct tg_mgraph tg_mgraph;
int tg_mgraph_create(tg_ctx* const* ctxs, uint32_t ndev, const uint64_t* offsets,
                     const uint64_t* targets, uint64_t n, uint64_t e, tg_mgraph** out);
int tg_mgraph_destroy(tg_mgraph* m);
/* bounds[ndev+1], edges[ndev] per block, indeg_ms = sharded K1 + reduction. */
int tg_mgraph_info(const tg_mgraph* m, uint64_t* bounds, uint64_t* edges, double* indeg_ms);
int tg_mgraph_in_degrees(tg_mgraph* m, uint64_t* out);
/* weighted != 0: scoring.cpp:86-102 with tid (host|device); else :78-84.
 * out: n f64 (host or device of the first context). */
int tg_mgraph_pagerank(tg_mgraph* m, uint32_t iterations, double damp, const uint64_t* tid,
                       uint64_t ntid, int weighted, double* out);

/* Fused exchange for a partitioned run: the step
 * also stores each of its rows into every peer's norm_out / score_out vector
 * (device pointers valid on this device: peer-mapped or CUDA-IPC), so no
 * all-gather follows. tg_peer_barrier_async then releases those stores, adds
 * 1 to each peer's arrival counter (peer_flags, u32) and waits on this
 * device until local_flag >= target; a wait over ~2 s sets *err_dev = 1 and
 * returns. With G ranks, target after step s (1-based) is s * (G - 1). */
int tg_pagerank_step_peers_async(tg_ctx* ctx, const tg_graph* g, const uint32_t* indeg_dev,
                                 double damp, const double* norm_in_dev, double* norm_out_dev,
                                 double* score_out_dev, uint64_t row_begin, uint64_t row_end,
                                 int last, double* const* peer_norm_out,
                                 double* const* peer_score_out, uint32_t n_peers);
int tg_peer_barrier_async(tg_ctx* ctx, uint32_t* local_flag, uint32_t* const* peer_flags,
                          uint32_t n_peers, uint32_t target, uint32_t* err_dev);

/* scoring.hpp:49 score_ordering (scoring.cpp:104-115): ids by descending
 * score, ties by ascending id. scores/out host|device. TG_ERR_DOMAIN names the
 * first non-finite or negative score. */
int tg_score_ordering(tg_ctx* ctx, const double* scores, uint64_t n, uint64_t* out_order);

/* ---------------------------------------------------------------- reorder
 * reorder.hpp:25 permutation_from_scores (reorder.cpp:23-29). out_new_id_of
 * (n x u64, host|device). out_order may be NULL or receives score_ordering. */
int tg_permutation_from_scores(tg_ctx* ctx, const double* scores, uint64_t n,
                               uint64_t* out_new_id_of, uint64_t* out_order);
/* reorder.hpp:21 validate_permutation (reorder.cpp:10-21) */
int tg_validate_permutation(tg_ctx* ctx, const uint64_t* perm, uint64_t n);
/* reorder.hpp:27 invert (reorder.cpp:31-37) */
int tg_invert(tg_ctx* ctx, const uint64_t* perm, uint64_t n, uint64_t* out);
/* reorder.hpp:40 reorder_features (reorder.cpp:97-117): new row perm[u] = old
 * row u. src/dst host|device, rows x row_bytes. */
int tg_reorder_features(tg_ctx* ctx, const void* src, uint64_t rows, uint64_t row_bytes,
                        const uint64_t* perm, uint64_t perm_len, void* dst);
/* reorder.hpp:33 reorder_graph (reorder.cpp:39-66, Algorithm 2). Inputs and
 * outputs host|device; out_offsets n+1, out_targets e. */
int tg_reorder_graph(tg_ctx* ctx, const uint64_t* offsets, const uint64_t* targets, uint64_t n,
                     uint64_t e, const uint64_t* perm, uint64_t perm_len, uint64_t* out_offsets,
                     uint64_t* out_targets);

/* ---------------------------------------------------------------- tiering
 * Host-side scalar logic (tiering.cpp:10-98); no device work. */
int tg_validate_layout(const tg_layout* layout);
int tg_validate_cost_model(double local_gbps, double peer_gbps, double host_gbps);
int tg_resolve(const tg_layout* layout, uint64_t row_id, uint32_t requesting_device,
               tg_location* out);
int tg_plan_layout(uint64_t num_rows, double hot_fraction, double replicated_fraction,
                   uint32_t num_devices, uint64_t feature_dim, uint32_t elem_bytes,
                   uint64_t per_device_budget_bytes, tg_layout* out);
double tg_report_hit_ratio(const tg_report* r);
double tg_report_est_transfer_seconds(const tg_report* r, double local_gbps, double peer_gbps,
                                      double host_gbps);

/* tiering.hpp:88-89 gather (tiering.cpp:100-125), accounting only, on the
 * GPU. ids host|device; report is ACCUMULATED like the reference's. On an
 * out-of-range id the ids before it stay accounted and TG_ERR_DOMAIN is
 * returned, exactly like the reference's throwing loop. */
int tg_gather_account(tg_ctx* ctx, const tg_layout* layout, const uint64_t* ids, uint64_t n,
                      uint32_t requesting_device, tg_report* report);

/* tiering.hpp:95 simulate_trace (tiering.cpp:127-162); counts host|device. */
int tg_simulate_trace(tg_ctx* ctx, const uint64_t* counts, uint64_t n, const tg_layout* layout,
                      tg_report* out);
/* tiering.hpp:98-99 counts_in_row_order (tiering.cpp:164-175) */
int tg_counts_in_row_order(tg_ctx* ctx, const uint64_t* counts, uint64_t n,
                           const uint64_t* ordering, uint64_t m, uint64_t* out);
/* tiering.hpp:110-117 hot_fraction_sweep (tiering.cpp:177-202). Per fraction i:
 * out_layouts[i], out_reports[i], out_replicated[i] (all host). */
int tg_hot_fraction_sweep(tg_ctx* ctx, const uint64_t* counts, uint64_t n,
                          const uint64_t* ordering, const double* fractions, uint64_t nf,
                          double replicated_fraction, uint32_t num_devices, uint64_t feature_dim,
                          uint32_t elem_bytes, uint64_t per_device_budget_bytes,
                          tg_layout* out_layouts, tg_report* out_reports,
                          double* out_replicated);

/* --------------------------------------------------- tiered feature store
 * The byte-moving gather the paper describes (Listing 1;
 * :346-353) and the reference only accounts for. One store per device
 * (device_index in [0, num_devices)): replicated rows [0, lb) and this
 * device's interleaved slice of [lb, mb) live in local HBM; cold rows
 * [mb, num_rows) live in pinned, mapped host memory read by UVA zero-copy.
 * Row ids are NEW ids (after permutation_from_scores), as resolve() takes. */
typedef struct tg_store tg_store;

#define TG_COLD_REORDERED 0u /* pinned copy of the cold rows in new-id order   */
#define TG_COLD_INDIRECT 1u  /* register the caller's original host matrix and  */
                             /* index it through the permutation (no host copy) */
#define TG_COLD_PAD128 2u    /* pad cold rows to a 128 B stride (PCIe lines)    */
#define TG_GATHER_BULK 4u    /* K8 via TMA bulk copies (cp.async.bulk) staged   */
                             /* through shared memory                            */
#define TG_GATHER_L2PF 8u    /* K8 LDG path with the L2::256B prefetch hint      */
#define TG_GATHER_SPREAD 16u /* K8: deal consecutive batches across CTAs         */
#define TG_COLD_SPLIT_TAIL 32u /* TG_COLD_REORDERED with R % 128 != 0: keep each  */
                             /* cold row's whole 128 B lines in host memory and */
                             /* the R mod 128 remainder in HBM (one PCIe read   */
                             /* request fewer per cold row)                      */
#define TG_GATHER_DYNAMIC 64u /* K8 bulk: after one statically spread round,     */
                             /* warps claim batches from a device counter        */

int tg_store_create(tg_ctx* ctx, const tg_layout* layout, uint32_t device_index, uint32_t flags,
                    tg_store** out);
int tg_store_destroy(tg_store* s);
/* K7 placement. features: the ORIGINAL matrix (old-id order, num_rows x
 * row_bytes, host|device); new_id_of: NodePermutation (host|device). Fills
 * this device's hot rows and (TG_COLD_REORDERED) the cold copy. */
int tg_store_place(tg_store* s, const void* features, const uint64_t* new_id_of);
/* Base of this store's local HBM region (replicated rows then the slice). */
/* K7 from a caller's row array: new id i holds source row row_of[i]
 * (rows: nrows x row_bytes, host (registered in place) or device; row_of:
 * N u32, host or device, each < nrows). tg_store_place is the case
 * rows = the original matrix, row_of = the inverse permutation. With
 * TG_COLD_INDIRECT the cold tier is read in place through row_of (e.g. a
 * host row cache in its own order). */
int tg_store_place_rows(tg_store* s, const void* rows, uint64_t nrows, const uint32_t* row_of);
void* tg_store_local_base(const tg_store* s);
uint64_t tg_store_local_rows(const tg_store* s);
/* Bytes of each cold row read over PCIe (row_bytes, or its whole 128 B lines
 * under TG_COLD_SPLIT_TAIL once placed). */
uint64_t tg_store_cold_host_bytes(const tg_store* s);
/* Point device d's slot of the combined-tensor table at a peer's local base
 * (same-process peer pointer, or a CUDA-IPC mapping from tg_ipc_open). */
int tg_store_set_peer(tg_store* s, uint32_t d, const void* peer_local_base);
/* Share one cold tier between stores/processes: use `host` (mapped pinned or
 * registered memory holding the cold rows in the store's cold format). */
int tg_store_share_cold(tg_store* s, const tg_store* owner);
/* Host bytes of this store's cold tier in its cold format (stride, split). */
uint64_t tg_store_cold_tier_bytes(const tg_store* s);
/* Use caller memory (mapped: registered or a tg_host_shared_map segment) as
 * the cold tier, before placement. fill != 0: this store's placement writes
 * the cold rows there; fill == 0: another store (typically another process
 * of the node) has written them and this one only reads. */
int tg_store_attach_cold(tg_store* s, void* host, uint64_t bytes, int fill);
/* One host segment per node shared by every process: POSIX shared memory
 * `name` ("/tg_cold_<job>") of `bytes`, created (create != 0, fails if it
 * exists) or opened, mapped and registered with the device (mapped |
 * portable). Unmap in every process, unlink once. */
int tg_host_shared_map(const char* name, uint64_t bytes, int create, void** out);
int tg_host_shared_unmap(void* p, uint64_t bytes);
int tg_host_shared_unlink(const char* name);

/* K8: copy rows ids[0..n) (host|device) into dst (n x row_bytes, host|device)
 * and accumulate the reference accounting into report (host). Synchronous:
 * returns once every row is in dst and the report is final (device dst: when
 * the kernel's last CTA has posted the counters to mapped host memory, before
 * the stream drains; host dst: after the copy back). */
int tg_gather_rows(tg_store* s, const uint64_t* ids, uint64_t n, void* dst, tg_report* report);
/* Same, stream-ordered: ids_dev/dst_dev device pointers, counters_dev = 3 x
 * u64 device accumulator {local, peer, host} accesses, err_dev = 1 x u64
 * device word receiving min(bad index)+1 (0 = ok). No synchronisation. */
int tg_gather_rows_async(tg_store* s, const uint64_t* ids_dev, uint64_t n, void* dst_dev,
                         uint64_t* counters_dev, uint64_t* err_dev);

/* Measurement of the synchronous path exactly as a C/C++ caller sees it:
 * k calls of tg_gather_rows (ids[i]: counts[i] host ids each, into dst),
 * each timed with steady_clock around the call; with flush_l2 a 256 MB
 * device memset runs (untimed) before every call. *seconds = the sum. */
int tg_time_gather_rows(tg_store* s, const uint64_t* const* ids, const uint64_t* counts, uint64_t k,
                        void* dst, int flush_l2, tg_report* report, double* seconds);

/* csr_graph.hpp:48 transpose (csr_graph.cpp:67-80) on the device: a stable
 * radix sort of the edges by target in CSR order, so every transposed row
 * lists its sources ascending, bit-identical to the reference. Inputs and
 * outputs host or device; n, e < 2^32. */
int tg_transpose(tg_ctx* ctx, const uint64_t* offsets, const uint64_t* targets, uint64_t n,
                 uint64_t e, uint64_t* out_offsets, uint64_t* out_targets);

/* ----------------------------------------------- containers into the tiers
 * the reference's binary containers (io.hpp:14-22) read
 * straight into device memory through pinned double-buffered staging, with
 * the reference's header errors (io.cpp:65-75, 95-110, 163-180: bad magic /
 * unsupported version / truncated -> TG_ERR_FORMAT; cannot open -> TG_ERR_IO).
 * tg_graph_load_csrg replaces load_csr (io.cpp:95-116) + tg_graph_create:
 * no u64 host copy of the CSR is made. tg_store_place_feat replaces
 * load_features (io.cpp:163-181) + reorder_features + tg_store_place: the
 * file's rows go to this device's HBM slots and the store's own pinned cold
 * tier by the permutation (new_id_of: host or device), without the N x R
 * matrix in host memory. The store must not be TG_COLD_INDIRECT. */
int tg_graph_load_csrg(tg_ctx* ctx, const char* path, tg_graph** out);
int tg_store_place_feat(tg_store* s, const char* path, const uint64_t* new_id_of);

/* ------------------------------------------------------------- peer memory */
int tg_enable_peer_access(int device, int peer);
int tg_ipc_get_handle(const void* dev_ptr, void* handle_out /* 64 bytes */);
int tg_ipc_open_handle(tg_ctx* ctx, const void* handle /* 64 bytes */, void** dev_ptr_out);
int tg_ipc_close_handle(void* dev_ptr);
/* Library-owned device allocation (cudaMalloc on the ctx device, zeroed):
 * the base of its own allocation, so a CUDA-IPC handle of it maps exactly
 * this buffer in another process (used for the cross-process fused
 * PageRank exchange: norm ping-pong, scores and arrival counters). */
int tg_device_alloc(tg_ctx* ctx, uint64_t bytes, void** out);
int tg_device_free(tg_ctx* ctx, void* p);
/* Register caller host memory as mapped pinned (cudaHostRegister). */
int tg_host_register(void* ptr, uint64_t bytes);
int tg_host_unregister(void* ptr);
/* Device address of pinned / registered host memory, NULL if not mapped. */
void* tg_mapped_device_ptr(const void* host);
int tg_host_alloc(uint64_t bytes, void** out); /* cudaHostAlloc Mapped|Portable */
int tg_host_free(void* p);

/* ------------------------------------------------------------ measurement
 * Zero-copy read bandwidth of `bytes` of mapped host memory in rows of
 * row_bytes (random order), timed with CUDA events on the ctx stream; and a
 * device-to-device copy for the HBM reference. Both return GB/s. */
int tg_measure_host_read_gbps(tg_ctx* ctx, uint64_t bytes, uint64_t row_bytes, int reps,
                              double* gbps);
/* Mean time (us) to read `rows` random rows (row_bytes each, at `stride`)
 * out of `region_rows` rows of an existing mapped host region, one launch
 * per rep with the L2 flushed before it: the practical floor of a gather's
 * cold part over the same region (GPU address translation included). */
/* Mean time (us) of this store's own gather (K8) over `rows` random COLD
 * ids only, L2 flushed before each launch: the cold part of a gather timed
 * alone, on the same region, mapping and load path. */
int tg_store_measure_cold_us(tg_store* s, uint64_t rows, int reps, double* us);
/* The platform ceiling of the same: `rows` random rows of the store's cold
 * tier (same region, stride, host bytes per row) by a plain one-warp-per-row
 * copy kernel, L2 flushed; mean us per launch. */
int tg_store_measure_cold_rows_us(tg_store* s, uint64_t rows, int reps, double* us);
int tg_measure_host_rows_us(tg_ctx* ctx, const void* host, uint64_t region_rows, uint64_t stride,
                            uint64_t row_bytes, uint64_t rows, int reps, double* us);
int tg_measure_hbm_copy_gbps(tg_ctx* ctx, uint64_t bytes, int reps, double* gbps);
/* The memory-system floor of one K3 step on graph g: the same E gathers
 * x[targets[e]] with no summation-order constraint (best of reps, us), in
 * the labelling K3 runs on (the relabelled twin when enabled; reps < 0:
 * |reps| repetitions in g's own labelling). */
int tg_measure_gather_floor_us(tg_ctx* ctx, const tg_graph* g, int reps, double* us);
/* K3 relabelling: whether the PageRank entry points run on g's
 * twin renumbered by in-degree (TIERGRAPH_PR_RELABEL=0|1, default: when the
 * norm vector exceeds half of L2), building it now if so; build_ms = the
 * one-time device time of that build. Results are bit-identical either way. */
int tg_pagerank_relabel_info(tg_ctx* ctx, const tg_graph* g, int* relabelled, double* build_ms);

/* ------------------------------------------------ host-side input producers
 * Not the hot path: the reference's CPU producers of the gather's id lists,
 * restated bit-exactly in C++ (csrc/host_producers.cpp). Outputs returned
 * through *_out pointers are malloc'ed; release them with tg_free. */
const char* tg_host_last_error(void);
void tg_free(void* p);
/* scoring.hpp:24 draw_random_train_ids (scoring.cpp:22-31); out has count ids */
int tg_draw_random_train_ids(uint64_t num_nodes, uint64_t count, uint64_t seed, uint64_t* out);
/* csr_graph.hpp:48 transpose (csr_graph.cpp:67-80), host arrays */
int tg_transpose_host(const uint64_t* off, const uint64_t* tgt, uint64_t n, uint64_t* t_off,
                      uint64_t* t_tgt);
/* One epoch of run_training_trace's schedule (sampling.cpp:106-123): shuffle
 * tid with key {0x5348, epoch}, split into batches, expand batches
 * [first_batch, first_batch+max_batches) with build_minibatch (sampling.cpp:56-90)
 * over the transposed graph. Lists are concatenated: batch i is
 * ids[off[i]..off[i+1]). threads <= 0 uses all OpenMP threads. */
int tg_epoch_minibatches(const uint64_t* gt_off, const uint64_t* gt_tgt, uint64_t n,
                         const uint64_t* tid, uint64_t ntid, const uint32_t* fanouts, uint32_t nf,
                         uint64_t batch_size, uint64_t seed, uint64_t epoch, uint64_t first_batch,
                         uint64_t max_batches, int threads, uint64_t** out_off, uint64_t* out_nb,
                         uint64_t** out_ids);

/* ------------------------------------------- GPU minibatch sampling (§8f)
 * sampling.cpp:35-90 build_minibatch on the device, bit-identical member
 * lists. `gt` is the TRANSPOSED graph (row v = in-neighbours of v, rows in
 * the reference transpose's order, csr_graph.cpp:67-80), uploaded with
 * tg_graph_create. The sampler owns per-node stamp arrays (2 x 4n bytes).
 * tg_sample_minibatch: seeds (host|device, ns >= 1, < n) expanded through
 * fanouts[0..nf) with BatchRng{rng_seed, epoch, batch}; writes the sorted
 * unique members to out (host|device, capacity cap) and their count to
 * *out_n (also set when cap is too small, with TG_ERR_DOMAIN). */
typedef struct tg_sampler tg_sampler;
int tg_sampler_create(tg_ctx* ctx, const tg_graph* gt, tg_sampler** out);
int tg_sampler_destroy(tg_sampler* s);
int tg_sample_minibatch(tg_sampler* s, const uint64_t* seeds, uint64_t ns, const uint32_t* fanouts,
                        uint32_t nf, uint64_t rng_seed, uint64_t epoch, uint64_t batch,
                        uint64_t* out, uint64_t cap, uint64_t* out_n);
/* Same, also returning every individual draw (build_minibatch's raw_draws,
 * sampling.hpp:48-55: each seed once as given, then every sampled node; order
 * unspecified, multiset deterministic) into raw (host|device, raw_cap). */
int tg_sample_minibatch_raw(tg_sampler* s, const uint64_t* seeds, uint64_t ns,
                            const uint32_t* fanouts, uint32_t nf, uint64_t rng_seed,
                            uint64_t epoch, uint64_t batch, uint64_t* out, uint64_t cap,
                            uint64_t* out_n, uint64_t* raw, uint64_t raw_cap, uint64_t* raw_n);
/* sampling.cpp:92-140 run_training_trace on the device: per epoch the seeded
 * shuffle, then every batch expanded; counts (n x u64, host|device) get one
 * per unique member per batch (dedup_per_batch) or one per raw access. The
 * sampler's graph is the TRANSPOSED graph; tid is a TrainIdSet (sorted). */
/* Many minibatches of one epoch in one call, no host round trip between
 * them: batch b (first_batch <= b < first_batch + nbatches) expands seeds
 * order[b*B, (b+1)*B) with BatchRng{rng_seed, epoch, b} (sampling.cpp:35-37,
 * 106-115). Members of batch k go to out_members[out_offsets[k],
 * out_offsets[k+1]) (sorted unique); out_offsets has nbatches + 1 entries.
 * Outputs host or device; cap = out_members entries. */
int tg_sample_batches(tg_sampler* s, const uint64_t* order, uint64_t n_order, uint64_t batch_size,
                      uint64_t first_batch, uint64_t nbatches, const uint32_t* fanouts,
                      uint32_t nf, uint64_t rng_seed, uint64_t epoch, uint64_t* out_members,
                      uint64_t cap, uint64_t* out_offsets);
int tg_sampler_trace(tg_sampler* s, const uint64_t* tid, uint64_t ntid, const uint32_t* fanouts,
                     uint32_t nf, uint64_t batch_size, uint64_t epochs, uint64_t rng_seed,
                     int dedup_per_batch, uint64_t* counts);
/* ------------------------------------ graph-structure tiering (§8f row 2)
 * the sampler's graph distributed like the features. The
 * reference only estimates it (tools/tiergraph_cli.cpp:389-406,
 * --structure-of). Row v of the TRANSPOSED, score-reordered graph (new ids)
 * is placed where resolve(v) (tiering.cpp:48-65) puts feature row v: rows
 * [0, lb) in every device's HBM, device (v-lb) % D's slice for [lb, mb), and
 * [mb, N) in pinned mapped host memory (UVA). Offsets (u64, host|device,
 * validated like tg_graph_create: FormatError "csr: ...") are kept as u32 on
 * every device. cold_host: optional caller memory mapped for the device
 * (tg_host_register / a shared segment), >= tg_sgraph_cold_bytes; with
 * cold_fill = 0 another tiered graph (process) writes it. Without cold_host
 * the graph allocates its own pinned cold tier. */
typedef struct tg_sgraph tg_sgraph;
uint64_t tg_sgraph_cold_bytes(const uint64_t* offsets, uint64_t n, const tg_layout* layout);
int tg_sgraph_create(tg_ctx* ctx, const tg_layout* layout, uint32_t device_index,
                     const uint64_t* offsets, const uint64_t* targets, uint64_t n, uint64_t e,
                     void* cold_host, uint64_t cold_bytes, int cold_fill, tg_sgraph** out);
int tg_sgraph_destroy(tg_sgraph* s);
/* This device's interleaved slice (for CUDA IPC) and a peer's slice base
 * (same process: its tg_sgraph_local_base; other process: the IPC mapping). */
void* tg_sgraph_local_base(const tg_sgraph* s);
int tg_sgraph_set_peer(tg_sgraph* s, uint32_t d, const void* peer_slice_base);
void* tg_sgraph_cold_host(const tg_sgraph* s);
/* out[4]: bytes of replicated rows (HBM), this device's slice (HBM), the cold
 * rows (host), and offsets + slice starts (HBM). */
int tg_sgraph_info(const tg_sgraph* s, uint64_t* out);
/* A sampler over a tiered graph: the same bit-identical build_minibatch
 * lists as tg_sampler_create on the whole graph. tg_sampler_structure_reads
 * returns the neighbour ids read since the last reset per tier {local HBM,
 * peer HBM, host}: min(deg, fanout) per frontier node, counted where the
 * node's row lives for this device. */
int tg_sampler_create_tiered(tg_ctx* ctx, const tg_sgraph* sg, tg_sampler** out);
int tg_sampler_structure_reads(tg_sampler* s, uint64_t* out, int reset);

/* sampling.cpp:106-109: the epoch's shuffled train-id order (Fisher-Yates,
 * key {0x5348, epoch}); batch b is order[b*batch_size ..). Host arrays. */
int tg_epoch_order(const uint64_t* tid, uint64_t ntid, uint64_t rng_seed, uint64_t epoch,
                   uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* TG_CAPI_H_ */
