/*
 * slimsell_b200.h — the C-ABI boundary of the B200-native SlimSell BFS-SpMV
 * path (libslimsell_b200.so, sm_100a).
 *
 * Every entry point replaces one function of the reference C++ library
 * (arXiv 2010.09913 artifact, /root/reference/proj); the citation next to each
 * declaration names the reference interface (file:line) it stands in for.
 * Conventions:
 *   - plain pointers and sizes only, no C++ or torch types;
 *   - every function returns an SSB_* status; the message of the last failure
 *     on the calling thread is ssb_last_error();
 *   - handles are opaque, owned by the caller, released with *_destroy;
 *   - host buffers are caller-allocated; every call is synchronous on return;
 *   - vertex ids are int64 at the boundary (reference vid_t/val_t, graph.hpp:12,
 *     semiring.hpp:17); the device stores int32 ids (n < 2^31).
 * Status -> reference exception (bfs.hpp / repr.hpp / semiring.hpp):
 *   SSB_EINVAL -> std::invalid_argument, SSB_ERANGE -> std::out_of_range,
 *   SSB_ECAP -> BfsCapError (partial dist still written),
 *   SSB_EPARSE -> ParseError, SSB_ECUDA / SSB_ENOMEM -> std::runtime_error.
 */
#ifndef SLIMSELL_B200_H
#define SLIMSELL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSB_OK 0
#define SSB_EINVAL 1
#define SSB_ERANGE 2
#define SSB_ECAP 3
#define SSB_ECUDA 4
#define SSB_ENOMEM 5
#define SSB_EPARSE 6 /* slimsell::ParseError (graph.hpp:15-21): "line N: ..." */

#define SSB_ABI_VERSION 2

/* Variant (semiring.hpp:25). */
#define SSB_TROPICAL 0
#define SSB_REAL 1
#define SSB_BOOLEAN 2
#define SSB_SELMAX 3

typedef struct ssb_edges ssb_edges; /* normalised Graph on the device (graph.hpp:31-51) */
typedef struct ssb_graph ssb_graph; /* SlimSellRepr on the device (repr.hpp:33-55) */
typedef struct ssb_ctx ssb_ctx;     /* the devices of a single-process multi-GPU job */
typedef struct ssb_sharded ssb_sharded; /* a SlimSellRepr sharded over a context's devices */

/* SlimSellRepr scalar fields (repr.hpp:33-45). n_cells = |col| = Σ C·cl of
 * the whole layout. A handle built for chunk segments
 * (ssb_build_slimsell_range / _segments) holds the cells of those chunks
 * only: range_cells of them, in range_segments segments spanning
 * [range_begin, range_end); a whole layout has one segment [0, n_chunks) and
 * range_cells = n_cells. */
typedef struct {
  int64_t C, sigma, n, n_padded, n_chunks, nonzeros, n_cells, padding, max_chunk_len;
  int64_t range_begin, range_end, range_cells, range_segments;
} ssb_layout_info;

/* BfsOptions (bfs.hpp:16-24). schedule and workers are accepted for API
 * compatibility and ignored: the device schedules its own work units. */
typedef struct {
  int32_t variant;        /* SSB_TROPICAL .. SSB_SELMAX */
  int32_t slimwork;       /* skip chunks whose real rows are all visited */
  int64_t slimchunk_len;  /* L: max columns per work unit; 0 = SlimChunk off */
  int32_t schedule;       /* ignored (Schedule, bfs.hpp:14) */
  int32_t workers;        /* ignored */
  int64_t max_iterations; /* <= 0 resolves to n + 1 (bfs.cpp:70-71) */
  int32_t want_parents;
  int32_t selmax_compat;  /* 1: reproduce the reference's sel-max root encoding
                             (SURVEY.md App. A.3); 0: corrected parents */
} ssb_bfs_options;

/* IterStats (bfs.hpp:26-34); elapsed_ns is device time of the iteration. */
typedef struct {
  int64_t iteration, elapsed_ns, chunks_processed, chunks_skipped, subchunks_processed,
      columns_processed, frontier_size;
} ssb_iter_stats;

const char* ssb_last_error(void);
int ssb_abi_version(void);
/* Selects the CUDA device for handles created afterwards on this thread. */
int ssb_set_device(int device);

/* ---- graph input (L1) -------------------------------------------------- */
/* Graph::from_pairs (graph.hpp:36, graph.cpp:65-86): orient u<v, drop
 * self-loops, sort, dedup — on the device. uv holds count (u,v) pairs;
 * n < 0 infers max id + 1. ERANGE for negative / out-of-range ids. */
int ssb_edges_from_pairs(const int64_t* uv, int64_t count, int64_t n, ssb_edges** out);
/* gen_kronecker (generator.hpp:55, generator.cpp:60-89), bit-exact, on the
 * device: counter-based SplitMix64 draws + from_pairs normalisation. */
int ssb_gen_kronecker(int64_t scale, int64_t edgefactor, uint64_t seed,
                      const double initiator[4], ssb_edges** out);
/* gen_erdos_renyi (generator.hpp:50, generator.cpp:15-58), bit-exact: the
 * counter-based geometric skips are drawn by all host threads with the same
 * libm as the reference, prefix-summed, and decoded to (u, v) on the device.
 * EINVAL for n < 0 or p outside [0, 1]. */
int ssb_gen_erdos_renyi(int64_t n, double p, uint64_t seed, ssb_edges** out);
/* from_edge_list (graph.hpp:50-56, graph.cpp:94-133): whitespace-separated
 * "u v" records, '#'/'%' comment lines, an optional leading "H n m" header that
 * pins n. SSB_REJECT_ASYMMETRIC requires the reverse of every non-loop record.
 * The text is parsed on the host; normalisation runs on the device. */
#define SSB_SYMMETRIZE 0
#define SSB_REJECT_ASYMMETRIC 1
int ssb_edges_from_edge_list(const char* text, int64_t len, int directive, ssb_edges** out);
/* from_matrix_market (graph.hpp:58-59, graph.cpp:135-210): coordinate
 * pattern|real, general|symmetric, square, 1-based entries. */
int ssb_edges_from_matrix_market(const char* text, int64_t len, ssb_edges** out);
/* The parsers alone (host only, no device work): *uv receives 2*count int64
 * (the records before normalisation, 0-based), release it with ssb_free;
 * *n = the declared vertex count (-1 when an edge list has no header). */
int ssb_parse_edge_list(const char* text, int64_t len, int directive, int64_t** uv,
                        int64_t* count, int64_t* n);
int ssb_parse_matrix_market(const char* text, int64_t len, int64_t** uv, int64_t* count,
                            int64_t* n);
void ssb_free(void* p);
/* Graph::num_vertices / num_edges (graph.hpp:42-43). */
int ssb_edges_info(const ssb_edges* e, int64_t* n, int64_t* m);
/* Graph::edges() (graph.hpp:44): 2*m int64, sorted (u<v) pairs. */
int ssb_edges_export(const ssb_edges* e, int64_t* uv);
/* to_csr (graph.hpp:71, graph.cpp:212-232): row n+1, col 2m, rows ascending. */
int ssb_to_csr(const ssb_edges* e, int64_t* row, int64_t* col);
void ssb_edges_destroy(ssb_edges* e);

/* ---- layout (L2) ------------------------------------------------------- */
/* build_slimsell (repr.hpp:66, repr.cpp:84-131) on the device: σ-window sort
 * by (degree desc, id asc), chunk height C, column-major col with -1 padding,
 * no value array. EINVAL for C <= 0 or sigma <= 0. */
int ssb_build_slimsell(const ssb_edges* e, int64_t C, int64_t sigma, ssb_graph** out);
/* One rank's share of a multi-GPU layout ("each GPU holds
 * its own col/cs/cl"): the same σ-sort, perm and chunk lengths as
 * ssb_build_slimsell for every chunk, but the cells of chunks
 * [chunk_begin, chunk_end) only (cs offsets into that partial col). Such a
 * handle serves the sharded BFS of an owned range inside it
 * (ssb_bfs_shard_*, ssb_p2p_attach / ssb_bfs_p2p[_group]), ssb_spmv_step on
 * chunks inside it, ssb_graph_info / degrees / col32 export of its cells;
 * whole-layout calls (ssb_bfs_run / ssb_bfs_spmv, col / cs export) return
 * EINVAL. chunk_end < 0 = n_chunks. */
int ssb_build_slimsell_range(const ssb_edges* e, int64_t C, int64_t sigma, int64_t chunk_begin,
                             int64_t chunk_end, ssb_graph** out);
/* The same for several chunk segments (bounds = 2·nseg chunk indices
 * [b0, e0, b1, e1, ...], disjoint): the round-robin partition that keeps the
 * ranks balanced once SlimWork skips the hub chunks. */
int ssb_build_slimsell_segments(const ssb_edges* e, int64_t C, int64_t sigma, const int64_t* bounds,
                                int64_t nseg, ssb_graph** out);
/* Uploads a host SlimSellRepr (the reference struct's arrays, int64). */
int ssb_graph_from_layout(int64_t n, int64_t C, int64_t sigma, int64_t nonzeros,
                          const int64_t* col, int64_t n_cells, const int64_t* cs,
                          const int64_t* cl, int64_t n_chunks, const int64_t* perm,
                          ssb_graph** out);
int ssb_graph_info(const ssb_graph* g, ssb_layout_info* info);
/* Materialises the SlimSellRepr arrays on the host (any pointer may be NULL):
 * col n_cells, cs n_chunks, cl n_chunks, perm n, inv_perm n. */
int ssb_graph_export(const ssb_graph* g, int64_t* col, int64_t* cs, int64_t* cl,
                     int64_t* perm, int64_t* inv_perm);
/* Row length (degree) of every ORIGINAL vertex id: n int64 (the
 * row[v+1]-row[v] of to_csr, graph.hpp:63-71). */
int ssb_graph_degrees(const ssb_graph* g, int64_t* deg);
/* Compact export of col as int32 (the device storage type). */
int ssb_graph_export_col32(const ssb_graph* g, int32_t* col);
void ssb_graph_destroy(ssb_graph* g);

/* ---- kernels (L2/L3) --------------------------------------------------- */
/* spmv_step (repr.hpp:90-92, repr.cpp:193-217): for chunks [chunk_begin,
 * chunk_end), out rows = plus({x_prev[v]} ∪ {times(x_prev[u], edge)}) with the
 * literal int64 semiring arithmetic (semiring.hpp:56-87). x_prev and out hold
 * n_padded values in the permuted numbering; rows outside the range are left
 * untouched. EINVAL for a bad range or variant. */
int ssb_spmv_step(const ssb_graph* g, int variant, const int64_t* x_prev, int64_t* out,
                  int64_t chunk_begin, int64_t chunk_end);
/* The same with x_prev / out in DEVICE memory (n_padded int64 each): one warp
 * per work unit of <= 1024 columns (hub chunks split, folded by 64-bit
 * atomics), no host copies. device_ms (may be NULL): CUDA-event time. */
int ssb_spmv_step_device(const ssb_graph* g, int variant, const int64_t* x_prev, int64_t* out,
                         int64_t chunk_begin, int64_t chunk_end, double* device_ms);
/* spmv_segment (repr.hpp:79-81, repr.cpp:20-35, 153-170): acc[lane] =
 * plus(acc[lane], times(x_prev[c], edge or pad)) over columns [col_begin,
 * col_begin + col_len) of `chunk`; x_prev n_padded int64, acc C int64 (in/out),
 * host memory. EINVAL for a chunk or column range outside the layout. */
int ssb_spmv_segment(const ssb_graph* g, int variant, const int64_t* x_prev, int64_t* acc, int64_t chunk,
                     int64_t col_begin, int64_t col_len);

/* bfs_spmv (bfs.hpp:80-81, bfs.cpp:222-246): algebraic BFS on the device.
 * dist: n int64 in original ids, INT64_MAX when unreached. parent: n int64
 * (may be NULL); *parent_len receives n when parents were produced, else 0 —
 * sel-max decodes its tracked parents (bfs.cpp:94-101); the other variants
 * derive them from dist like dp_transform (semiring.cpp:159-187) over the
 * layout's adjacency. stats: up to stats_cap IterStats. ERANGE for a bad root,
 * ECAP when the iteration cap is hit (dist holds the partial result). */
int ssb_bfs_spmv(ssb_graph* g, int64_t root, const ssb_bfs_options* opts, int64_t* dist,
                 int64_t* parent, int64_t* parent_len, ssb_iter_stats* stats,
                 int64_t stats_cap, int64_t* iterations);

/* A batch of bfs_spmv calls (Graph500 runs a root list): root i's result is
 * written to dist[i] / parent[i] (parent may be NULL or hold NULLs; entries may
 * alias — root i's result then replaces root i-1's), as ssb_bfs_spmv would.
 * Root i's result crosses PCIe and is widened on the host while root i+1's
 * BFS runs on the device. ERANGE for a bad root (nothing run); ECAP when a
 * root hits the iteration cap: *capped_at = its index (its dist delivered, no
 * parents, later roots not run), else -1. iterations (may be NULL): per root. */
int ssb_bfs_spmv_batch(ssb_graph* g, const int64_t* roots, int64_t nroots, const ssb_bfs_options* opts,
                       int64_t* const* dist, int64_t* const* parent, int64_t* iterations,
                       int64_t* capped_at);

/* Device-resident form used by benchmarks: runs the BFS and leaves the
 * result on the device. device_ms = CUDA-event time of the iteration loop on
 * the handle's stream. */
int ssb_bfs_run(ssb_graph* g, int64_t root, const ssb_bfs_options* opts,
                ssb_iter_stats* stats, int64_t stats_cap, int64_t* iterations,
                double* device_ms);
/* Copies the last ssb_bfs_run result out (original ids), as ssb_bfs_spmv. */
int ssb_bfs_fetch(ssb_graph* g, int want_parents, int64_t* dist, int64_t* parent,
                  int64_t* parent_len);
/* Timing of the last ssb_bfs_run: CUDA-event time of the main BFS kernel
 * launches alone (kernel_ms) and how many kernels the BFS launched. */
int ssb_bfs_last_timing(ssb_graph* g, double* kernel_ms, int64_t* launches);
/* Columns the last run actually streamed from HBM, summed over iterations:
 * the early-exit sweeps stop a work unit once every row of it is decided, so
 * this is <= Σ IterStats.columns_processed (the reference's counter). The
 * roofline's algorithmic bytes are 4·C per swept column. */
int ssb_bfs_columns_swept(ssb_graph* g, int64_t* swept);
/* ---- multi-GPU: chunk-range shards -------------------
 * Each rank builds (or holds) the layout, owns chunks [chunk_begin, chunk_end)
 * (C = 32: chunk i <-> frontier word i) and the replicated 1-bit frontier.
 * Per BFS iteration: ssb_bfs_shard_step sweeps the owned chunks and copies the
 * owned frontier words (chunk_end - chunk_begin uint32, device memory) to
 * owned_words; the caller all-gathers them (NCCL) into the full n_chunks-word
 * frontier and sums |newly| over ranks; ssb_bfs_shard_exchange installs it.
 * Stop after the iteration whose global newly count is 0 (is_converged,
 * semiring.cpp:152-157). ssb_bfs_shard_fetch writes dist/parent (original
 * ids) of the owned rows only; other entries of the host arrays are kept. */
int ssb_bfs_shard_begin(ssb_graph* g, int64_t root, const ssb_bfs_options* opts,
                        int64_t chunk_begin, int64_t chunk_end);
int ssb_bfs_shard_step(ssb_graph* g, ssb_iter_stats* local, uint32_t* owned_words);
int ssb_bfs_shard_exchange(ssb_graph* g, const uint32_t* frontier_words, int64_t newly_total);
int ssb_bfs_shard_fetch(ssb_graph* g, int want_parents, int64_t* dist, int64_t* parent);
/* The same iteration without a host round trip (the NCCL form of SURVEY.md
 * §8(e)): the sweep reads |F_{k-1}|, the active task list and the retired-
 * chunk count from a device-resident carry, so nothing returns to the host
 * between iterations. Per iteration k:
 *   ssb_bfs_shard_step_async      sweep + owned words copied out, on the
 *                                 graph's stream (ssb_graph_stream);
 *   <the caller's all-gather>     enqueued on that same stream (NCCL);
 *   ssb_bfs_shard_exchange_async  full frontier installed, summary rebuilt,
 *                                 global |F_k| counted on the device.
 * ssb_bfs_shard_front(k) waits for iteration k's exchange only and returns
 * |F_k| (poll k-1 while k is queued; an iteration queued after convergence
 * does nothing). ssb_bfs_shard_finish(iterations) returns this rank's
 * per-iteration counters (local to its chunks: sum them over ranks once per
 * BFS) and the device time since begin. Then ssb_bfs_shard_fetch. */
int ssb_graph_stream(ssb_graph* g, void** stream);
int ssb_bfs_shard_begin_async(ssb_graph* g, int64_t root, const ssb_bfs_options* opts,
                              int64_t chunk_begin, int64_t chunk_end);
int ssb_bfs_shard_step_async(ssb_graph* g, uint32_t* owned_words);
int ssb_bfs_shard_exchange_async(ssb_graph* g, const uint32_t* frontier_words);
int ssb_bfs_shard_front(ssb_graph* g, int64_t k, int64_t* front);
int ssb_bfs_shard_finish(ssb_graph* g, int64_t iterations, ssb_iter_stats* stats, int64_t stats_cap,
                         double* device_ms);
/* ---- multi-GPU, fused: chunk-range shards whose frontier exchange runs
 * inside the BFS kernel (replaces the per-iteration host
 * round trip of ssb_bfs_shard_*). Each rank's frontier bitmaps live in a
 * device WINDOW that every peer maps (CUDA IPC, peer access over NVLink):
 * after its sweep a rank stores its owned frontier words and ORs its summary
 * words into every peer's window, publishes its |newly| count and meets the
 * others at a counter barrier in its own window — one cooperative launch per
 * BFS on every rank, no host step between iterations.
 * ssb_p2p_window: allocates this rank's window; ipc_handle (may be NULL)
 *   receives its cudaIpcMemHandle_t (64 bytes) for the peers.
 * ssb_p2p_attach: maps the peers' windows; ipc_handles = world handles in
 *   rank order (this rank's entry is ignored); [chunk_begin, chunk_end) is
 *   the owned range. Every rank attaches before any rank starts a BFS, and
 *   all ranks run the same GPU model (equal CTA counts).
 * ssb_bfs_p2p: one BFS from `root` on this rank; every rank calls it with
 *   the same root and options. stats: this rank's counters (sum over ranks
 *   for the reference's IterStats). Results: ssb_bfs_shard_fetch (owned rows).
 * ssb_bfs_p2p_group: `world` shards (2..8 handles on THIS device) run as one
 *   cooperative launch — the same kernel and exchange code, peers being
 *   plain device memory; stats summed. */
int ssb_p2p_window(ssb_graph* g, void* ipc_handle, int64_t* window_bytes);
int ssb_p2p_attach(ssb_graph* g, int rank, int world, const void* ipc_handles,
                   int64_t chunk_begin, int64_t chunk_end);
/* ... owning several chunk segments (bounds = 2·nseg, disjoint, nseg <= 8). */
int ssb_p2p_attach_segments(ssb_graph* g, int rank, int world, const void* ipc_handles,
                            const int64_t* bounds, int64_t nseg);
int ssb_bfs_p2p(ssb_graph* g, int64_t root, const ssb_bfs_options* opts, ssb_iter_stats* stats,
                int64_t stats_cap, int64_t* iterations, double* device_ms);
/* bounds: every rank's segments in rank order; seg_counts[i] = rank i's
 * segment count (NULL: one each, bounds = 2·world). */
int ssb_bfs_p2p_group(ssb_graph* const* shards, int world, const int64_t* bounds,
                      const int64_t* seg_counts, int64_t root, const ssb_bfs_options* opts,
                      ssb_iter_stats* stats, int64_t stats_cap, int64_t* iterations,
                      double* device_ms);
/* ---- checking at scale --------------------------------
 * bfs_traditional (bfs.hpp:83, bfs.cpp:248-286) on the device: an independent
 * level-synchronous queue BFS over the CSR of original ids; parent = the
 * smallest neighbour one level closer, root self-parented, unreached -1 /
 * INT64_MAX. stats: per level {iteration, elapsed_ns, frontier_size}, as the
 * reference fills them. ERANGE for a bad root. */
int ssb_bfs_traditional(ssb_edges* e, int64_t root, int64_t* dist, int64_t* parent,
                        ssb_iter_stats* stats, int64_t stats_cap, int64_t* iterations);
/* The parent-tree checks of verify_against_oracle (cli.cpp:73-112: unreached
 * => parent -1, root self-parented, parent a neighbour one level closer) plus
 * the Graph500 edge checks that replace the oracle's distances (edges join
 * levels at most 1 apart, never a reached and an unreached vertex; only the
 * root at level 0), on the device. parent may be NULL (distances only).
 * *violations = number of failed checks; report (NUL-terminated, up to
 * report_cap bytes, may be NULL) lists the first few. flags:
 * SSB_VALIDATE_SELMAX_COMPAT skips the parents of levels 0 and 1, which the
 * reference's sel-max encoding sets to perm[root]. */
#define SSB_VALIDATE_SELMAX_COMPAT 1
int ssb_validate_bfs(ssb_edges* e, int64_t root, const int64_t* dist, const int64_t* parent,
                     int flags, int64_t* violations, char* report, int64_t report_cap);
/* Bit-exact parents at any scale: ssb_validate_bfs plus, for every reached
 * vertex, parent == the value the reference returns —
 *   SSB_VALIDATE_MIN_PARENT_EXACT: the smallest original-id neighbour one level
 *     closer, root self-parented (dp_transform semiring.cpp:159-187 ==
 *     bfs_traditional bfs.cpp:248-291; tropical / real / boolean);
 *   SSB_VALIDATE_SELMAX_EXACT: perm[max{inv_perm[u] : u ∈ N(v), d(u) = d(v)-1}]
 *     (selmax_parents bfs.cpp:94-101); with SSB_VALIDATE_SELMAX_COMPAT the root
 *     and its depth-1 vertices must hold perm[root] (the reference's root
 *     encoding), else root.
 * layout supplies perm / inv_perm (required for SELMAX_EXACT, may be NULL
 * otherwise); it must be the layout the BFS ran on. O(m) device work. */
#define SSB_VALIDATE_MIN_PARENT_EXACT 2
#define SSB_VALIDATE_SELMAX_EXACT 4
int ssb_validate_bfs_exact(ssb_edges* e, const ssb_graph* layout, int64_t root, const int64_t* dist,
                           const int64_t* parent, int flags, int64_t* violations, char* report,
                           int64_t report_cap);
/* ---- single-process multi-device (SURVEY.md §8(b) ssb_ctx_create) --------
 * A context names the ranks' devices. All distinct: peer access is enabled
 * between every pair (ECUDA if a pair has no peer path) and each BFS runs one
 * cooperative launch per device, the frontier exchange fused over NVLink peer
 * stores (the ssb_bfs_p2p path with raw peer pointers instead of IPC). All the
 * same device: the ranks run as ONE cooperative launch there (the emulated
 * group of ssb_bfs_p2p_group). Mixed lists are EINVAL.
 * ssb_ctx_build: the layout (C = 32) sharded into segments_per_rank
 * round-robin, cell-balanced chunk segments per rank; rank i
 * holds only its segments' cells, on its device. e may live on any device of
 * the context and must be the CURRENT device's handle.
 * ssb_sharded_bfs: bfs_spmv over the shards, outputs as ssb_bfs_spmv (dist in
 * original ids; sel-max parents when want_parents, parent_len = n, else 0;
 * counters summed over the ranks). ERANGE bad root, ECAP at the cap.
 * ssb_sharded_info: ranks, n, cells and segments per rank (arrays of n_ranks,
 * may be NULL). */
int ssb_ctx_create(int n_ranks, const int* device_ids, ssb_ctx** out);
/* The partition ssb_ctx_build uses (host only, no device): k·world contiguous
 * chunk pieces of near-equal C·cl + 1 weight dealt to the ranks in snake
 * order; bounds receives world·k pairs [b, e) rank by rank (2·world·k int64). */
int ssb_partition_segments(const int32_t* cl, int64_t n_chunks, int64_t C, int world, int k, int64_t* bounds);
void ssb_ctx_destroy(ssb_ctx* ctx);
int ssb_ctx_build(ssb_ctx* ctx, const ssb_edges* e, int64_t C, int64_t sigma, int segments_per_rank,
                  ssb_sharded** out);
int ssb_sharded_info(const ssb_sharded* sh, int* n_ranks, int64_t* n, int64_t* cells_per_rank,
                     int64_t* segments_per_rank);
int ssb_sharded_bfs(ssb_sharded* sh, int64_t root, const ssb_bfs_options* opts, int64_t* dist,
                    int64_t* parent, int64_t* parent_len, ssb_iter_stats* stats, int64_t stats_cap,
                    int64_t* iterations, double* device_ms);
void ssb_sharded_destroy(ssb_sharded* sh);

/* m_cc of the last run: Σ_{reached v} deg(v) / 2 (the GTEPS numerator). */
int ssb_bfs_edges_traversed(ssb_graph* g, int64_t* m_cc);

#ifdef __cplusplus
}
#endif
#endif /* SLIMSELL_B200_H */
