// Internal declarations shared by the sm_100a translation units of
// libslimsell_b200.so. Not installed; the public surface is
// include/slimsell_b200.h (C-ABI) and include/slimsell_b200/*.hpp (C++ façade).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "slimsell_b200.h"

namespace ssb {

// Status-carrying exception; the C-ABI layer maps it to SSB_* codes and the
// thread-local last-error string.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    fail(e == cudaErrorMemoryAllocation ? SSB_ENOMEM : SSB_ECUDA,
         std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
             std::to_string(line) + ")");
  }
}
#define SSB_CUDA(x) ::ssb::cuda_check((x), #x, __FILE__, __LINE__)

// RAII device buffer (cudaMalloc; stream-ordered frees are not needed here:
// every C-ABI call is synchronous on return).
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) SSB_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void ensure(size_t count) { if (count > n) alloc(count); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// One stream + timing events per handle.
struct StreamCtx {
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaEvent_t e_end = nullptr;  // end of the last BFS launch's device work (before any host sync)
  StreamCtx() {
    SSB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    SSB_CUDA(cudaEventCreate(&e0));
    SSB_CUDA(cudaEventCreate(&e1));
    SSB_CUDA(cudaEventCreateWithFlags(&e_end, cudaEventBlockingSync));
  }
  ~StreamCtx() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (e_end) cudaEventDestroy(e_end);
    if (s) cudaStreamDestroy(s);
  }
  void sync() { SSB_CUDA(cudaStreamSynchronize(s)); }
};

int num_sms();

}  // namespace ssb

// ---- opaque handle bodies --------------------------------------------------

// Device-resident normalised edge set (the reference Graph, graph.hpp:31-51):
// m keys (u << bits) | v with u < v, sorted ascending, unique.
struct ssb_edges {
  int64_t n = 0;
  int64_t m = 0;
  int bits = 1;  // bits per endpoint in a key
  ssb::DevBuf<uint64_t> keys;
  std::shared_ptr<void> csr;  // device CSR (validate.cu), built on first use
  ssb::StreamCtx sc;
};

// Work unit of the C=32 engine: one SlimChunk segment (bfs.hpp:58-66).
struct ssb_unit {
  int32_t chunk;
  int32_t col_begin;
  int32_t col_len;
  int32_t split;  // index of the split-chunk scratch slot, -1 = whole chunk
};

struct ssb_bfs_plan {  // cached per slimchunk_len
  int64_t L = -1;
  int64_t Lu = -1;  // columns per work unit: min(L, balance cap)
  int64_t cap_auto = 0;               // balance cap of the segments below
  int64_t budget_auto = 512;          // task budget (columns) of the same segments
  std::vector<int64_t> cap_segs;
  int64_t n_units = 0;
  int64_t n_tasks = 0;
  int64_t n_split = 0;
  int64_t empty_chunks = 0;  // chunks with cl == 0 (no unit)
  std::vector<int64_t> segs;  // chunk segments the plan covers (a shard, or all)
  bool built = false;
  ssb::DevBuf<ssb_unit> units;
  ssb::DevBuf<int32_t> task_begin;    // n_tasks + 1
  ssb::DevBuf<int32_t> split_units;   // units per split chunk
  ssb::DevBuf<uint32_t> split_hit;    // n_split
  ssb::DevBuf<int32_t> split_best;    // n_split * 32
  ssb::DevBuf<uint32_t> split_count;  // n_split
  ssb::DevBuf<int32_t> tlist;         // 2 * n_tasks: active task lists (ping-pong)
  ssb::DevBuf<uint8_t> tskip;         // n_tasks: all units skipped last time
};

// Device-resident SlimSellRepr (repr.hpp:33-55) plus the BFS workspace.
struct ssb_graph {
  int64_t C = 1, sigma = 1, n = 0, n_padded = 0, n_chunks = 0, nonzeros = 0;
  int64_t n_cells = 0, padding = 0, max_cl = 0;  // n_cells: cells held (the built range)
  int64_t total_cells = 0;                 // Σ C·cl over the whole layout
  // chunk segments whose cells this handle holds, [b0, e0, b1, e1, ...]
  // ascending and disjoint; empty = the whole layout
  std::vector<int64_t> segs;
  ssb::DevBuf<uint8_t> held;               // per chunk: cells held (partial handles)
  int64_t build_passes = 0;                // arc sort passes the builder needed
  bool partial() const { return !segs.empty(); }
  // every chunk of [cb, ce) is held
  bool holds(int64_t cb, int64_t ce) const {
    if (cb >= ce || !partial()) return true;
    for (size_t i = 0; i + 1 < segs.size(); i += 2)
      if (cb >= segs[i] && ce <= segs[i + 1]) return true;
    return false;
  }
  bool holds_segments(const std::vector<int64_t>& o) const {
    for (size_t i = 0; i + 1 < o.size(); i += 2) {
      if (o[i] >= o[i + 1]) continue;
      bool in = false;
      for (size_t j = 0; !in && j + 1 < segs.size(); j += 2) in = o[i] >= segs[j] && o[i + 1] <= segs[j + 1];
      if (partial() && !in) return false;
    }
    return true;
  }
  void need_full(const char* what) const {
    if (partial()) ssb::fail(SSB_EINVAL, std::string(what) + " needs the whole layout (this handle holds "
                                          "the cells of " + std::to_string(segs.size() / 2) + " chunk segment(s) only)");
  }
  ssb::DevBuf<int32_t> col;       // n_cells, -1 = padding cell
  ssb::DevBuf<int64_t> cs;        // n_chunks + 1 (cs[n_chunks] = n_cells)
  ssb::DevBuf<int32_t> cl;        // n_chunks
  ssb::DevBuf<int32_t> perm;      // n: position -> original id
  ssb::DevBuf<int32_t> inv_perm;  // n: original id -> position
  ssb::DevBuf<int32_t> deg;       // n_padded: row length per position
  std::vector<int32_t> cl_host;   // for host-side work planning

  // BFS workspace (allocated on first use).
  ssb::DevBuf<uint32_t> bits;     // visited | F0 | F1 | S0 | S1 | S2
  ssb::DevBuf<int32_t> level;     // n_padded, valid where visited
  ssb::DevBuf<int32_t> parent;    // n_padded, sel-max parent position
  ssb::DevBuf<int64_t> dstats;    // per-iteration counters
  ssb::DevBuf<uint32_t> dctrl;    // task counters + control words
  ssb::DevBuf<uint8_t> gbytes;    // generic engine: skip flags / frontier bytes
  ssb::DevBuf<int64_t> stage;     // fetch staging for pageable host outputs (2n)
  ssb::DevBuf<int> flag;          // small device flag
  ssb_bfs_plan plan;

  // Last BFS (device-resident result).
  int64_t last_root = -1;
  int32_t last_variant = -1;
  int32_t last_compat = 1;
  int64_t last_iterations = 0;
  bool last_valid = false;
  double last_kernel_ms = 0;  // CUDA-event time of the main BFS kernel launches
  int64_t last_launches = 0;  // kernels launched by the last BFS
  int64_t last_swept = 0;     // columns the last BFS actually streamed (Σ over iterations)
  std::shared_ptr<void> shard;  // state of a sharded (multi-GPU) BFS in progress
  ssb::DevBuf<uint8_t> wire;       // result fetch: uint8 levels | int32 parents (original ids)
  std::shared_ptr<void> wire_host; // ... its pinned host copy and chunk events (bfs.cu)
  ssb::DevBuf<uint32_t> p2p_win;  // fused multi-GPU BFS: the peer-mapped frontier window
  std::shared_ptr<void> p2p;      // ... and its peer table (bfs.cu)
  std::shared_ptr<void> geom;   // cached shared-memory image geometry (bfs.cu)
  std::shared_ptr<void> spmv_plan;  // work units of the last spmv_step chunk range (spmv.cu)
  std::shared_ptr<void> gen_plan;   // work units + per-row hit slots of the C != 32 engine (bfs.cu)
  std::shared_ptr<void> rec_host;   // pinned landing buffer of the launch records (bfs.cu)

  ssb::StreamCtx sc;
};

// Single-process multi-device context: one rank per entry
// of devs (all distinct: peer-mapped fused exchange; all equal: the ranks
// emulated as one cooperative launch on that device).
struct ssb_ctx {
  std::vector<int> devs;
  bool group = false;
};

// A layout sharded over a context's ranks: rank i holds the cells of its
// round-robin chunk segments on devs[i].
struct ssb_sharded {
  ssb_ctx* ctx = nullptr;
  int64_t n = 0;
  std::vector<std::vector<int64_t>> segs;  // per rank: [b0, e0, b1, e1, ...]
  std::vector<std::unique_ptr<ssb_graph>> g;
  ~ssb_sharded() {
    int prev = 0;
    cudaGetDevice(&prev);
    for (size_t i = 0; i < g.size(); ++i) {  // free each shard on its own device
      if (ctx && i < ctx->devs.size()) cudaSetDevice(ctx->devs[i]);
      g[i].reset();
    }
    cudaSetDevice(prev);
  }
};

namespace ssb {
// bfs.cu: the context
ssb_ctx* ctx_create(int n_ranks, const int* device_ids);
ssb_sharded* ctx_build(ssb_ctx& c, const ssb_edges& e, int64_t C, int64_t sigma, int segments_per_rank);
int sharded_bfs(ssb_sharded& sh, int64_t root, const ssb_bfs_options& o, int64_t* dist, int64_t* parent,
                int64_t* parent_len, ssb_iter_stats* stats, int64_t stats_cap, int64_t* iterations,
                double* device_ms);
std::vector<std::vector<int64_t>> partition_segments_host(const std::vector<int32_t>& cl, int64_t C, int world,
                                                          int k);
// builder.cu
ssb_graph* build_from_edges(const ssb_edges& e, int64_t C, int64_t sigma);
ssb_graph* build_range_from_edges(const ssb_edges& e, int64_t C, int64_t sigma,
                                  const std::vector<int64_t>& segs);
// segments: [b0, e0, b1, e1, ...] chunk bounds; checked, sorted, merged
std::vector<int64_t> normalize_segments(const int64_t* bounds, int64_t nseg, int64_t n_chunks);
ssb_graph* graph_from_host_layout(int64_t n, int64_t C, int64_t sigma, int64_t nonzeros,
                                  const int64_t* col, int64_t n_cells, const int64_t* cs,
                                  const int64_t* cl, int64_t n_chunks, const int64_t* perm);
// generator.cu
ssb_edges* edges_from_pairs(const int64_t* uv, int64_t count, int64_t n);
ssb_edges* gen_kronecker(int64_t scale, int64_t ef, uint64_t seed, const double init[4]);
ssb_edges* gen_erdos_renyi(int64_t n, double p, uint64_t seed);
void edges_to_csr(const ssb_edges& e, int64_t* row, int64_t* col);
// spmv.cu
void spmv_step(const ssb_graph& g, int variant, const int64_t* x_prev, int64_t* out,
               int64_t chunk_begin, int64_t chunk_end);
void spmv_step_device(const ssb_graph& g, int variant, const int64_t* x_prev, int64_t* out,
                      int64_t chunk_begin, int64_t chunk_end, double* device_ms);
void spmv_segment(const ssb_graph& g, int variant, const int64_t* x_prev, int64_t* acc, int64_t chunk,
                  int64_t col_begin, int64_t col_len);
// bfs.cu
int bfs_run(ssb_graph& g, int64_t root, const ssb_bfs_options& o, ssb_iter_stats* stats,
            int64_t stats_cap, int64_t* iterations, double* device_ms);
void bfs_fetch(ssb_graph& g, int want_parents, int64_t* dist, int64_t* parent,
               int64_t* parent_len);
int64_t bfs_batch(ssb_graph& g, const int64_t* roots, int64_t nroots, const ssb_bfs_options& o,
                  int64_t* const* dist, int64_t* const* parent, int64_t* iterations);
int64_t bfs_edges_traversed(ssb_graph& g);
void shard_begin(ssb_graph& g, int64_t root, const ssb_bfs_options& o, int64_t cb, int64_t ce);
void shard_step(ssb_graph& g, ssb_iter_stats* local, uint32_t* owned_words);
void shard_exchange(ssb_graph& g, const uint32_t* frontier_words, int64_t newly_total);
void shard_fetch(ssb_graph& g, int want_parents, int64_t* dist, int64_t* parent);
void shard_begin_async(ssb_graph& g, int64_t root, const ssb_bfs_options& o, int64_t cb, int64_t ce);
void shard_step_async(ssb_graph& g, uint32_t* owned_words);
void shard_exchange_async(ssb_graph& g, const uint32_t* frontier_words);
int64_t shard_front(ssb_graph& g, int64_t k);
void shard_finish(ssb_graph& g, int64_t iterations, ssb_iter_stats* out, int64_t cap, double* device_ms);
void p2p_window(ssb_graph& g, void* ipc_handle, int64_t* bytes);
void p2p_attach(ssb_graph& g, int rank, int world, const void* handles, const int64_t* bounds,
                int64_t nseg);
int bfs_p2p(ssb_graph* const* gs, int n_local, const int64_t* bounds, const int64_t* seg_counts,
            int64_t root, const ssb_bfs_options& o, ssb_iter_stats* stats, int64_t stats_cap,
            int64_t* iterations, double* device_ms);
// hostio.cpp: widen the uint8 / int32 wire chunks into int64 host arrays on a
// persistent host thread pool, chunk c once ready[c] has completed
// (packed_bits > 0: `par` holds packed words level << packed_bits | parent id,
// all ones = unreached, and `lev` is unused)
void widen_chunks(const std::vector<int64_t>& bounds, const std::vector<cudaEvent_t>& ready,
                  const uint8_t* lev, const int32_t* par, int64_t* dist, int64_t* parent,
                  int packed_bits = 0);
int host_threads();
// ingest.cu
void parse_edge_list(std::string_view text, int directive, std::vector<int64_t>& uv, int64_t& n);
void parse_matrix_market(std::string_view text, std::vector<int64_t>& uv, int64_t& n);
// validate.cu
int64_t bfs_traditional(ssb_edges& e, int64_t root, int64_t* dist, int64_t* parent,
                        std::vector<ssb_iter_stats>& per_iter);
int64_t validate_bfs(ssb_edges& e, int64_t root, const int64_t* dist, const int64_t* parent,
                     int flags, std::string& report_text, const ssb_graph* layout = nullptr);
}  // namespace ssb
