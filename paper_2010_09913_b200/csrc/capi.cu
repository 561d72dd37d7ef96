// extern "C" entry points of libslimsell_b200.so (include/slimsell_b200.h).
// Each maps C++ exceptions to SSB_* status codes and a thread-local message,
// mirroring the reference's exception contract.
#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "ssb_internal.cuh"

namespace {
thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return SSB_OK;
  } catch (const ssb::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_last_error = std::string("host allocation failed: ") + e.what();
    return SSB_ENOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SSB_ECUDA;
  }
}

void need(const void* p, const char* what) {
  if (p == nullptr) ssb::fail(SSB_EINVAL, std::string(what) + " is NULL");
}
}  // namespace

extern "C" {

const char* ssb_last_error(void) { return g_last_error.c_str(); }

int ssb_abi_version(void) { return SSB_ABI_VERSION; }

int ssb_set_device(int device) {
  return guarded([&] { SSB_CUDA(cudaSetDevice(device)); });
}

int ssb_edges_from_pairs(const int64_t* uv, int64_t count, int64_t n, ssb_edges** out) {
  return guarded([&] {
    need(out, "out");
    if (count > 0) need(uv, "uv");
    *out = ssb::edges_from_pairs(uv, count, n);
  });
}

int ssb_gen_kronecker(int64_t scale, int64_t edgefactor, uint64_t seed,
                      const double initiator[4], ssb_edges** out) {
  return guarded([&] {
    need(out, "out");
    const double def[4] = {0.57, 0.19, 0.19, 0.05};
    *out = ssb::gen_kronecker(scale, edgefactor, seed, initiator ? initiator : def);
  });
}

int ssb_gen_erdos_renyi(int64_t n, double p, uint64_t seed, ssb_edges** out) {
  return guarded([&] {
    need(out, "out");
    *out = ssb::gen_erdos_renyi(n, p, seed);
  });
}

namespace {
int64_t* copy_out(const std::vector<int64_t>& v) {
  auto* p = static_cast<int64_t*>(std::malloc(std::max<size_t>(v.size(), 1) * sizeof(int64_t)));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(int64_t));
  return p;
}
}  // namespace

int ssb_parse_edge_list(const char* text, int64_t len, int directive, int64_t** uv,
                        int64_t* count, int64_t* n) {
  return guarded([&] {
    need(uv, "uv");
    need(count, "count");
    need(n, "n");
    if (len > 0) need(text, "text");
    std::vector<int64_t> v;
    ssb::parse_edge_list(std::string_view(text ? text : "", size_t(std::max<int64_t>(len, 0))),
                         directive, v, *n);
    *uv = copy_out(v);
    *count = int64_t(v.size() / 2);
  });
}

int ssb_parse_matrix_market(const char* text, int64_t len, int64_t** uv, int64_t* count,
                            int64_t* n) {
  return guarded([&] {
    need(uv, "uv");
    need(count, "count");
    need(n, "n");
    if (len > 0) need(text, "text");
    std::vector<int64_t> v;
    ssb::parse_matrix_market(std::string_view(text ? text : "", size_t(std::max<int64_t>(len, 0))),
                             v, *n);
    *uv = copy_out(v);
    *count = int64_t(v.size() / 2);
  });
}

void ssb_free(void* p) { std::free(p); }

int ssb_edges_from_edge_list(const char* text, int64_t len, int directive, ssb_edges** out) {
  return guarded([&] {
    need(out, "out");
    if (len > 0) need(text, "text");
    std::vector<int64_t> v;
    int64_t n = -1;
    ssb::parse_edge_list(std::string_view(text ? text : "", size_t(std::max<int64_t>(len, 0))),
                         directive, v, n);
    *out = ssb::edges_from_pairs(v.data(), int64_t(v.size() / 2), n);
  });
}

int ssb_edges_from_matrix_market(const char* text, int64_t len, ssb_edges** out) {
  return guarded([&] {
    need(out, "out");
    if (len > 0) need(text, "text");
    std::vector<int64_t> v;
    int64_t n = 0;
    ssb::parse_matrix_market(std::string_view(text ? text : "", size_t(std::max<int64_t>(len, 0))),
                             v, n);
    *out = ssb::edges_from_pairs(v.data(), int64_t(v.size() / 2), n);
  });
}

int ssb_edges_info(const ssb_edges* e, int64_t* n, int64_t* m) {
  return guarded([&] {
    need(e, "edges");
    if (n) *n = e->n;
    if (m) *m = e->m;
  });
}

int ssb_edges_export(const ssb_edges* e, int64_t* uv) {
  return guarded([&] {
    need(e, "edges");
    need(uv, "uv");
    if (e->m == 0) return;
    ssb_edges& me = const_cast<ssb_edges&>(*e);
    std::vector<uint64_t> keys(e->m);
    SSB_CUDA(cudaMemcpyAsync(keys.data(), e->keys.p, 8 * e->m, cudaMemcpyDeviceToHost, me.sc.s));
    me.sc.sync();
    const uint64_t mask = (uint64_t{1} << e->bits) - 1;
    for (int64_t i = 0; i < e->m; ++i) {
      uv[2 * i] = int64_t(keys[i] >> e->bits);
      uv[2 * i + 1] = int64_t(keys[i] & mask);
    }
  });
}

int ssb_to_csr(const ssb_edges* e, int64_t* row, int64_t* col) {
  return guarded([&] {
    need(e, "edges");
    need(row, "row");
    if (e->m) need(col, "col");
    ssb::edges_to_csr(*e, row, col);
  });
}

void ssb_edges_destroy(ssb_edges* e) { delete e; }

int ssb_build_slimsell_range(const ssb_edges* e, int64_t C, int64_t sigma, int64_t chunk_begin,
                             int64_t chunk_end, ssb_graph** out) {
  return guarded([&] {
    need(e, "edges");
    need(out, "out");
    if (C <= 0) ssb::fail(SSB_EINVAL, "chunk height must be positive");
    const int64_t nc = (e->n + C - 1) / C;
    const int64_t b[2] = {chunk_begin, chunk_end < 0 ? nc : chunk_end};
    if (b[0] < 0 || b[0] > b[1] || b[1] > nc) ssb::fail(SSB_EINVAL, "chunk range out of bounds");
    // an empty range holds no cells (metadata only); [0, n_chunks) is the whole layout
    std::vector<int64_t> segs = {b[0], b[1]};
    if (b[0] == b[1]) segs = {0, 0};
    *out = ssb::build_range_from_edges(*e, C, sigma, segs);
  });
}

int ssb_build_slimsell_segments(const ssb_edges* e, int64_t C, int64_t sigma, const int64_t* bounds,
                                int64_t nseg, ssb_graph** out) {
  return guarded([&] {
    need(e, "edges");
    need(out, "out");
    if (C <= 0) ssb::fail(SSB_EINVAL, "chunk height must be positive");
    if (nseg < 1) ssb::fail(SSB_EINVAL, "need at least one segment");
    need(bounds, "bounds");
    std::vector<int64_t> segs(bounds, bounds + 2 * nseg);
    ssb::normalize_segments(segs.data(), nseg, (e->n + C - 1) / C);  // validates
    bool empty = true;
    for (int64_t i = 0; i < nseg; ++i) empty = empty && segs[size_t(2 * i)] == segs[size_t(2 * i + 1)];
    if (empty) segs = {0, 0};
    *out = ssb::build_range_from_edges(*e, C, sigma, segs);
  });
}

int ssb_build_slimsell(const ssb_edges* e, int64_t C, int64_t sigma, ssb_graph** out) {
  return guarded([&] {
    need(e, "edges");
    need(out, "out");
    *out = ssb::build_from_edges(*e, C, sigma);
  });
}

int ssb_graph_from_layout(int64_t n, int64_t C, int64_t sigma, int64_t nonzeros,
                          const int64_t* col, int64_t n_cells, const int64_t* cs,
                          const int64_t* cl, int64_t n_chunks, const int64_t* perm,
                          ssb_graph** out) {
  return guarded([&] {
    need(out, "out");
    if (n_cells) need(col, "col");
    if (n_chunks) { need(cs, "cs"); need(cl, "cl"); }
    if (n) need(perm, "perm");
    *out = ssb::graph_from_host_layout(n, C, sigma, nonzeros, col, n_cells, cs, cl, n_chunks, perm);
  });
}

int ssb_graph_info(const ssb_graph* g, ssb_layout_info* info) {
  return guarded([&] {
    need(g, "graph");
    need(info, "info");
    info->C = g->C;
    info->sigma = g->sigma;
    info->n = g->n;
    info->n_padded = g->n_padded;
    info->n_chunks = g->n_chunks;
    info->nonzeros = g->nonzeros;
    info->n_cells = g->total_cells;
    info->padding = g->padding;
    info->max_chunk_len = g->max_cl;
    info->range_begin = g->partial() ? g->segs.front() : 0;
    info->range_end = g->partial() ? g->segs.back() : g->n_chunks;
    info->range_cells = g->n_cells;
    info->range_segments = g->partial() ? int64_t(g->segs.size() / 2) : 1;
  });
}

int ssb_graph_export(const ssb_graph* cg, int64_t* col, int64_t* cs, int64_t* cl, int64_t* perm,
                     int64_t* inv_perm) {
  return guarded([&] {
    need(cg, "graph");
    ssb_graph& g = const_cast<ssb_graph&>(*cg);
    if (col || cs) g.need_full("ssb_graph_export of col / cs");
    cudaStream_t s = g.sc.s;
    auto widen32 = [&](const int32_t* src, int64_t count, int64_t* dst) {
      if (!dst || count == 0) return;
      const int64_t slab = int64_t{1} << 26;
      std::vector<int32_t> tmp(std::min(slab, count));
      for (int64_t off = 0; off < count; off += slab) {
        const int64_t c = std::min(slab, count - off);
        SSB_CUDA(cudaMemcpyAsync(tmp.data(), src + off, 4 * c, cudaMemcpyDeviceToHost, s));
        g.sc.sync();
        for (int64_t i = 0; i < c; ++i) dst[off + i] = tmp[i];
      }
    };
    widen32(g.col.p, g.n_cells, col);
    if (cs && g.n_chunks) {
      SSB_CUDA(cudaMemcpyAsync(cs, g.cs.p, 8 * g.n_chunks, cudaMemcpyDeviceToHost, s));
      g.sc.sync();
    }
    widen32(g.cl.p, g.n_chunks, cl);
    widen32(g.perm.p, g.n, perm);
    widen32(g.inv_perm.p, g.n, inv_perm);
  });
}

int ssb_graph_degrees(const ssb_graph* cg, int64_t* deg) {
  return guarded([&] {
    need(cg, "graph");
    need(deg, "deg");
    ssb_graph& g = const_cast<ssb_graph&>(*cg);
    if (g.n == 0) return;
    std::vector<int32_t> d(g.n), p(g.n);
    SSB_CUDA(cudaMemcpyAsync(d.data(), g.deg.p, 4 * g.n, cudaMemcpyDeviceToHost, g.sc.s));
    SSB_CUDA(cudaMemcpyAsync(p.data(), g.perm.p, 4 * g.n, cudaMemcpyDeviceToHost, g.sc.s));
    g.sc.sync();
    for (int64_t i = 0; i < g.n; ++i) deg[p[i]] = d[i];
  });
}

int ssb_graph_export_col32(const ssb_graph* cg, int32_t* col) {
  return guarded([&] {
    need(cg, "graph");
    need(col, "col");
    ssb_graph& g = const_cast<ssb_graph&>(*cg);
    if (g.n_cells) {
      SSB_CUDA(cudaMemcpyAsync(col, g.col.p, 4 * g.n_cells, cudaMemcpyDeviceToHost, g.sc.s));
      g.sc.sync();
    }
  });
}

void ssb_graph_destroy(ssb_graph* g) { delete g; }

int ssb_spmv_step(const ssb_graph* g, int variant, const int64_t* x_prev, int64_t* out,
                  int64_t chunk_begin, int64_t chunk_end) {
  return guarded([&] {
    need(g, "graph");
    need(x_prev, "x_prev");
    need(out, "out");
    ssb::spmv_step(*g, variant, x_prev, out, chunk_begin, chunk_end);
  });
}

int ssb_spmv_step_device(const ssb_graph* g, int variant, const int64_t* x_prev, int64_t* out,
                         int64_t chunk_begin, int64_t chunk_end, double* device_ms) {
  return guarded([&] {
    need(g, "graph");
    need(x_prev, "x_prev");
    need(out, "out");
    ssb::spmv_step_device(*g, variant, x_prev, out, chunk_begin, chunk_end, device_ms);
  });
}

int ssb_spmv_segment(const ssb_graph* g, int variant, const int64_t* x_prev, int64_t* acc, int64_t chunk,
                     int64_t col_begin, int64_t col_len) {
  return guarded([&] {
    need(g, "graph");
    need(x_prev, "x_prev");
    need(acc, "acc");
    ssb::spmv_segment(*g, variant, x_prev, acc, chunk, col_begin, col_len);
  });
}

int ssb_bfs_run(ssb_graph* g, int64_t root, const ssb_bfs_options* opts, ssb_iter_stats* stats,
                int64_t stats_cap, int64_t* iterations, double* device_ms) {
  int rc = SSB_OK;
  const int st = guarded([&] {
    need(g, "graph");
    need(opts, "opts");
    rc = ssb::bfs_run(*g, root, *opts, stats, stats_cap, iterations, device_ms);
  });
  if (st != SSB_OK) return st;
  if (rc == SSB_ECAP) g_last_error = "iteration cap reached before fixed point";
  return rc;
}

int ssb_bfs_fetch(ssb_graph* g, int want_parents, int64_t* dist, int64_t* parent,
                  int64_t* parent_len) {
  return guarded([&] {
    need(g, "graph");
    ssb::bfs_fetch(*g, want_parents, dist, parent, parent_len);
  });
}

int ssb_bfs_spmv(ssb_graph* g, int64_t root, const ssb_bfs_options* opts, int64_t* dist,
                 int64_t* parent, int64_t* parent_len, ssb_iter_stats* stats,
                 int64_t stats_cap, int64_t* iterations) {
  int rc = ssb_bfs_run(g, root, opts, stats, stats_cap, iterations, nullptr);
  if (rc != SSB_OK && rc != SSB_ECAP) return rc;
  const std::string cap_msg = g_last_error;
  // bfs.cpp:86-90: on the cap the partial result carries dist, no parents.
  const int want = rc == SSB_OK && opts->want_parents && parent != nullptr;
  const int f = guarded([&] {
    need(dist, "dist");
    ssb::bfs_fetch(*g, want, dist, want ? parent : nullptr, parent_len);
  });
  if (f != SSB_OK) return f;
  if (rc == SSB_ECAP) g_last_error = cap_msg;
  return rc;
}

int ssb_bfs_spmv_batch(ssb_graph* g, const int64_t* roots, int64_t nroots, const ssb_bfs_options* opts,
                       int64_t* const* dist, int64_t* const* parent, int64_t* iterations,
                       int64_t* capped_at) {
  int64_t cap_i = -1;
  const int st = guarded([&] {
    need(g, "graph");
    need(opts, "opts");
    if (nroots < 0) ssb::fail(SSB_EINVAL, "nroots < 0");
    if (nroots > 0) need(roots, "roots");
    need(dist, "dist");
    for (int64_t i = 0; i < nroots; ++i) {
      need(dist[i], "dist[i]");
      if (roots[i] < 0 || roots[i] >= g->n)
        ssb::fail(SSB_ERANGE, "root " + std::to_string(roots[i]) + " outside [0, " + std::to_string(g->n) + ")");
    }
    cap_i = ssb::bfs_batch(*g, roots, nroots, *opts, dist, parent, iterations);
  });
  if (capped_at) *capped_at = cap_i;
  if (st != SSB_OK) return st;
  if (cap_i >= 0) {
    g_last_error = "iteration cap reached before fixed point (root index " + std::to_string(cap_i) + ")";
    return SSB_ECAP;
  }
  return SSB_OK;
}

int ssb_bfs_last_timing(ssb_graph* g, double* kernel_ms, int64_t* launches) {
  return guarded([&] {
    need(g, "graph");
    if (!g->last_valid && !g->shard) ssb::fail(SSB_EINVAL, "no BFS result on this graph");
    if (kernel_ms) *kernel_ms = g->last_kernel_ms;
    if (launches) *launches = g->last_launches;
  });
}

int ssb_bfs_columns_swept(ssb_graph* g, int64_t* swept) {
  return guarded([&] {
    need(g, "graph");
    need(swept, "swept");
    if (!g->last_valid) ssb::fail(SSB_EINVAL, "no BFS result on this graph");
    *swept = g->last_swept;
  });
}

int ssb_bfs_traditional(ssb_edges* e, int64_t root, int64_t* dist, int64_t* parent,
                        ssb_iter_stats* stats, int64_t stats_cap, int64_t* iterations) {
  return guarded([&] {
    need(e, "edges");
    need(dist, "dist");
    std::vector<ssb_iter_stats> st;
    const int64_t k = ssb::bfs_traditional(*e, root, dist, parent, st);
    if (iterations) *iterations = k;
    if (stats)
      for (int64_t i = 0; i < std::min<int64_t>(stats_cap, int64_t(st.size())); ++i) stats[i] = st[size_t(i)];
  });
}

int ssb_validate_bfs(ssb_edges* e, int64_t root, const int64_t* dist, const int64_t* parent,
                     int flags, int64_t* violations, char* report, int64_t report_cap) {
  return ssb_validate_bfs_exact(e, nullptr, root, dist, parent, flags,
                                violations, report, report_cap);
}

int ssb_validate_bfs_exact(ssb_edges* e, const ssb_graph* layout, int64_t root, const int64_t* dist,
                           const int64_t* parent, int flags, int64_t* violations, char* report,
                           int64_t report_cap) {
  return guarded([&] {
    need(e, "edges");
    need(dist, "dist");
    need(violations, "violations");
    std::string text;
    *violations = ssb::validate_bfs(*e, root, dist, parent, flags, text, layout);
    if (report && report_cap > 0) {
      const size_t k = std::min<size_t>(text.size(), size_t(report_cap - 1));
      std::memcpy(report, text.data(), k);
      report[k] = 0;
    }
  });
}

int ssb_bfs_shard_begin(ssb_graph* g, int64_t root, const ssb_bfs_options* opts,
                        int64_t chunk_begin, int64_t chunk_end) {
  return guarded([&] {
    need(g, "graph");
    need(opts, "opts");
    ssb::shard_begin(*g, root, *opts, chunk_begin, chunk_end);
  });
}

int ssb_bfs_shard_step(ssb_graph* g, ssb_iter_stats* local, uint32_t* owned_words) {
  return guarded([&] {
    need(g, "graph");
    ssb::shard_step(*g, local, owned_words);
  });
}

int ssb_bfs_shard_exchange(ssb_graph* g, const uint32_t* frontier_words, int64_t newly_total) {
  return guarded([&] {
    need(g, "graph");
    ssb::shard_exchange(*g, frontier_words, newly_total);
  });
}

int ssb_graph_stream(ssb_graph* g, void** stream) {
  return guarded([&] {
    need(g, "graph");
    need(stream, "stream");
    *stream = static_cast<void*>(g->sc.s);
  });
}

int ssb_bfs_shard_begin_async(ssb_graph* g, int64_t root, const ssb_bfs_options* opts,
                              int64_t chunk_begin, int64_t chunk_end) {
  return guarded([&] {
    need(g, "graph");
    need(opts, "opts");
    ssb::shard_begin_async(*g, root, *opts, chunk_begin, chunk_end);
  });
}

int ssb_bfs_shard_step_async(ssb_graph* g, uint32_t* owned_words) {
  return guarded([&] {
    need(g, "graph");
    ssb::shard_step_async(*g, owned_words);
  });
}

int ssb_bfs_shard_exchange_async(ssb_graph* g, const uint32_t* frontier_words) {
  return guarded([&] {
    need(g, "graph");
    ssb::shard_exchange_async(*g, frontier_words);
  });
}

int ssb_bfs_shard_front(ssb_graph* g, int64_t k, int64_t* front) {
  return guarded([&] {
    need(g, "graph");
    need(front, "front");
    *front = ssb::shard_front(*g, k);
  });
}

int ssb_bfs_shard_finish(ssb_graph* g, int64_t iterations, ssb_iter_stats* stats, int64_t stats_cap,
                         double* device_ms) {
  return guarded([&] {
    need(g, "graph");
    if (stats_cap > 0) need(stats, "stats");
    ssb::shard_finish(*g, iterations, stats, stats_cap, device_ms);
  });
}

int ssb_bfs_shard_fetch(ssb_graph* g, int want_parents, int64_t* dist, int64_t* parent) {
  return guarded([&] {
    need(g, "graph");
    ssb::shard_fetch(*g, want_parents, dist, parent);
  });
}

int ssb_p2p_window(ssb_graph* g, void* ipc_handle, int64_t* window_bytes) {
  return guarded([&] {
    need(g, "graph");
    ssb::p2p_window(*g, ipc_handle, window_bytes);
  });
}

int ssb_p2p_attach(ssb_graph* g, int rank, int world, const void* ipc_handles, int64_t chunk_begin,
                   int64_t chunk_end) {
  return guarded([&] {
    need(g, "graph");
    const int64_t b[2] = {chunk_begin, chunk_end};
    ssb::p2p_attach(*g, rank, world, ipc_handles, b, 1);
  });
}

int ssb_p2p_attach_segments(ssb_graph* g, int rank, int world, const void* ipc_handles,
                            const int64_t* bounds, int64_t nseg) {
  return guarded([&] {
    need(g, "graph");
    if (nseg > 0) need(bounds, "bounds");
    ssb::p2p_attach(*g, rank, world, ipc_handles, bounds, nseg);
  });
}

int ssb_bfs_p2p(ssb_graph* g, int64_t root, const ssb_bfs_options* opts, ssb_iter_stats* stats,
                int64_t stats_cap, int64_t* iterations, double* device_ms) {
  int rc = SSB_OK;
  const int st = guarded([&] {
    need(g, "graph");
    need(opts, "opts");
    rc = ssb::bfs_p2p(&g, 1, nullptr, nullptr, root, *opts, stats, stats_cap, iterations, device_ms);
  });
  if (st != SSB_OK) return st;
  if (rc == SSB_ECAP) g_last_error = "iteration cap reached before fixed point";
  return rc;
}

int ssb_bfs_p2p_group(ssb_graph* const* shards, int world, const int64_t* bounds,
                      const int64_t* seg_counts, int64_t root, const ssb_bfs_options* opts,
                      ssb_iter_stats* stats, int64_t stats_cap, int64_t* iterations,
                      double* device_ms) {
  int rc = SSB_OK;
  const int st = guarded([&] {
    need(shards, "shards");
    need(bounds, "bounds");
    need(opts, "opts");
    if (world < 2) ssb::fail(SSB_EINVAL, "a group needs at least 2 shards");
    for (int i = 0; i < world; ++i) need(shards[i], "shard");
    rc = ssb::bfs_p2p(shards, world, bounds, seg_counts, root, *opts, stats, stats_cap, iterations,
                      device_ms);
  });
  if (st != SSB_OK) return st;
  if (rc == SSB_ECAP) g_last_error = "iteration cap reached before fixed point";
  return rc;
}

int ssb_bfs_edges_traversed(ssb_graph* g, int64_t* m_cc) {
  return guarded([&] {
    need(g, "graph");
    need(m_cc, "m_cc");
    *m_cc = ssb::bfs_edges_traversed(*g);
  });
}

int ssb_partition_segments(const int32_t* cl, int64_t n_chunks, int64_t C, int world, int k, int64_t* bounds) {
  return guarded([&] {
    need(bounds, "bounds");
    if (n_chunks > 0) need(cl, "cl");
    if (world < 1 || k < 1) ssb::fail(SSB_EINVAL, "world and k must be >= 1");
    const std::vector<int32_t> v(cl, cl + n_chunks);
    const auto segs = ssb::partition_segments_host(v, C, world, k);
    int64_t at = 0;
    for (const auto& s : segs)
      for (int64_t x : s) bounds[at++] = x;
  });
}

int ssb_ctx_create(int n_ranks, const int* device_ids, ssb_ctx** out) {
  return guarded([&] {
    need(out, "out");
    *out = ssb::ctx_create(n_ranks, device_ids);
  });
}

void ssb_ctx_destroy(ssb_ctx* c) { delete c; }

int ssb_ctx_build(ssb_ctx* c, const ssb_edges* e, int64_t C, int64_t sigma, int segments_per_rank,
                  ssb_sharded** out) {
  return guarded([&] {
    need(c, "ctx");
    need(e, "edges");
    need(out, "out");
    *out = ssb::ctx_build(*c, *e, C, sigma, segments_per_rank);
  });
}

int ssb_sharded_info(const ssb_sharded* sh, int* n_ranks, int64_t* n, int64_t* cells_per_rank,
                     int64_t* segments_per_rank) {
  return guarded([&] {
    need(sh, "sharded");
    if (n_ranks) *n_ranks = int(sh->g.size());
    if (n) *n = sh->n;
    for (size_t i = 0; i < sh->g.size(); ++i) {
      if (cells_per_rank) cells_per_rank[i] = sh->g[i]->n_cells;
      if (segments_per_rank) segments_per_rank[i] = int64_t(sh->segs[i].size() / 2);
    }
  });
}

int ssb_sharded_bfs(ssb_sharded* sh, int64_t root, const ssb_bfs_options* opts, int64_t* dist,
                    int64_t* parent, int64_t* parent_len, ssb_iter_stats* stats, int64_t stats_cap,
                    int64_t* iterations, double* device_ms) {
  int rc = SSB_OK;
  const int grc = guarded([&] {
    need(sh, "sharded");
    need(opts, "opts");
    rc = ssb::sharded_bfs(*sh, root, *opts, dist, parent, parent_len, stats, stats_cap, iterations, device_ms);
    if (rc == SSB_ECAP) g_last_error = "iteration cap reached before fixed point";
  });
  return grc != SSB_OK ? grc : rc;
}

void ssb_sharded_destroy(ssb_sharded* sh) { delete sh; }

}  // extern "C"
