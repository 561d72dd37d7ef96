// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A C-ABI shim over the UNMODIFIED reference library (compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libslimsell_ref.so). It lets the Python tests, the golden-vector
// generator and bench.py's reference arm call the reference's own public C++
// API through ctypes. Nothing here re-implements the reference: every entry
// point forwards to the reference function named in its comment.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "slimsell/bfs.hpp"
#include "slimsell/cli.hpp"
#include "slimsell/generator.hpp"
#include "slimsell/graph.hpp"
#include "slimsell/repr.hpp"
#include "slimsell/semiring.hpp"

using namespace slimsell;

namespace {
thread_local std::string g_err;

enum : int { kOk = 0, kEInval = 1, kERange = 2, kECap = 3, kEOther = 4, kEParse = 6 };

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kEInval;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return kERange;
  } catch (const ParseError& e) {
    g_err = e.what();
    return kEParse;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kEOther;
  }
}

struct RefGraph {
  Graph g;
  std::unique_ptr<CsrView> csr;
  const CsrView& get_csr() {
    if (!csr) csr = std::make_unique<CsrView>(to_csr(g));
    return *csr;
  }
};

Variant to_variant(int v) {
  if (v < 0 || v > 3) throw std::invalid_argument("bad variant");
  return static_cast<Variant>(v);
}

void copy_stats(const BfsResult& res, int64_t* stats, int64_t cap) {
  if (stats == nullptr) return;
  const int64_t n = std::min<int64_t>(cap, static_cast<int64_t>(res.per_iter.size()));
  for (int64_t i = 0; i < n; ++i) {
    const IterStats& s = res.per_iter[i];
    int64_t* o = stats + 7 * i;
    o[0] = s.iteration;
    o[1] = s.elapsed_ns;
    o[2] = s.chunks_processed;
    o[3] = s.chunks_skipped;
    o[4] = s.subchunks_processed;
    o[5] = s.columns_processed;
    o[6] = s.frontier_size;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// generator.hpp:55 gen_kronecker
int ref_gen_kronecker(int64_t scale, int64_t ef, uint64_t seed, const double* init,
                      void** out) {
  return guarded([&] {
    std::array<double, 4> a = {init[0], init[1], init[2], init[3]};
    *out = new RefGraph{gen_kronecker(scale, ef, seed, a), nullptr};
  });
}

// generator.hpp:50 gen_erdos_renyi
int ref_gen_erdos_renyi(int64_t n, double p, uint64_t seed, void** out) {
  return guarded([&] { *out = new RefGraph{gen_erdos_renyi(n, p, seed), nullptr}; });
}

// generator.hpp:62-64 gen_path / gen_clique / gen_star (kind 0/1/2)
int ref_gen_named(int kind, int64_t n, void** out) {
  return guarded([&] {
    Graph g = kind == 0 ? gen_path(n) : kind == 1 ? gen_clique(n) : gen_star(n);
    *out = new RefGraph{std::move(g), nullptr};
  });
}

// graph.hpp:36 Graph::from_pairs
int ref_graph_from_pairs(const int64_t* uv, int64_t count, int64_t n, void** out) {
  return guarded([&] {
    std::vector<std::pair<vid_t, vid_t>> pairs(count);
    for (int64_t i = 0; i < count; ++i) pairs[i] = {uv[2 * i], uv[2 * i + 1]};
    *out = new RefGraph{Graph::from_pairs(std::move(pairs), n), nullptr};
  });
}

int64_t ref_graph_n(void* g) { return static_cast<RefGraph*>(g)->g.num_vertices(); }
int64_t ref_graph_m(void* g) { return static_cast<RefGraph*>(g)->g.num_edges(); }

void ref_graph_edges(void* g, int64_t* uv) {
  const auto& e = static_cast<RefGraph*>(g)->g.edges();
  for (size_t i = 0; i < e.size(); ++i) {
    uv[2 * i] = e[i].first;
    uv[2 * i + 1] = e[i].second;
  }
}

// graph.hpp:71 to_csr
void ref_graph_csr(void* g, int64_t* row, int64_t* col) {
  const CsrView& c = static_cast<RefGraph*>(g)->get_csr();
  std::memcpy(row, c.row.data(), c.row.size() * sizeof(int64_t));
  std::memcpy(col, c.col.data(), c.col.size() * sizeof(int64_t));
}

void ref_graph_free(void* g) { delete static_cast<RefGraph*>(g); }

// FNV-1a-64 over little-endian int64 bytes (the golden-vector fingerprint),
// computed in place so an S26 graph / layout is hashed without a 17 GB copy.
static uint64_t fnv_i64(const int64_t* a, size_t count, uint64_t h = 0xcbf29ce484222325ULL) {
  const unsigned char* p = reinterpret_cast<const unsigned char*>(a);
  for (size_t i = 0; i < count * 8; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

// graph.hpp:42 Graph::edges() as the flattened (u, v) int64 pairs
uint64_t ref_graph_edges_fnv(void* g) {
  const auto& e = static_cast<RefGraph*>(g)->g.edges();
  static_assert(sizeof(e[0]) == 16, "pair<int64,int64>");
  return fnv_i64(reinterpret_cast<const int64_t*>(e.data()), e.size() * 2);
}

// deg[v] = |N(v)| over the normalised edge set (the CSR row lengths of
// graph.cpp:212-232, without materialising the CSR).
void ref_graph_degrees(void* g, int64_t* deg) {
  const auto& G = static_cast<RefGraph*>(g)->g;
  std::memset(deg, 0, sizeof(int64_t) * size_t(G.num_vertices()));
  for (auto [u, v] : G.edges()) {
    ++deg[u];
    ++deg[v];
  }
}

// Drops the cached CsrView (to_csr) to give its memory back between phases.
void ref_graph_drop_csr(void* g) { static_cast<RefGraph*>(g)->csr.reset(); }

// graph.hpp:55-59 from_edge_list / from_matrix_market
int ref_from_edge_list(const char* text, int64_t len, int directive, void** out) {
  return guarded([&] {
    *out = new RefGraph{from_edge_list(std::string_view(text, size_t(len)),
                                       directive ? InputDirective::reject_asymmetric
                                                 : InputDirective::symmetrize),
                        nullptr};
  });
}

int ref_from_matrix_market(const char* text, int64_t len, void** out) {
  return guarded([&] {
    *out = new RefGraph{from_matrix_market(std::string_view(text, size_t(len))), nullptr};
  });
}

// repr.hpp:66 build_slimsell
int ref_build_slimsell(void* g, int64_t C, int64_t sigma, void** out) {
  return guarded([&] {
    *out = new SlimSellRepr(build_slimsell(static_cast<RefGraph*>(g)->g, C, sigma));
  });
}

// Materialises a reference SlimSellRepr from arrays (e.g. a layout built on
// the device and exported), so the reference's stock bfs_spmv can run on it.
int ref_repr_from_arrays(int64_t n, int64_t C, int64_t sigma, int64_t nonzeros,
                         const int32_t* col, int64_t n_cells, const int64_t* cs,
                         const int64_t* cl, int64_t n_chunks, const int64_t* perm,
                         const int64_t* inv_perm, void** out) {
  return guarded([&] {
    auto r = std::make_unique<SlimSellRepr>();
    r->C = C;
    r->sigma = sigma;
    r->n = n;
    r->n_chunks = n_chunks;
    r->n_padded = n_chunks * C;
    r->nonzeros = nonzeros;
    r->col.assign(col, col + n_cells);
    r->cs.assign(cs, cs + n_chunks);
    r->cl.assign(cl, cl + n_chunks);
    r->perm.assign(perm, perm + n);
    r->inv_perm.assign(inv_perm, inv_perm + n);
    r->padding = n_cells - nonzeros;
    *out = r.release();
  });
}

// info = {C, sigma, n, n_padded, n_chunks, nonzeros, n_cells, padding}
void ref_repr_info(void* r, int64_t* info) {
  const auto* s = static_cast<SlimSellRepr*>(r);
  info[0] = s->C;
  info[1] = s->sigma;
  info[2] = s->n;
  info[3] = s->n_padded;
  info[4] = s->n_chunks;
  info[5] = s->nonzeros;
  info[6] = static_cast<int64_t>(s->col.size());
  info[7] = s->padding;
}

void ref_repr_export(void* r, int64_t* col, int64_t* cs, int64_t* cl, int64_t* perm,
                     int64_t* inv_perm) {
  const auto* s = static_cast<SlimSellRepr*>(r);
  if (col) std::memcpy(col, s->col.data(), s->col.size() * 8);
  if (cs) std::memcpy(cs, s->cs.data(), s->cs.size() * 8);
  if (cl) std::memcpy(cl, s->cl.data(), s->cl.size() * 8);
  if (perm) std::memcpy(perm, s->perm.data(), s->perm.size() * 8);
  if (inv_perm) std::memcpy(inv_perm, s->inv_perm.data(), s->inv_perm.size() * 8);
}

void ref_repr_free(void* r) { delete static_cast<SlimSellRepr*>(r); }

// FNV of one SlimSellRepr array in place: which = 0 col, 1 cs, 2 cl, 3 perm, 4 inv_perm.
uint64_t ref_repr_fnv(void* r, int which) {
  const auto* s = static_cast<SlimSellRepr*>(r);
  const std::vector<int64_t>* v[] = {&s->col, &s->cs, &s->cl, &s->perm, &s->inv_perm};
  if (which < 0 || which > 4) return 0;
  return fnv_i64(v[which]->data(), v[which]->size());
}

// repr.hpp:90 spmv_step (chunk range form); out must hold n_padded values
// (rows outside the range are left untouched, as in the reference).
int ref_spmv_step(void* r, int variant, const int64_t* x_prev, int64_t* out,
                  int64_t chunk_begin, int64_t chunk_end) {
  return guarded([&] {
    const auto* s = static_cast<SlimSellRepr*>(r);
    const size_t np = static_cast<size_t>(s->n_padded);
    spmv_step(*s, semiring(to_variant(variant)), std::span<const val_t>(x_prev, np),
              std::span<val_t>(out, np), chunk_begin, chunk_end);
  });
}

// repr.hpp:104-107 permute_in / permute_out
int ref_permute_in(void* r, const int64_t* v, int64_t fill, int64_t* out) {
  return guarded([&] {
    const auto* s = static_cast<SlimSellRepr*>(r);
    auto o = permute_in(std::span<const val_t>(v, s->n), *s, fill);
    std::memcpy(out, o.data(), o.size() * 8);
  });
}

int ref_permute_out(void* r, const int64_t* v, int64_t* out) {
  return guarded([&] {
    const auto* s = static_cast<SlimSellRepr*>(r);
    auto o = permute_out(std::span<const val_t>(v, s->n_padded), *s);
    std::memcpy(out, o.data(), o.size() * 8);
  });
}

// bfs.hpp:80 bfs_spmv. csr_graph may be null (then non-selmax parents are
// empty, as in the reference). stats holds 7 int64 per iteration:
// {iteration, elapsed_ns, chunks_processed, chunks_skipped,
//  subchunks_processed, columns_processed, frontier_size}.
// *parent_len receives res.parent.size(). workers <= 0 means all host threads.
int ref_bfs_spmv(void* r, int64_t root, int variant, int slimwork, int64_t L,
                 int schedule, int workers, int64_t max_iterations, int want_parents,
                 void* csr_graph, int64_t* dist, int64_t* parent, int64_t* parent_len,
                 int64_t* iterations, int64_t* stats, int64_t stats_cap) {
  const auto* s = static_cast<SlimSellRepr*>(r);
  BfsOptions o;
  int rc = guarded([&] { o.variant = to_variant(variant); });
  if (rc) return rc;
  o.slimwork = slimwork != 0;
  o.slimchunk_len = L;
  o.schedule = schedule == 0 ? Schedule::static_blocks : Schedule::dynamic_queue;
  o.workers = workers > 0 ? workers : static_cast<int>(std::thread::hardware_concurrency());
  o.max_iterations = max_iterations;
  o.want_parents = want_parents != 0;
  const CsrView* csr =
      csr_graph ? &static_cast<RefGraph*>(csr_graph)->get_csr() : nullptr;
  auto emit = [&](const BfsResult& res) {
    std::memcpy(dist, res.dist.data(), res.dist.size() * 8);
    if (parent && !res.parent.empty())
      std::memcpy(parent, res.parent.data(), res.parent.size() * 8);
    if (parent_len) *parent_len = static_cast<int64_t>(res.parent.size());
    if (iterations) *iterations = res.iterations;
    copy_stats(res, stats, stats_cap);
  };
  try {
    BfsResult res = bfs_spmv(*s, root, o, csr);
    emit(res);
    return kOk;
  } catch (const BfsCapError& e) {
    g_err = e.what();
    emit(e.partial());
    return kECap;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kEInval;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return kERange;
  } catch (const ParseError& e) {
    g_err = e.what();
    return kEParse;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kEOther;
  }
}

// bfs.hpp:85 bfs_traditional (the reference's own queue-BFS oracle)
int ref_bfs_traditional(void* g, int64_t root, int64_t* dist, int64_t* parent,
                        int64_t* iterations) {
  return guarded([&] {
    BfsResult res = bfs_traditional(static_cast<RefGraph*>(g)->get_csr(), root);
    std::memcpy(dist, res.dist.data(), res.dist.size() * 8);
    std::memcpy(parent, res.parent.data(), res.parent.size() * 8);
    *iterations = res.iterations;
  });
}

// As ref_bfs_traditional, plus elapsed_ns = sum of its IterStats.elapsed_ns
// (the timed part of the queue BFS, bfs.cpp:264-287).
int ref_bfs_traditional_timed(void* g, int64_t root, int64_t* dist, int64_t* parent,
                              int64_t* iterations, int64_t* elapsed_ns) {
  return guarded([&] {
    BfsResult res = bfs_traditional(static_cast<RefGraph*>(g)->get_csr(), root);
    if (dist) std::memcpy(dist, res.dist.data(), res.dist.size() * 8);
    if (parent) std::memcpy(parent, res.parent.data(), res.parent.size() * 8);
    *iterations = res.iterations;
    int64_t t = 0;
    for (const IterStats& s : res.per_iter) t += s.elapsed_ns;
    *elapsed_ns = t;
  });
}

// semiring.hpp:124 dp_transform
int ref_dp_transform(void* g, const int64_t* d, int64_t* parent) {
  return guarded([&] {
    const CsrView& c = static_cast<RefGraph*>(g)->get_csr();
    auto p = dp_transform(c, std::span<const val_t>(d, c.num_vertices()));
    std::memcpy(parent, p.data(), p.size() * 8);
  });
}

// cli.hpp:70 cmd_selftest; writes stdout+stderr text into buf.
int ref_selftest(uint64_t seed, int workers, char* buf, int64_t cap) {
  cli::SelftestConfig cfg;
  cfg.seed = seed;
  cfg.workers = workers;
  std::ostringstream out, err;
  const int rc = cli::cmd_selftest(cfg, out, err);
  const std::string text = out.str() + err.str();
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>(text.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, text.data(), n);
    buf[n] = '\0';
  }
  return rc;
}

}  // extern "C"
