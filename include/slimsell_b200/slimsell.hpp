// slimsell_b200/slimsell.hpp — header-only C++ façade of the B200 BFS-SpMV
// path with the reference library's spelling (namespace slimsell, the types
// and functions of /root/reference/proj/include/slimsell/{graph,generator,
// repr,semiring,bfs}.hpp). Every data-path call crosses the C-ABI in
// <slimsell_b200.h> into libslimsell_b200.so (sm_100a); link with
// -lslimsell_b200. There is no CPU fallback: a device failure throws.
//
// Everything lives in the inline namespace slimsell::b200, so user code keeps
// writing slimsell::bfs_spmv(...) while the mangled names differ from the
// reference's — both libraries can be linked into one test binary.
// A translation unit that ALSO includes the reference's headers defines
// SLIMSELL_B200_ALONGSIDE_REFERENCE first: b200 is then an ordinary nested
// namespace, slimsell::X names the reference's X and slimsell::b200::X ours.
//
// Differences a maintainer should know:
//  * Graph and SlimSellRepr own DEVICE handles; their host arrays
//    (Graph::edges(), SlimSellRepr::col/cs/cl/perm/inv_perm) are exported
//    lazily on first access and cached.
//  * BfsOptions::schedule / workers are accepted and ignored.
//  * BfsOptions::selmax_compat (default true) reproduces the reference's
//    sel-max root encoding; false gives corrected parents.
//  * bfs_traditional (both overloads) runs the reference's queue BFS on the
//    device; the CsrView overload expects a symmetric CSR (as to_csr returns).
//  * A layout the REFERENCE built on the host (any struct with the
//    repr.hpp:33-55 members, e.g. slimsell::SlimSellRepr) goes through
//    upload(): copied to the device once and cached by a fingerprint, so the
//    bfs_spmv / spmv_step / spmv_segment overloads taking it cost one upload.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <optional>
#include <type_traits>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "slimsell_b200.h"

namespace slimsell {
#ifdef SLIMSELL_B200_ALONGSIDE_REFERENCE
namespace b200 {
#else
inline namespace b200 {
#endif

// ---- graph.hpp ----------------------------------------------------------
using vid_t = std::int64_t;

/// graph.hpp:15-21 — malformed input text, with its 1-based line.
class ParseError : public std::runtime_error {
 public:
  ParseError(std::int64_t line, const std::string& what_with_line)
      : std::runtime_error(what_with_line), line_(line) {}
  std::int64_t line() const { return line_; }

 private:
  std::int64_t line_;
};

namespace detail {
[[noreturn]] inline void raise(int rc) {
  const std::string msg = ssb_last_error();
  switch (rc) {
    case SSB_EINVAL: throw std::invalid_argument(msg);
    case SSB_ERANGE: throw std::out_of_range(msg);
    case SSB_EPARSE: {  // "line N: ..."
      std::int64_t line = 0;
      if (msg.rfind("line ", 0) == 0) line = std::strtoll(msg.c_str() + 5, nullptr, 10);
      throw ParseError(line, msg);
    }
    default: throw std::runtime_error("slimsell_b200: " + msg);
  }
}
inline void check(int rc) {
  if (rc != SSB_OK) raise(rc);
}
}  // namespace detail

/// Normalised undirected graph (graph.hpp:31-51) held on the device.
class Graph {
 public:
  Graph() = default;

  /// graph.hpp:36 — orient, drop self-loops, sort, dedup (on the device).
  static Graph from_pairs(std::vector<std::pair<vid_t, vid_t>> pairs, vid_t n = -1) {
    std::vector<std::int64_t> uv(2 * pairs.size());
    for (std::size_t i = 0; i < pairs.size(); ++i) {
      uv[2 * i] = pairs[i].first;
      uv[2 * i + 1] = pairs[i].second;
    }
    ssb_edges* h = nullptr;
    detail::check(ssb_edges_from_pairs(uv.data(), static_cast<std::int64_t>(pairs.size()), n, &h));
    return Graph(h);
  }

  vid_t num_vertices() const { return n_; }
  vid_t num_edges() const { return m_; }

  /// graph.hpp:44 — exported from the device on first use.
  const std::vector<std::pair<vid_t, vid_t>>& edges() const {
    if (!edges_cache_) {
      std::vector<std::int64_t> uv(2 * m_);
      if (m_) detail::check(ssb_edges_export(h_.get(), uv.data()));
      auto e = std::make_shared<std::vector<std::pair<vid_t, vid_t>>>(m_);
      for (vid_t i = 0; i < m_; ++i) (*e)[i] = {uv[2 * i], uv[2 * i + 1]};
      edges_cache_ = std::move(e);
    }
    return *edges_cache_;
  }

  bool has_edge(vid_t u, vid_t v) const {  // graph.cpp:88-92
    if (u == v) return false;
    if (u > v) std::swap(u, v);
    const auto& e = edges();
    auto it = std::lower_bound(e.begin(), e.end(), std::make_pair(u, v));
    return it != e.end() && *it == std::make_pair(u, v);
  }

  ssb_edges* handle() const { return h_.get(); }
  explicit Graph(ssb_edges* h) : h_(h, &ssb_edges_destroy) {
    detail::check(ssb_edges_info(h, &n_, &m_));
  }

 private:
  std::shared_ptr<ssb_edges> h_;
  vid_t n_ = 0, m_ = 0;
  mutable std::shared_ptr<std::vector<std::pair<vid_t, vid_t>>> edges_cache_;
};

/// graph.hpp:63-69
struct CsrView {
  std::vector<vid_t> row;
  std::vector<vid_t> col;
  vid_t num_vertices() const { return static_cast<vid_t>(row.size()) - 1; }
  bool has_edge(vid_t u, vid_t v) const {
    if (u < 0 || u >= num_vertices() || v < 0 || v >= num_vertices()) return false;
    return std::binary_search(col.begin() + row[u], col.begin() + row[u + 1], v);
  }
};

/// graph.hpp:50
enum class InputDirective { symmetrize, reject_asymmetric };

/// graph.hpp:55-56 (graph.cpp:94-133) — parsed on the host, normalised on the device.
inline Graph from_edge_list(std::string_view text,
                            InputDirective directive = InputDirective::symmetrize) {
  ssb_edges* h = nullptr;
  detail::check(ssb_edges_from_edge_list(text.data(), static_cast<std::int64_t>(text.size()),
                                         directive == InputDirective::reject_asymmetric
                                             ? SSB_REJECT_ASYMMETRIC
                                             : SSB_SYMMETRIZE,
                                         &h));
  return Graph(h);
}

/// graph.hpp:58-59 (graph.cpp:135-210).
inline Graph from_matrix_market(std::string_view text) {
  ssb_edges* h = nullptr;
  detail::check(
      ssb_edges_from_matrix_market(text.data(), static_cast<std::int64_t>(text.size()), &h));
  return Graph(h);
}

/// graph.hpp:71 (graph.cpp:212-232), on the device.
inline CsrView to_csr(const Graph& g) {
  CsrView c;
  c.row.resize(g.num_vertices() + 1);
  c.col.resize(2 * g.num_edges());
  detail::check(ssb_to_csr(g.handle(), c.row.data(), c.col.data()));
  return c;
}

// ---- generator.hpp ------------------------------------------------------
/// generator.hpp:55 — bit-exact counter-based generation on the device.
inline Graph gen_kronecker(std::int64_t scale, std::int64_t edgefactor, std::uint64_t seed,
                           const std::array<double, 4>& initiator = {0.57, 0.19, 0.19, 0.05}) {
  ssb_edges* h = nullptr;
  detail::check(ssb_gen_kronecker(scale, edgefactor, seed, initiator.data(), &h));
  return Graph(h);
}

/// generator.hpp:50 — bit-exact (host-drawn skips, device decode).
inline Graph gen_erdos_renyi(vid_t n, double p, std::uint64_t seed) {
  ssb_edges* h = nullptr;
  detail::check(ssb_gen_erdos_renyi(n, p, seed, &h));
  return Graph(h);
}

inline Graph gen_path(vid_t n) {  // generator.hpp:62
  if (n < 1) throw std::invalid_argument("path needs n >= 1");
  std::vector<std::pair<vid_t, vid_t>> p;
  for (vid_t i = 0; i + 1 < n; ++i) p.emplace_back(i, i + 1);
  return Graph::from_pairs(std::move(p), n);
}

inline Graph gen_clique(vid_t n) {  // generator.hpp:63
  if (n < 1) throw std::invalid_argument("clique needs n >= 1");
  std::vector<std::pair<vid_t, vid_t>> p;
  for (vid_t u = 0; u < n; ++u)
    for (vid_t v = u + 1; v < n; ++v) p.emplace_back(u, v);
  return Graph::from_pairs(std::move(p), n);
}

inline Graph gen_star(vid_t n) {  // generator.hpp:64
  if (n < 1) throw std::invalid_argument("star needs n >= 1");
  std::vector<std::pair<vid_t, vid_t>> p;
  for (vid_t v = 1; v < n; ++v) p.emplace_back(0, v);
  return Graph::from_pairs(std::move(p), n);
}

// ---- semiring.hpp -------------------------------------------------------
using val_t = std::int64_t;
inline constexpr val_t kInf = std::numeric_limits<val_t>::max();
inline constexpr vid_t kNoParent = -1;

enum class Variant { tropical, real, boolean, selmax };
inline constexpr Variant kAllVariants[] = {Variant::tropical, Variant::real, Variant::boolean,
                                           Variant::selmax};

/// semiring.hpp:37-49 — the scalar algebra, for API parity (the device
/// kernels implement the same operations).
struct SemiringSpec {
  Variant variant;
  const char* name;
  val_t zero, one, edge_value, pad_value;
  val_t (*plus)(val_t, val_t);
  val_t (*times)(val_t, val_t);
};

inline const SemiringSpec& semiring(Variant v) {
  static const SemiringSpec specs[] = {
      {Variant::tropical, "tropical", kInf, 0, 1, kInf,
       [](val_t a, val_t b) { return a < b ? a : b; },
       [](val_t a, val_t b) { return (a == kInf || b == kInf) ? kInf : a + b; }},
      {Variant::real, "real", 0, 1, 1, 0,
       [](val_t a, val_t b) { return static_cast<val_t>(static_cast<std::uint64_t>(a) + static_cast<std::uint64_t>(b)); },
       [](val_t a, val_t b) { return static_cast<val_t>(static_cast<std::uint64_t>(a) * static_cast<std::uint64_t>(b)); }},
      {Variant::boolean, "boolean", 0, 1, 1, 0, [](val_t a, val_t b) { return a | b; },
       [](val_t a, val_t b) { return a & b; }},
      {Variant::selmax, "selmax", 0, 1, 1, 0, [](val_t a, val_t b) { return a > b ? a : b; },
       [](val_t a, val_t b) { return static_cast<val_t>(static_cast<std::uint64_t>(a) * static_cast<std::uint64_t>(b)); }},
  };
  return specs[static_cast<int>(v)];
}

inline const char* variant_name(Variant v) { return semiring(v).name; }

inline std::optional<Variant> parse_variant(std::string_view name) {
  for (Variant v : kAllVariants)
    if (name == semiring(v).name) return v;
  return std::nullopt;
}

// ---- repr.hpp -----------------------------------------------------------
inline constexpr vid_t kPadMarker = -1;

namespace detail {
/// A host view of one layout array, exported from the device on first use.
class LazyArray {
 public:
  using Fill = std::function<void(std::vector<std::int64_t>&)>;
  LazyArray() = default;
  explicit LazyArray(Fill f) : fill_(std::make_shared<Fill>(std::move(f))) {}
  const std::vector<std::int64_t>& get() const {
    if (!cache_) {
      cache_ = std::make_shared<std::vector<std::int64_t>>();
      (*fill_)(*cache_);
    }
    return *cache_;
  }
  std::int64_t operator[](std::size_t i) const { return get()[i]; }
  std::size_t size() const { return get().size(); }
  const std::int64_t* data() const { return get().data(); }
  auto begin() const { return get().begin(); }
  auto end() const { return get().end(); }
  operator const std::vector<std::int64_t>&() const { return get(); }

 private:
  std::shared_ptr<Fill> fill_;
  mutable std::shared_ptr<std::vector<std::int64_t>> cache_;
};
}  // namespace detail

/// repr.hpp:33-55 — the SlimSell layout, resident on the device.
struct SlimSellRepr {
  std::int64_t C = 1;
  std::int64_t sigma = 1;
  vid_t n = 0;
  vid_t n_padded = 0;
  std::int64_t n_chunks = 0;
  vid_t nonzeros = 0;
  detail::LazyArray col, cs, cl, perm, inv_perm;
  std::int64_t padding = 0;

  vid_t chunk_row_begin(std::int64_t chunk) const { return static_cast<vid_t>(chunk * C); }
  vid_t chunk_row_end(std::int64_t chunk) const {
    const vid_t end = static_cast<vid_t>((chunk + 1) * C);
    return end < n ? end : n;
  }
  std::int64_t n_cells() const { return n_cells_; }
  ssb_graph* handle() const { return h_.get(); }

  explicit SlimSellRepr(ssb_graph* h) : h_(h, &ssb_graph_destroy) {
    ssb_layout_info info;
    detail::check(ssb_graph_info(h, &info));
    C = info.C;
    sigma = info.sigma;
    n = info.n;
    n_padded = info.n_padded;
    n_chunks = info.n_chunks;
    nonzeros = info.nonzeros;
    padding = info.padding;
    n_cells_ = info.n_cells;
    auto hp = h_;
    auto exp = [hp](int which, std::int64_t count) {
      return [hp, which, count](std::vector<std::int64_t>& v) {
        v.resize(static_cast<std::size_t>(count));
        std::int64_t* p[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
        p[which] = v.data();
        if (count) detail::check(ssb_graph_export(hp.get(), p[0], p[1], p[2], p[3], p[4]));
      };
    };
    col = detail::LazyArray(exp(0, n_cells_));
    cs = detail::LazyArray(exp(1, n_chunks));
    cl = detail::LazyArray(exp(2, n_chunks));
    perm = detail::LazyArray(exp(3, n));
    inv_perm = detail::LazyArray(exp(4, n));
  }

 private:
  std::shared_ptr<ssb_graph> h_;
  std::int64_t n_cells_ = 0;
};

/// repr.hpp:66 — built on the device. Throws invalid_argument for C<=0, σ<=0.
inline SlimSellRepr build_slimsell(const Graph& g, std::int64_t C, std::int64_t sigma) {
  ssb_graph* h = nullptr;
  detail::check(ssb_build_slimsell(g.handle(), C, sigma, &h));
  return SlimSellRepr(h);
}

inline std::int64_t storage_cells(const SlimSellRepr& r) {  // repr.hpp:62 (col + cs + cl)
  return r.n_cells() + 2 * r.n_chunks;
}

/// repr.hpp:90-92 — chunk-range product with the literal int64 semiring.
inline void spmv_step(const SlimSellRepr& r, const SemiringSpec& s, std::span<const val_t> x_prev,
                      std::span<val_t> out, std::int64_t chunk_begin, std::int64_t chunk_end) {
  if (x_prev.size() != static_cast<std::size_t>(r.n_padded) ||
      out.size() != static_cast<std::size_t>(r.n_padded))
    throw std::invalid_argument("x_prev/out length must be n_padded");
  if (r.n_padded == 0) {
    if (chunk_begin != 0 || chunk_end != 0) throw std::invalid_argument("chunk range out of bounds");
    return;
  }
  detail::check(ssb_spmv_step(r.handle(), static_cast<int>(s.variant), x_prev.data(), out.data(),
                              chunk_begin, chunk_end));
}

/// repr.hpp:97-98
inline std::vector<val_t> spmv_step(const SlimSellRepr& r, const SemiringSpec& s,
                                    std::span<const val_t> x_prev) {
  std::vector<val_t> out(x_prev.size());
  spmv_step(r, s, x_prev, out, 0, r.n_chunks);
  return out;
}

/// repr.hpp:79-81 (repr.cpp:20-35) — one chunk's column range folded into
/// C accumulators with the literal int64 semiring, on the device.
inline void spmv_segment(const SlimSellRepr& r, const SemiringSpec& s, std::span<const val_t> x_prev,
                         std::span<val_t> acc, std::int64_t chunk, std::int64_t col_begin,
                         std::int64_t col_len) {
  if (x_prev.size() != static_cast<std::size_t>(r.n_padded)) throw std::invalid_argument("x_prev length");
  if (acc.size() != static_cast<std::size_t>(r.C)) throw std::invalid_argument("acc length must be C");
  detail::check(ssb_spmv_segment(r.handle(), static_cast<int>(s.variant), x_prev.data(), acc.data(), chunk,
                                 col_begin, col_len));
}

// ---- host layouts built by the reference (repr.hpp:33-55) -----------------
namespace detail {
template <class R, class = void>
struct is_host_repr : std::false_type {};
template <class R>
struct is_host_repr<R, std::void_t<decltype(std::declval<const R&>().col.data()),
                                   decltype(std::declval<const R&>().cs.data()),
                                   decltype(std::declval<const R&>().cl.data()),
                                   decltype(std::declval<const R&>().perm.data()),
                                   decltype(std::declval<const R&>().n_padded),
                                   decltype(std::declval<const R&>().nonzeros)>>
    : std::bool_constant<!std::is_same_v<std::decay_t<R>, SlimSellRepr> &&
                         std::is_convertible_v<decltype(std::declval<const R&>().col.data()),
                                               const std::int64_t*>> {};

inline std::uint64_t fnv_mix(std::uint64_t h, std::int64_t v) {
  for (int b = 0; b < 8; ++b) {
    h ^= (static_cast<std::uint64_t>(v) >> (8 * b)) & 0xffu;
    h *= 0x100000001b3ull;
  }
  return h;
}
/// Cheap identity of a host layout: the scalars, cs.back(),
/// and col / perm / cl sampled — their first and last 4096 entries in full
/// (cli.cpp:200-207's corrupt_repr rewrites the FIRST real cell) plus 4096
/// strided samples. Arbitrary rewrites in the middle of col can escape it:
/// call upload(r, true) after mutating a layout in place.
template <class R>
std::uint64_t layout_fingerprint(const R& r) {
  std::uint64_t h = 0xcbf29ce484222325ull;
  for (std::int64_t v : {std::int64_t(r.C), std::int64_t(r.sigma), std::int64_t(r.n), std::int64_t(r.n_chunks),
                         std::int64_t(r.nonzeros), std::int64_t(r.col.size()), std::int64_t(r.cs.size())})
    h = fnv_mix(h, v);
  auto sample = [&h](const auto& v) {
    const std::size_t n = v.size();
    const std::size_t head = std::min<std::size_t>(n, 4096);
    for (std::size_t i = 0; i < head; ++i) h = fnv_mix(h, v[i]);
    for (std::size_t i = n > 4096 ? n - 4096 : head; i < n; ++i) h = fnv_mix(h, v[i]);
    if (n > 8192)
      for (std::size_t k = 0; k < 4096; ++k) h = fnv_mix(h, v[(n / 4096) * k + k % 7]);
  };
  sample(r.col);
  sample(r.cs);
  sample(r.cl);
  sample(r.perm);
  return h;
}
struct UploadCache {
  std::mutex mu;
  std::uint64_t key = 0;
  std::optional<SlimSellRepr> dev;
};
inline UploadCache& upload_cache() {
  static UploadCache c;
  return c;
}
}  // namespace detail

/// A host SlimSellRepr built by the reference (repr.hpp:33-55: C, sigma, n,
/// n_chunks, nonzeros, col, cs, cl, perm) on the device — uploaded through
/// ssb_graph_from_layout once, then served from a one-entry cache keyed by
/// detail::layout_fingerprint (force = true re-uploads).
template <class HostRepr, std::enable_if_t<detail::is_host_repr<HostRepr>::value, int> = 0>
inline SlimSellRepr upload(const HostRepr& r, bool force = false) {
  auto& c = detail::upload_cache();
  std::lock_guard<std::mutex> lock(c.mu);
  const std::uint64_t key = detail::layout_fingerprint(r);
  if (!force && c.dev && c.key == key) return *c.dev;
  ssb_graph* h = nullptr;
  detail::check(ssb_graph_from_layout(r.n, r.C, r.sigma, r.nonzeros, r.col.data(),
                                      static_cast<std::int64_t>(r.col.size()), r.cs.data(), r.cl.data(),
                                      static_cast<std::int64_t>(r.cs.size()), r.perm.data(), &h));
  c.dev.emplace(h);
  c.key = key;
  return *c.dev;
}

// The semiring may be the reference's own SemiringSpec (its variant selects
// the device algebra).
template <class HostRepr, class Semi, std::enable_if_t<detail::is_host_repr<HostRepr>::value, int> = 0>
inline void spmv_step(const HostRepr& r, const Semi& s, std::span<const val_t> x_prev,
                      std::span<val_t> out, std::int64_t chunk_begin, std::int64_t chunk_end) {
  spmv_step(upload(r), semiring(static_cast<Variant>(static_cast<int>(s.variant))), x_prev, out,
            chunk_begin, chunk_end);
}

template <class HostRepr, class Semi, std::enable_if_t<detail::is_host_repr<HostRepr>::value, int> = 0>
inline std::vector<val_t> spmv_step(const HostRepr& r, const Semi& s, std::span<const val_t> x_prev) {
  return spmv_step(upload(r), semiring(static_cast<Variant>(static_cast<int>(s.variant))), x_prev);
}

template <class HostRepr, class Semi, std::enable_if_t<detail::is_host_repr<HostRepr>::value, int> = 0>
inline void spmv_segment(const HostRepr& r, const Semi& s, std::span<const val_t> x_prev,
                         std::span<val_t> acc, std::int64_t chunk, std::int64_t col_begin,
                         std::int64_t col_len) {
  spmv_segment(upload(r), semiring(static_cast<Variant>(static_cast<int>(s.variant))), x_prev, acc,
               chunk, col_begin, col_len);
}

/// repr.hpp:104-107 (repr.cpp:239-253) — pure relabelling through perm.
inline std::vector<val_t> permute_in(std::span<const val_t> v, const SlimSellRepr& r, val_t fill) {
  if (v.size() != static_cast<std::size_t>(r.n)) throw std::invalid_argument("input vector length");
  std::vector<val_t> out(r.n_padded, fill);
  for (vid_t p = 0; p < r.n; ++p) out[p] = v[r.perm[p]];
  return out;
}

inline std::vector<val_t> permute_out(std::span<const val_t> v, const SlimSellRepr& r) {
  if (v.size() != static_cast<std::size_t>(r.n_padded))
    throw std::invalid_argument("permuted vector length");
  std::vector<val_t> out(r.n);
  for (vid_t p = 0; p < r.n; ++p) out[r.perm[p]] = v[p];
  return out;
}

// ---- bfs.hpp ------------------------------------------------------------
enum class Schedule { static_blocks, dynamic_queue };

struct BfsOptions {  // bfs.hpp:16-24
  Variant variant = Variant::tropical;
  bool slimwork = false;
  std::int64_t slimchunk_len = 0;
  Schedule schedule = Schedule::static_blocks;  // ignored
  int workers = 1;                              // ignored
  std::int64_t max_iterations = 0;
  bool want_parents = true;
  bool selmax_compat = true;
};

struct IterStats {  // bfs.hpp:26-34
  std::int64_t iteration = 0;
  std::int64_t elapsed_ns = 0;
  std::int64_t chunks_processed = 0;
  std::int64_t chunks_skipped = 0;
  std::int64_t subchunks_processed = 0;
  std::int64_t columns_processed = 0;
  std::int64_t frontier_size = 0;
};

struct BfsResult {  // bfs.hpp:36-42
  std::vector<val_t> dist;
  std::vector<vid_t> parent;
  std::int64_t iterations = 0;
  std::vector<IterStats> per_iter;
};

class BfsCapError : public std::runtime_error {  // bfs.hpp:46-54
 public:
  BfsCapError(std::string what, BfsResult partial)
      : std::runtime_error(std::move(what)), partial_(std::move(partial)) {}
  const BfsResult& partial() const { return partial_; }

 private:
  BfsResult partial_;
};

struct SubchunkPlan {  // bfs.hpp:58-66
  struct Segment {
    std::int64_t chunk = 0;
    std::int64_t col_begin = 0;
    std::int64_t col_len = 0;
  };
  std::vector<Segment> segments;
  std::vector<std::int64_t> chunk_first;
};

/// bfs.hpp:69 (bfs.cpp:10-22) — the reference's segment list; the device
/// builds the same segments as its work units.
inline SubchunkPlan plan_subchunks(const SlimSellRepr& r, std::int64_t L) {
  if (L < 1) throw std::invalid_argument("subchunk length must be >= 1");
  SubchunkPlan plan;
  plan.chunk_first.reserve(r.n_chunks + 1);
  for (std::int64_t i = 0; i < r.n_chunks; ++i) {
    plan.chunk_first.push_back(static_cast<std::int64_t>(plan.segments.size()));
    for (std::int64_t c = 0; c < r.cl[i]; c += L)
      plan.segments.push_back({i, c, std::min(L, r.cl[i] - c)});
  }
  plan.chunk_first.push_back(static_cast<std::int64_t>(plan.segments.size()));
  return plan;
}

/// bfs.hpp:73-74
inline std::vector<val_t> combine_partials(const SemiringSpec& s,
                                           const std::vector<std::vector<val_t>>& partials) {
  if (partials.empty()) return {};
  std::vector<val_t> out = partials.front();
  for (std::size_t i = 1; i < partials.size(); ++i) {
    if (partials[i].size() != out.size())
      throw std::invalid_argument("partial accumulator length mismatch");
    for (std::size_t j = 0; j < out.size(); ++j) out[j] = s.plus(out[j], partials[i][j]);
  }
  return out;
}

/// bfs.hpp:80-81 — algebraic BFS on the device. As the reference: sel-max
/// parents always (when want_parents), the other variants only with a CSR
/// (dp_transform semantics, evaluated on the device over the layout).
namespace detail {
inline BfsResult bfs_spmv_device(const SlimSellRepr& r, vid_t root, const BfsOptions& opts,
                                 bool csr_given) {
  ssb_bfs_options o{};
  o.variant = static_cast<std::int32_t>(opts.variant);
  o.slimwork = opts.slimwork;
  o.slimchunk_len = opts.slimchunk_len;
  o.schedule = static_cast<std::int32_t>(opts.schedule);
  o.workers = opts.workers;
  o.max_iterations = opts.max_iterations;
  o.want_parents = opts.want_parents && (opts.variant == Variant::selmax || csr_given);
  o.selmax_compat = opts.selmax_compat;
  BfsResult res;
  res.dist.resize(r.n);
  res.parent.resize(r.n);
  std::int64_t plen = 0, iters = 0;
  std::vector<ssb_iter_stats> st(std::min<std::int64_t>(r.n + 2, 1 << 16));
  int rc = ssb_bfs_spmv(r.handle(), root, &o, res.dist.data(), res.parent.data(), &plen, st.data(),
                        static_cast<std::int64_t>(st.size()), &iters);
  if (rc == SSB_OK || rc == SSB_ECAP) {
    if (iters > static_cast<std::int64_t>(st.size())) {  // very deep BFS: rerun with room
      st.resize(iters);
      rc = ssb_bfs_spmv(r.handle(), root, &o, res.dist.data(), res.parent.data(), &plen, st.data(),
                        static_cast<std::int64_t>(st.size()), &iters);
    }
  }
  if (rc != SSB_OK && rc != SSB_ECAP) detail::raise(rc);
  res.parent.resize(plen);
  res.iterations = iters;
  for (std::int64_t i = 0; i < iters; ++i) {
    const auto& s = st[i];
    res.per_iter.push_back({s.iteration, s.elapsed_ns, s.chunks_processed, s.chunks_skipped,
                            s.subchunks_processed, s.columns_processed, s.frontier_size});
  }
  if (rc == SSB_ECAP) throw BfsCapError(ssb_last_error(), std::move(res));
  return res;
}
}  // namespace detail

inline BfsResult bfs_spmv(const SlimSellRepr& r, vid_t root, const BfsOptions& opts,
                          const CsrView* csr_for_parents = nullptr) {
  return detail::bfs_spmv_device(r, root, opts, csr_for_parents != nullptr);
}

/// bfs.hpp:80-81 on a layout the reference built on the host (upload()). The
/// CSR may be the reference's own CsrView: only its presence matters (the
/// parents are dp_transform's, evaluated on the device over the layout).
template <class HostRepr, class Csr = CsrView,
          std::enable_if_t<detail::is_host_repr<HostRepr>::value, int> = 0>
inline BfsResult bfs_spmv(const HostRepr& r, vid_t root, const BfsOptions& opts,
                          const Csr* csr_for_parents = nullptr) {
  return detail::bfs_spmv_device(upload(r), root, opts, csr_for_parents != nullptr);
}

/// Extension: a Graph500 root list through ssb_bfs_spmv_batch — results as
/// from bfs_spmv per root (no per_iter records), root i's host fetch
/// overlapped with root i+1's BFS on the device.
inline std::vector<BfsResult> bfs_spmv_batch(const SlimSellRepr& r, const std::vector<vid_t>& roots,
                                             const BfsOptions& opts,
                                             const CsrView* csr_for_parents = nullptr) {
  ssb_bfs_options o{};
  o.variant = static_cast<std::int32_t>(opts.variant);
  o.slimwork = opts.slimwork;
  o.slimchunk_len = opts.slimchunk_len;
  o.schedule = static_cast<std::int32_t>(opts.schedule);
  o.workers = opts.workers;
  o.max_iterations = opts.max_iterations;
  o.want_parents = opts.want_parents &&
                   (opts.variant == Variant::selmax || csr_for_parents != nullptr);
  o.selmax_compat = opts.selmax_compat;
  std::vector<BfsResult> out(roots.size());
  std::vector<std::int64_t*> dp(roots.size()), pp(roots.size());
  for (std::size_t i = 0; i < roots.size(); ++i) {
    out[i].dist.resize(r.n);
    out[i].parent.resize(o.want_parents ? r.n : 0);
    dp[i] = out[i].dist.data();
    pp[i] = o.want_parents ? out[i].parent.data() : nullptr;
  }
  std::vector<std::int64_t> iters(roots.size() + 1);
  std::int64_t capped = -1;
  const int rc = ssb_bfs_spmv_batch(r.handle(), roots.data(), static_cast<std::int64_t>(roots.size()),
                                    &o, dp.data(), pp.data(), iters.data(), &capped);
  for (std::size_t i = 0; i < roots.size(); ++i) out[i].iterations = iters[i];
  if (rc == SSB_ECAP) {
    BfsResult partial = std::move(out[static_cast<std::size_t>(capped)]);
    partial.parent.clear();
    throw BfsCapError(ssb_last_error(), std::move(partial));
  }
  if (rc != SSB_OK) detail::raise(rc);
  return out;
}

/// bfs.hpp:86 (bfs.cpp:248-291) — the reference's queue BFS, run on the
/// device over the graph's CSR: dist, parent = smallest neighbour one level
/// closer (root self-parented), per_iter {iteration, elapsed_ns,
/// frontier_size}.
inline BfsResult bfs_traditional(const Graph& g, vid_t root) {
  BfsResult res;
  res.dist.resize(g.num_vertices());
  res.parent.resize(g.num_vertices());
  std::vector<ssb_iter_stats> st(std::min<std::int64_t>(g.num_vertices() + 2, 1 << 16));
  std::int64_t iters = 0;
  int rc = ssb_bfs_traditional(g.handle(), root, res.dist.data(), res.parent.data(), st.data(),
                               static_cast<std::int64_t>(st.size()), &iters);
  if (rc == SSB_OK && iters > static_cast<std::int64_t>(st.size())) {
    st.resize(iters);
    rc = ssb_bfs_traditional(g.handle(), root, res.dist.data(), res.parent.data(), st.data(),
                             static_cast<std::int64_t>(st.size()), &iters);
  }
  if (rc != SSB_OK) detail::raise(rc);
  res.iterations = iters;
  for (std::int64_t i = 0; i < iters; ++i) {
    IterStats s;
    s.iteration = st[i].iteration;
    s.elapsed_ns = st[i].elapsed_ns;
    s.frontier_size = st[i].frontier_size;
    res.per_iter.push_back(s);
  }
  return res;
}

/// bfs.hpp:85 (bfs.cpp:248-291) on a CSR: its arcs become the normalised
/// edge set on the device (a symmetric CSR, as to_csr returns, gives exactly
/// the reference's traversal), then the device queue BFS.
template <class Csr,
          std::enable_if_t<std::is_same_v<std::decay_t<decltype(std::declval<const Csr&>().row[0])>,
                                          vid_t> &&
                               std::is_same_v<std::decay_t<decltype(std::declval<const Csr&>().col[0])>,
                                              vid_t>,
                           int> = 0>
inline BfsResult bfs_traditional(const Csr& csr, vid_t root) {
  const vid_t n = static_cast<vid_t>(csr.row.size()) - 1;
  auto has_edge = [&](vid_t u, vid_t v) {
    return std::binary_search(csr.col.begin() + csr.row[u], csr.col.begin() + csr.row[u + 1], v);
  };
  if (root < 0 || root >= n)
    throw std::out_of_range("root " + std::to_string(root) + " outside [0, " + std::to_string(n) + ")");
  std::vector<std::int64_t> uv;
  uv.reserve(csr.col.size());
  for (vid_t u = 0; u < n; ++u)
    for (vid_t e = csr.row[u]; e < csr.row[u + 1]; ++e)
      if (u < csr.col[e]) {
        uv.push_back(u);
        uv.push_back(csr.col[e]);
      } else if (csr.col[e] < u && !has_edge(csr.col[e], u)) {  // an arc with no mirror
        uv.push_back(csr.col[e]);
        uv.push_back(u);
      }
  ssb_edges* h = nullptr;
  detail::check(ssb_edges_from_pairs(uv.data(), static_cast<std::int64_t>(uv.size() / 2), n, &h));
  return bfs_traditional(Graph(h), root);
}

// ---- one process, several B200s (ssb_ctx_*) -------
/// The devices of a single-process multi-GPU job: all distinct (peer access
/// between every pair, the frontier exchange fused over NVLink) or all the
/// same (the ranks emulated as one cooperative launch on it).
class Context {
 public:
  explicit Context(const std::vector<int>& device_ids) {
    ssb_ctx* h = nullptr;
    detail::check(ssb_ctx_create(static_cast<int>(device_ids.size()), device_ids.data(), &h));
    h_.reset(h, &ssb_ctx_destroy);
    ranks_ = static_cast<int>(device_ids.size());
  }
  ssb_ctx* handle() const { return h_.get(); }
  int ranks() const { return ranks_; }

 private:
  std::shared_ptr<ssb_ctx> h_;
  int ranks_ = 0;
};

/// A SlimSellRepr sharded over a Context (segments_per_rank round-robin,
/// cell-balanced chunk segments per rank; each rank holds only its cells).
class ShardedRepr {
 public:
  ShardedRepr(const Context& ctx, const Graph& g, std::int64_t C, std::int64_t sigma, int segments_per_rank = 4)
      : ctx_(ctx) {
    ssb_sharded* h = nullptr;
    detail::check(ssb_ctx_build(ctx.handle(), g.handle(), C, sigma, segments_per_rank, &h));
    h_.reset(h, &ssb_sharded_destroy);
    int nr = 0;
    detail::check(ssb_sharded_info(h, &nr, &n_, nullptr, nullptr));
    cells_.resize(static_cast<std::size_t>(nr));
    detail::check(ssb_sharded_info(h, &nr, nullptr, cells_.data(), nullptr));
  }
  ssb_sharded* handle() const { return h_.get(); }
  vid_t n() const { return n_; }
  const std::vector<std::int64_t>& cells_per_rank() const { return cells_; }

 private:
  Context ctx_;  // keeps the context alive
  std::shared_ptr<ssb_sharded> h_;
  vid_t n_ = 0;
  std::vector<std::int64_t> cells_;
};

/// bfs.hpp:80-81 over the shards of a context (sel-max parents when
/// want_parents; the other variants return dist only).
inline BfsResult bfs_spmv(const ShardedRepr& r, vid_t root, const BfsOptions& opts) {
  ssb_bfs_options o{};
  o.variant = static_cast<std::int32_t>(opts.variant);
  o.slimwork = opts.slimwork;
  o.slimchunk_len = opts.slimchunk_len;
  o.max_iterations = opts.max_iterations;
  o.want_parents = opts.want_parents && opts.variant == Variant::selmax;
  o.selmax_compat = opts.selmax_compat;
  BfsResult res;
  res.dist.resize(r.n());
  res.parent.resize(r.n());
  std::int64_t plen = 0, iters = 0;
  std::vector<ssb_iter_stats> st(std::min<std::int64_t>(r.n() + 2, 1 << 16));
  const int rc = ssb_sharded_bfs(r.handle(), root, &o, res.dist.data(), res.parent.data(), &plen, st.data(),
                                 static_cast<std::int64_t>(st.size()), &iters, nullptr);
  if (rc != SSB_OK && rc != SSB_ECAP) detail::raise(rc);
  res.parent.resize(plen);
  res.iterations = iters;
  for (std::int64_t i = 0; i < std::min<std::int64_t>(iters, static_cast<std::int64_t>(st.size())); ++i) {
    const auto& s = st[i];
    res.per_iter.push_back({s.iteration, s.elapsed_ns, s.chunks_processed, s.chunks_skipped,
                            s.subchunks_processed, s.columns_processed, s.frontier_size});
  }
  if (rc == SSB_ECAP) {
    res.parent.clear();
    throw BfsCapError(ssb_last_error(), std::move(res));
  }
  return res;
}

/// cli.cpp:73-112 (verify_against_oracle's tree checks) + Graph500 edge
/// checks, on the device. Empty optional = valid, else a diff report.
inline std::optional<std::string> validate_bfs(const Graph& g, vid_t root, const BfsResult& run,
                                               bool selmax_compat = false) {
  std::int64_t bad = 0;
  char report[1024];
  const int rc = ssb_validate_bfs(g.handle(), root, run.dist.data(),
                                  run.parent.empty() ? nullptr : run.parent.data(),
                                  selmax_compat ? SSB_VALIDATE_SELMAX_COMPAT : 0, &bad, report,
                                  static_cast<std::int64_t>(sizeof report));
  if (rc != SSB_OK) detail::raise(rc);
  if (bad == 0) return std::nullopt;
  return std::to_string(bad) + " violation(s):\n" + report;
}

}  // namespace b200
}  // namespace slimsell
