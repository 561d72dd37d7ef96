// C++ parity tests of the header-only façade (include/slimsell_b200/*.hpp),
// written the way the reference's own doctest suite reads
// (proj/tests/test_graph.cpp), checked against the C oracle
// (oracle/slimsell_oracle.c, test infrastructure only).
//
// Build (tests/test_cpp.py does this):
//   g++ -std=c++20 -Iinclude -Ioracle tests/cpp/test_facade.cpp
//       -Lpaper_2010_09913_b200 -lslimsell_b200 -Loracle -loracle
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "slimsell_b200/bfs.hpp"
#include "slimsell_b200/generator.hpp"
#include "slimsell_b200/graph.hpp"
#include "slimsell_b200/repr.hpp"
#include "slimsell_oracle.h"

static int g_failed = 0, g_checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_failed;                                                          \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                 \
  do {                                                \
    bool thrown = false;                              \
    try {                                             \
      (void)(expr);                                   \
    } catch (const T&) {                              \
      thrown = true;                                  \
    }                                                 \
    CHECK(thrown);                                    \
  } while (0)
#define TEST_CASE(name) static void name()

using namespace slimsell;

static std::vector<std::int64_t> vec(const detail::LazyArray& a) { return a.get(); }

TEST_CASE(csr_layout_of_path4) {  // test_graph.cpp:93-98
  Graph g = gen_path(4);
  CsrView c = to_csr(g);
  CHECK((c.row == std::vector<vid_t>{0, 1, 3, 5, 6}));
  CHECK((c.col == std::vector<vid_t>{1, 0, 2, 1, 3, 2}));
}

TEST_CASE(from_pairs_normalises) {
  Graph g = Graph::from_pairs({{3, 1}, {1, 3}, {2, 2}, {0, 1}}, 5);
  CHECK(g.num_vertices() == 5);
  CHECK(g.num_edges() == 2);
  CHECK((g.edges() == std::vector<std::pair<vid_t, vid_t>>{{0, 1}, {1, 3}}));
  CHECK(g.has_edge(3, 1) && !g.has_edge(2, 2));
  CHECK_THROWS_AS(Graph::from_pairs({{0, 9}}, 5), std::out_of_range);
}

TEST_CASE(spec_layout_kats) {
  Graph g = gen_path(4);
  SlimSellRepr a = build_slimsell(g, 2, 1);
  CHECK((vec(a.cs) == std::vector<std::int64_t>{0, 4}));
  CHECK((vec(a.cl) == std::vector<std::int64_t>{2, 2}));
  CHECK((vec(a.col) == std::vector<std::int64_t>{1, 0, -1, 2, 1, 2, 3, -1}));
  CHECK(a.padding == 2);
  SlimSellRepr b = build_slimsell(g, 2, 4);
  CHECK((vec(b.perm) == std::vector<std::int64_t>{1, 2, 0, 3}));
  CHECK((vec(b.col) == std::vector<std::int64_t>{1, 0, 2, 3, 0, 1}));
  CHECK(b.padding == 0);
  CHECK_THROWS_AS(build_slimsell(g, 0, 1), std::invalid_argument);
}

TEST_CASE(spec_spmv_kats) {
  SlimSellRepr r = build_slimsell(gen_path(4), 2, 1);
  std::vector<val_t> x = {0, kInf, kInf, kInf};
  CHECK((spmv_step(r, semiring(Variant::tropical), x) == std::vector<val_t>{0, 1, kInf, kInf}));
  x = {1, 0, 0, 0};
  CHECK((spmv_step(r, semiring(Variant::selmax), x) == std::vector<val_t>{1, 1, 0, 0}));
  x = {1, 1, 0, 1};
  CHECK((spmv_step(r, semiring(Variant::real), x) == std::vector<val_t>{2, 2, 2, 1}));
}

TEST_CASE(spec_bfs_kats) {
  Graph g = gen_path(4);
  CsrView csr = to_csr(g);
  for (std::int64_t C : {2, 32}) {
    SlimSellRepr r = build_slimsell(g, C, 1);
    for (Variant v : kAllVariants) {
      BfsOptions o;
      o.variant = v;
      BfsResult res = bfs_spmv(r, 0, o, &csr);
      CHECK((res.dist == std::vector<val_t>{0, 1, 2, 3}));
      CHECK(res.iterations == 4);
      CHECK(res.per_iter[3].frontier_size == 0);
    }
    SlimSellRepr r4 = build_slimsell(g, C, 4);
    BfsOptions o;
    o.variant = Variant::selmax;
    // the reference's sel-max root encoding
    CHECK((bfs_spmv(r4, 0, o).parent == std::vector<vid_t>{1, 1, 1, 2}));
    CHECK((bfs_spmv(r4, 2, o).parent == std::vector<vid_t>{1, 0, 0, 0}));
    o.selmax_compat = false;
    CHECK((bfs_spmv(r4, 2, o).parent == std::vector<vid_t>{1, 2, 2, 2}));
    CHECK_THROWS_AS(bfs_spmv(r4, 4, o), std::out_of_range);
    o.max_iterations = 2;
    CHECK_THROWS_AS(bfs_spmv(r4, 0, o), BfsCapError);
  }
}

TEST_CASE(kronecker_matches_oracle) {
  const std::int64_t scale = 12;
  Graph g = gen_kronecker(scale, 16, 3);
  // oracle graph
  std::vector<std::int64_t> uv(2 * (std::int64_t{16} << scale));
  const double init[4] = {0.57, 0.19, 0.19, 0.05};
  so_gen_kronecker_pairs(scale, 16, 3, init, uv.data());
  std::int64_t n = 0;
  const std::int64_t m = so_normalize_pairs(uv.data(), 16 << scale, 1 << scale, &n);
  CHECK(m == g.num_edges());
  const auto& e = g.edges();
  bool same = true;
  for (std::int64_t i = 0; i < m && same; ++i) same = e[i].first == uv[2 * i] && e[i].second == uv[2 * i + 1];
  CHECK(same);
  std::vector<std::int64_t> row(n + 1), col(2 * m);
  so_to_csr(n, uv.data(), m, row.data(), col.data());
  CsrView csr = to_csr(g);
  CHECK(csr.row == row && csr.col == col);
  for (auto [C, sigma] : {std::pair<std::int64_t, std::int64_t>{32, n}, {8, 8}, {3, 1}}) {
    SlimSellRepr r = build_slimsell(g, C, sigma);
    so_repr L;
    so_build_slimsell(n, row.data(), col.data(), C, sigma, &L);
    CHECK(std::equal(L.col, L.col + L.n_cells, r.col.begin()));
    CHECK(std::equal(L.perm, L.perm + n, r.perm.begin()));
    for (Variant v : kAllVariants) {
      for (std::int64_t root : {std::int64_t{0}, std::int64_t{77}}) {
        BfsOptions o;
        o.variant = v;
        o.slimwork = true;
        o.slimchunk_len = 16;
        BfsResult res = bfs_spmv(r, root, o, &csr);
        std::vector<std::int64_t> d(n), p(n), st(7 * (n + 2));
        std::int64_t plen = 0, it = 0;
        so_bfs_spmv(&L, root, static_cast<int>(v), 1, 16, 0, 1, row.data(), col.data(), d.data(),
                    p.data(), &plen, &it, st.data(), n + 2);
        CHECK(res.iterations == it);
        CHECK(res.dist == d);
        p.resize(plen);
        CHECK(res.parent == p);
        bool counters = true;
        for (std::int64_t k = 0; k < it; ++k) {
          const auto& s = res.per_iter[k];
          const std::int64_t* q = st.data() + 7 * k;
          counters = counters && s.chunks_processed == q[2] && s.chunks_skipped == q[3] &&
                     s.subchunks_processed == q[4] && s.columns_processed == q[5] &&
                     s.frontier_size == q[6];
        }
        CHECK(counters);
      }
      // the batch extension delivers the same results as per-root calls
      if (C == 32) {
        BfsOptions o;
        o.variant = v;
        o.slimwork = true;
        o.slimchunk_len = 16;
        const std::vector<vid_t> roots = {0, 77, 5};
        std::vector<BfsResult> batch = bfs_spmv_batch(r, roots, o, &csr);
        bool same = batch.size() == roots.size();
        for (std::size_t i = 0; same && i < roots.size(); ++i) {
          const BfsResult one = bfs_spmv(r, roots[i], o, &csr);
          same = one.dist == batch[i].dist && one.parent == batch[i].parent &&
                 one.iterations == batch[i].iterations;
        }
        CHECK(same);
      }
    }
    so_repr_free(&L);
  }
}

// graph.hpp:55-59 readers, bfs.hpp:86 bfs_traditional, and the validator.
void ingest_and_checks() {
  Graph g = from_edge_list("# path 0-1-2-3 plus 5-6\nH 7 4\n0 1\n2 1\n3 2\n5 6\n");
  CHECK(g.num_vertices() == 7 && g.num_edges() == 4);
  Graph h = from_matrix_market(
      "%%MatrixMarket matrix coordinate pattern symmetric\n7 7 4\n2 1\n3 2\n4 3\n7 6\n");
  CHECK(h.edges() == g.edges());
  bool threw = false;
  try {
    from_edge_list("0 1\n1 x\n");
  } catch (const ParseError& e) {
    threw = e.line() == 2;
  }
  CHECK(threw);
  threw = false;
  try {
    from_edge_list("0 1\n", InputDirective::reject_asymmetric);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  BfsResult t = bfs_traditional(g, 1);
  CHECK(t.dist[0] == 1 && t.dist[3] == 2 && t.parent[3] == 2 && t.parent[1] == 1);
  CHECK(t.dist[5] == kInf && t.parent[5] == kNoParent);
  CHECK(!validate_bfs(g, 1, t).has_value());
  BfsResult bad = t;
  bad.parent[3] = 0;  // not a neighbour of 3
  CHECK(validate_bfs(g, 1, bad).has_value());
}

// A layout the reference built on the host (here: the oracle's restatement,
// shaped like repr.hpp:33-55) goes through upload(): bfs_spmv / spmv_step /
// spmv_segment on it equal the oracle; rewriting its first real cell (what
// cli.cpp:200-207's corrupt_repr does) is seen by the fingerprint cache.
struct HostRepr {  // the reference's SlimSellRepr members (repr.hpp:33-55)
  std::int64_t C = 1, sigma = 1;
  vid_t n = 0, n_padded = 0;
  std::int64_t n_chunks = 0;
  vid_t nonzeros = 0;
  std::vector<vid_t> col, cs, cl, perm, inv_perm;
  std::int64_t padding = 0;
};

TEST_CASE(host_layout_upload_and_segment) {
  const std::int64_t scale = 11;
  std::vector<std::int64_t> uv(2 * (std::int64_t{16} << scale));
  const double init[4] = {0.57, 0.19, 0.19, 0.05};
  so_gen_kronecker_pairs(scale, 16, 5, init, uv.data());
  std::int64_t n = 0;
  const std::int64_t m = so_normalize_pairs(uv.data(), 16 << scale, 1 << scale, &n);
  std::vector<std::int64_t> row(n + 1), col(2 * m);
  so_to_csr(n, uv.data(), m, row.data(), col.data());
  for (std::int64_t C : {8, 32}) {
    so_repr L;
    so_build_slimsell(n, row.data(), col.data(), C, n, &L);
    HostRepr h;
    h.C = L.C;
    h.sigma = L.sigma;
    h.n = L.n;
    h.n_padded = L.n_padded;
    h.n_chunks = L.n_chunks;
    h.nonzeros = L.nonzeros;
    h.padding = L.padding;
    h.col.assign(L.col, L.col + L.n_cells);
    h.cs.assign(L.cs, L.cs + L.n_chunks);
    h.cl.assign(L.cl, L.cl + L.n_chunks);
    h.perm.assign(L.perm, L.perm + n);
    h.inv_perm.assign(L.inv_perm, L.inv_perm + n);
    auto oracle_bfs = [&](const so_repr* R, std::int64_t root, std::vector<std::int64_t>& d,
                          std::vector<std::int64_t>& p) {
      std::vector<std::int64_t> st(7 * (n + 2));
      std::int64_t plen = 0, it = 0;
      d.assign(n, 0);
      p.assign(n, 0);
      so_bfs_spmv(R, root, 3, 1, 16, 0, 1, nullptr, nullptr, d.data(), p.data(), &plen, &it, st.data(), n + 2);
      p.resize(plen);
    };
    BfsOptions o;
    o.variant = Variant::selmax;
    o.slimwork = true;
    o.slimchunk_len = 16;
    std::vector<std::int64_t> d, p;
    oracle_bfs(&L, 3, d, p);
    BfsResult a = bfs_spmv(h, 3, o);  // uploads
    CHECK(a.dist == d && a.parent == p);
    BfsResult b = bfs_spmv(h, 3, o);  // cached
    CHECK(b.dist == d && b.parent == p);
    // spmv_step / spmv_segment on the host layout vs the oracle
    std::vector<val_t> x(h.n_padded);
    for (std::size_t i = 0; i < x.size(); ++i) x[i] = static_cast<val_t>((i * 2654435761u) % 1000);
    for (Variant v : kAllVariants) {
      std::vector<val_t> out(h.n_padded, 7), want(h.n_padded, 7);
      spmv_step(h, semiring(v), x, out, 0, h.n_chunks);
      so_spmv_step(&L, static_cast<int>(v), x.data(), want.data(), 0, h.n_chunks);
      CHECK(out == want);
      std::int64_t ch = 0;
      for (std::int64_t i = 0; i < h.n_chunks; ++i)
        if (h.cl[i] > h.cl[ch]) ch = i;
      std::vector<val_t> acc(C, 3), exp(C, 3);
      const std::int64_t cb = h.cl[ch] / 3, len = h.cl[ch] - cb;
      spmv_segment(h, semiring(v), x, acc, ch, cb, len);
      const SemiringSpec& s = semiring(v);
      for (std::int64_t j = cb; j < cb + len; ++j)
        for (std::int64_t l = 0; l < C; ++l) {
          const std::int64_t c = h.col[h.cs[ch] + j * C + l];
          exp[l] = s.plus(exp[l], s.times(x[c < 0 ? 0 : c], c < 0 ? s.pad_value : s.edge_value));
        }
      CHECK(acc == exp);
      CHECK_THROWS_AS(spmv_segment(h, semiring(v), x, acc, ch, 0, h.cl[ch] + 1), std::invalid_argument);
    }
    // corrupt_repr (cli.cpp:200-207): the first real cell is rewritten in place
    for (std::int64_t i = 0; i < L.n_cells; ++i)
      if (L.col[i] >= 0) {
        L.col[i] = (L.col[i] + 1) % n;
        h.col[i] = L.col[i];
        break;
      }
    oracle_bfs(&L, 3, d, p);
    BfsResult c = bfs_spmv(h, 3, o);
    CHECK(c.dist == d && c.parent == p);
    so_repr_free(&L);
  }
  // bfs.hpp:85 — the CsrView overload equals the Graph overload
  Graph g = Graph::from_pairs([&] {
    std::vector<std::pair<vid_t, vid_t>> pr;
    for (std::int64_t i = 0; i < m; ++i) pr.emplace_back(uv[2 * i], uv[2 * i + 1]);
    return pr;
  }(), n);
  CsrView csr;
  csr.row = row;
  csr.col = col;
  BfsResult t1 = bfs_traditional(csr, 3), t2 = bfs_traditional(g, 3);
  CHECK(t1.dist == t2.dist && t1.parent == t2.parent && t1.iterations == t2.iterations);
  CHECK_THROWS_AS(bfs_traditional(csr, n), std::out_of_range);
}

// one process, several ranks (here all on device 0: the emulated group)
TEST_CASE(context_sharded_bfs) {
  Graph g = gen_kronecker(13, 16, 2);
  SlimSellRepr r = build_slimsell(g, 32, g.num_vertices());
  Context ctx({0, 0, 0});
  ShardedRepr sh(ctx, g, 32, g.num_vertices(), 2);
  std::int64_t cells = 0;
  for (auto c : sh.cells_per_rank()) cells += c;
  CHECK(cells == r.n_cells());
  for (Variant v : {Variant::selmax, Variant::tropical}) {
    BfsOptions o;
    o.variant = v;
    o.slimwork = true;
    o.slimchunk_len = 32;
    BfsResult a = bfs_spmv(sh, 11, o), b = bfs_spmv(r, 11, o);
    CHECK(a.dist == b.dist && a.iterations == b.iterations);
    if (v == Variant::selmax) CHECK(a.parent == b.parent);
    bool same = a.per_iter.size() == b.per_iter.size();
    for (std::size_t k = 0; same && k < a.per_iter.size(); ++k)
      same = a.per_iter[k].columns_processed == b.per_iter[k].columns_processed &&
             a.per_iter[k].chunks_skipped == b.per_iter[k].chunks_skipped &&
             a.per_iter[k].frontier_size == b.per_iter[k].frontier_size;
    CHECK(same);
  }
  CHECK_THROWS_AS(Context({0, 99}), std::invalid_argument);
}

int main() {
  context_sharded_bfs();
  host_layout_upload_and_segment();
  ingest_and_checks();
  csr_layout_of_path4();
  from_pairs_normalises();
  spec_layout_kats();
  spec_spmv_kats();
  spec_bfs_kats();
  kronecker_matches_oracle();
  std::printf("%d checks, %d failed\n", g_checks, g_failed);
  return g_failed ? 1 : 0;
}
