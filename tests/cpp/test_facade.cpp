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

int main() {
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
