// The façade and the UNMODIFIED reference in one translation unit and one
// binary: the mixed use INTEGRATION.md describes for a caller that keeps the
// reference's host builder (cli.cpp:195) and hands its layout to the device.
// Test infrastructure (it links oracle/_ref/libslimsell_ref.so, the reference
// compiled from its own sources); built by oracle/Makefile target
// `alongside` next to that library, so it travels to the GPU box prebuilt.
//
//   slimsell::X        — the reference's X (its headers)
//   slimsell::b200::X  — the façade's X (SLIMSELL_B200_ALONGSIDE_REFERENCE)
//
// Every check compares the device result with the reference's own call on the
// same host objects: bfs_spmv over the reference-built layout for every
// semiring and SlimWork/SlimChunk setting (dist, parents, per-iteration
// counters), the layout mutated in place as cli.cpp:200-207's corrupt_repr
// does (re-uploaded through the fingerprint), spmv_step / spmv_segment with
// the reference's SemiringSpec, and bfs_traditional on the reference's CSR.
#include <slimsell/bfs.hpp>
#include <slimsell/generator.hpp>
#include <slimsell/graph.hpp>
#include <slimsell/repr.hpp>
#include <slimsell/semiring.hpp>

#define SLIMSELL_B200_ALONGSIDE_REFERENCE
#include "slimsell_b200/slimsell.hpp"

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace ref = slimsell;
namespace dev = slimsell::b200;

static int g_failed = 0, g_checks = 0;
#define CHECK(cond, ...)                                                        \
  do {                                                                          \
    ++g_checks;                                                                 \
    if (!(cond)) {                                                              \
      ++g_failed;                                                               \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed ", __FILE__, __LINE__, #cond); \
      std::fprintf(stderr, __VA_ARGS__);                                        \
      std::fprintf(stderr, "\n");                                               \
    }                                                                           \
  } while (0)

static bool same_counters(const ref::BfsResult& a, const dev::BfsResult& b) {
  if (a.iterations != b.iterations || a.per_iter.size() != b.per_iter.size()) return false;
  for (std::size_t i = 0; i < a.per_iter.size(); ++i) {
    const auto& x = a.per_iter[i];
    const auto& y = b.per_iter[i];
    if (x.iteration != y.iteration || x.chunks_processed != y.chunks_processed ||
        x.chunks_skipped != y.chunks_skipped || x.subchunks_processed != y.subchunks_processed ||
        x.columns_processed != y.columns_processed || x.frontier_size != y.frontier_size)
      return false;
  }
  return true;
}

static std::vector<ref::vid_t> some_roots(const ref::CsrView& csr, int want) {
  std::vector<ref::vid_t> out;
  const ref::vid_t n = static_cast<ref::vid_t>(csr.row.size()) - 1;
  for (ref::vid_t v = 0; v < n && static_cast<int>(out.size()) < want; v += 1 + n / (2 * want))
    if (csr.row[v + 1] > csr.row[v]) out.push_back(v);
  return out;
}

// bfs_spmv on the reference's host layout, every semiring, SlimWork on/off,
// SlimChunk off/64: dist, parents (the reference's dp_transform over its own
// CsrView, or sel-max's encoding) and the counters equal.
static void bfs_on_reference_layout(const ref::Graph& g, const ref::CsrView& csr, std::int64_t C,
                                    std::int64_t sigma, const char* tag) {
  const ref::SlimSellRepr host = ref::build_slimsell(g, C, sigma);
  for (const ref::vid_t root : some_roots(csr, 4)) {
    for (int v = 0; v < 4; ++v) {
      for (const bool sw : {false, true}) {
        for (const std::int64_t L : {std::int64_t{0}, std::int64_t{64}}) {
          ref::BfsOptions ro;
          ro.variant = static_cast<ref::Variant>(v);
          ro.slimwork = sw;
          ro.slimchunk_len = L;
          dev::BfsOptions o;
          o.variant = static_cast<dev::Variant>(v);
          o.slimwork = sw;
          o.slimchunk_len = L;
          const ref::BfsResult a = ref::bfs_spmv(host, root, ro, &csr);
          const dev::BfsResult b = dev::bfs_spmv(host, root, o, &csr);  // the reference's CsrView
          CHECK(a.dist == b.dist, "%s dist root %lld variant %d sw %d L %lld", tag, (long long)root, v,
                int(sw), (long long)L);
          CHECK(a.parent == b.parent, "%s parent root %lld variant %d", tag, (long long)root, v);
          CHECK(same_counters(a, b), "%s IterStats root %lld variant %d", tag, (long long)root, v);
        }
      }
    }
  }
}

// cli.cpp:200-207: the first real cell of col is rewritten in place after the
// build; the façade's cache must notice (fingerprint) and the device must see
// the corrupted layout exactly as the reference's bfs_spmv does.
static void corrupted_layout_in_place(const ref::Graph& g, const ref::CsrView& csr) {
  ref::SlimSellRepr host = ref::build_slimsell(g, 32, g.num_vertices());
  const ref::vid_t n = g.num_vertices();
  dev::BfsOptions o;
  o.variant = dev::Variant::selmax;
  o.slimwork = true;
  ref::BfsOptions ro;
  ro.variant = ref::Variant::selmax;
  ro.slimwork = true;
  (void)dev::bfs_spmv(host, some_roots(csr, 1)[0], o);  // cached upload of the clean layout
  for (auto& c : host.col) {
    if (c >= 0) {
      c = (c + 1) % n;
      break;
    }
  }
  for (const ref::vid_t r : some_roots(csr, 8)) {
    const ref::BfsResult a = ref::bfs_spmv(host, r, ro);
    const dev::BfsResult b = dev::bfs_spmv(host, r, o);
    CHECK(a.dist == b.dist && a.parent == b.parent && same_counters(a, b),
          "corrupted layout root %lld", (long long)r);
    // tropical with the (uncorrupted) CSR for dp_transform's parents
    ref::BfsOptions rt;
    rt.slimwork = true;
    dev::BfsOptions t;
    t.slimwork = true;
    const ref::BfsResult c = ref::bfs_spmv(host, r, rt, &csr);
    const dev::BfsResult d = dev::bfs_spmv(host, r, t, &csr);
    CHECK(c.dist == d.dist && same_counters(c, d), "corrupted layout tropical root %lld", (long long)r);
    CHECK(c.parent == d.parent, "corrupted layout tropical parents root %lld", (long long)r);
  }
}

// repr.hpp:90-98 / 79-81 with the reference's SemiringSpec.
static void spmv_with_reference_semiring(const ref::Graph& g) {
  const ref::SlimSellRepr host = ref::build_slimsell(g, 8, 64);
  std::uint64_t s = 0x9E3779B97F4A7C15ull;
  for (int v = 0; v < 4; ++v) {
    const ref::SemiringSpec& sr = ref::semiring(static_cast<ref::Variant>(v));
    std::vector<ref::val_t> x(host.n_padded);
    for (auto& e : x) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      e = sr.sample_scalar(s);
    }
    const std::vector<ref::val_t> a = ref::spmv_step(host, sr, x);
    const std::vector<ref::val_t> b = dev::spmv_step(host, sr, x);
    CHECK(a == b, "spmv_step variant %d", v);
    for (const std::int64_t k : {std::int64_t{0}, host.n_chunks / 2, host.n_chunks - 1}) {
      const std::int64_t len = host.cl[k];
      std::vector<ref::val_t> acc_a(host.C, sr.zero), acc_b(host.C, sr.zero);
      ref::spmv_segment(host, sr, x, acc_a, k, len / 3, len - len / 3);
      dev::spmv_segment(host, sr, x, acc_b, k, len / 3, len - len / 3);
      CHECK(acc_a == acc_b, "spmv_segment variant %d chunk %lld", v, (long long)k);
    }
  }
}

// bfs.hpp:85 on the reference's CsrView.
static void traditional_on_reference_csr(const ref::CsrView& csr) {
  for (const ref::vid_t root : some_roots(csr, 4)) {
    const ref::BfsResult a = ref::bfs_traditional(csr, root);
    const dev::BfsResult b = dev::bfs_traditional(csr, root);
    CHECK(a.dist == b.dist && a.parent == b.parent, "bfs_traditional root %lld", (long long)root);
  }
}

int main() {
  if (ssb_set_device(0) != SSB_OK) {  // built and linked here; run on a B200
    std::printf("no device: %s\n", ssb_last_error());
    return 0;
  }
  const ref::Graph kron = ref::gen_kronecker(12, 16, 1);
  const ref::CsrView kcsr = ref::to_csr(kron);
  bfs_on_reference_layout(kron, kcsr, 32, kron.num_vertices(), "kron12 C32");
  bfs_on_reference_layout(kron, kcsr, 8, 64, "kron12 C8 s64");
  const ref::Graph er = ref::gen_erdos_renyi(3000, 4.0 / 2999, 7);
  const ref::CsrView ecsr = ref::to_csr(er);
  bfs_on_reference_layout(er, ecsr, 32, er.num_vertices(), "er3000 C32");
  corrupted_layout_in_place(kron, kcsr);
  spmv_with_reference_semiring(kron);
  traditional_on_reference_csr(kcsr);
  traditional_on_reference_csr(ecsr);
  std::printf("alongside reference: %d checks, %d failed\n", g_checks, g_failed);
  return g_failed ? 1 : 0;
}
