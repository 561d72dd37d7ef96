// Graph ingest: the edge-list and MatrixMarket
// readers of the reference (graph.hpp:50-59, graph.cpp:94-210), host-side
// text parsing feeding the device normalisation (Graph::from_pairs,
// edges_from_pairs). The accepted syntax, the error kinds and their messages
// follow the reference:
//   ParseError (graph.hpp:15-21)     -> SSB_EPARSE  "line N: ..."
//   std::invalid_argument            -> SSB_EINVAL
//   std::out_of_range                -> SSB_ERANGE
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdint>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "ssb_internal.cuh"

namespace ssb {
namespace {

[[noreturn]] void parse_fail(int64_t line, const std::string& what) {
  fail(SSB_EPARSE, "line " + std::to_string(line) + ": " + what);
}

inline bool is_space(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }

// Visits the lines of `text` (split at '\n', a trailing '\r' dropped) with
// 1-based numbers; like the reference, the empty remainder after a final
// newline is a line of its own.
template <typename Fn>
void lines(std::string_view text, Fn&& fn) {
  int64_t no = 0;
  size_t pos = 0;
  for (;;) {
    size_t end = text.find('\n', pos);
    const bool last = end == std::string_view::npos;
    if (last) end = text.size();
    std::string_view line = text.substr(pos, end - pos);
    if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
    fn(line, ++no);
    if (last) break;
    pos = end + 1;
  }
}

// '#' or '%' as the first non-blank character, or nothing but blanks
bool skippable(std::string_view line) {
  for (char c : line)
    if (!is_space(c)) return c == '#' || c == '%';
  return true;
}

void tokens(std::string_view line, std::vector<std::string_view>& out) {
  out.clear();
  size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && is_space(line[i])) ++i;
    const size_t b = i;
    while (i < line.size() && !is_space(line[i])) ++i;
    if (i > b) out.push_back(line.substr(b, i - b));
  }
}

// An unsigned decimal that fits int64 (vid_t).
int64_t vertex_id(std::string_view tok, int64_t line) {
  uint64_t v = 0;
  const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (r.ec == std::errc::result_out_of_range || v > uint64_t(INT64_MAX))
    fail(SSB_ERANGE, "line " + std::to_string(line) + ": vertex id out of range: " + std::string(tok));
  if (r.ec != std::errc() || r.ptr != tok.data() + tok.size())
    parse_fail(line, "expected unsigned integer, got '" + std::string(tok) + "'");
  return int64_t(v);
}

}  // namespace

// from_edge_list (graph.cpp:94-133): "u v" records, an optional leading
// "H n m" header, '#'/'%' comments. reject_asymmetric: every non-loop record
// needs its reverse.
void parse_edge_list(std::string_view text, int directive, std::vector<int64_t>& uv, int64_t& n) {
  uv.clear();
  n = -1;
  bool data = false;
  std::vector<std::string_view> t;
  lines(text, [&](std::string_view line, int64_t no) {
    if (skippable(line)) return;
    tokens(line, t);
    if (t[0] == "H") {
      if (data) parse_fail(no, "header after edge records");
      if (n >= 0) parse_fail(no, "duplicate header");
      if (t.size() != 3) parse_fail(no, "header needs 'H n m'");
      n = vertex_id(t[1], no);
      vertex_id(t[2], no);  // the declared m is informational
      return;
    }
    if (t.size() != 2)
      parse_fail(no, "expected 'u v', got " + std::to_string(t.size()) + " tokens");
    uv.push_back(vertex_id(t[0], no));
    uv.push_back(vertex_id(t[1], no));
    data = true;
  });
  if (directive == SSB_REJECT_ASYMMETRIC) {
    std::vector<std::pair<int64_t, int64_t>> arcs;
    arcs.reserve(uv.size() / 2);
    for (size_t i = 0; i < uv.size(); i += 2)
      if (uv[i] != uv[i + 1]) arcs.emplace_back(uv[i], uv[i + 1]);
    std::sort(arcs.begin(), arcs.end());
    arcs.erase(std::unique(arcs.begin(), arcs.end()), arcs.end());
    for (const auto& [a, b] : arcs)
      if (!std::binary_search(arcs.begin(), arcs.end(), std::make_pair(b, a)))
        fail(SSB_EINVAL, "asymmetric input: (" + std::to_string(a) + ", " + std::to_string(b) +
                             ") has no reverse record");
  } else if (directive != SSB_SYMMETRIZE) {
    fail(SSB_EINVAL, "bad input directive");
  }
}

// from_matrix_market (graph.cpp:135-210): coordinate pattern|real,
// general|symmetric, square, 1-based entries, the declared entry count.
void parse_matrix_market(std::string_view text, std::vector<int64_t>& uv, int64_t& n) {
  uv.clear();
  bool banner = false, sized = false, symmetric = false, pattern = false;
  int64_t rows = 0, declared = 0, seen = 0;
  std::vector<std::string_view> t;
  lines(text, [&](std::string_view line, int64_t no) {
    if (!banner) {
      tokens(line, t);
      if (t.size() < 5 || t[0] != "%%MatrixMarket" || t[1] != "matrix")
        parse_fail(no, "missing '%%MatrixMarket matrix' banner");
      if (t[2] != "coordinate")
        fail(SSB_EINVAL, "unsupported MatrixMarket format '" + std::string(t[2]) + "' (need coordinate)");
      if (t[3] == "pattern") pattern = true;
      else if (t[3] != "real")
        fail(SSB_EINVAL,
             "unsupported MatrixMarket field '" + std::string(t[3]) + "' (need pattern or real)");
      if (t[4] == "symmetric") symmetric = true;
      else if (t[4] != "general")
        fail(SSB_EINVAL, "unsupported MatrixMarket symmetry '" + std::string(t[4]) +
                             "' (need general or symmetric)");
      banner = true;
      return;
    }
    if (skippable(line)) return;
    tokens(line, t);
    if (!sized) {
      if (t.size() != 3) parse_fail(no, "expected 'rows cols nnz'");
      rows = vertex_id(t[0], no);
      const int64_t cols = vertex_id(t[1], no);
      declared = vertex_id(t[2], no);
      if (rows != cols)
        fail(SSB_EINVAL, "adjacency matrix must be square, got " + std::to_string(rows) + "x" +
                             std::to_string(cols));
      sized = true;
      return;
    }
    const size_t want = pattern ? 2 : 3;
    if (t.size() != want) parse_fail(no, "expected " + std::to_string(want) + " tokens");
    const int64_t i = vertex_id(t[0], no), j = vertex_id(t[1], no);
    if (i < 1 || i > rows || j < 1 || j > rows)
      fail(SSB_ERANGE, "line " + std::to_string(no) + ": entry outside matrix bounds");
    if (++seen > declared) return;  // counted, reported below
    uv.push_back(i - 1);
    uv.push_back(j - 1);
    if (symmetric) {
      uv.push_back(j - 1);
      uv.push_back(i - 1);
    }
  });
  if (!banner) parse_fail(1, "empty MatrixMarket input");
  if (!sized) parse_fail(1, "missing MatrixMarket size line");
  if (seen != declared)
    fail(SSB_EINVAL, "MatrixMarket entry count mismatch: header says " + std::to_string(declared) +
                         ", found " + std::to_string(seen));
  n = rows;
}

}  // namespace ssb
