// Device-side BFS checking for large graphs: at S26+
// the host oracle needs hundreds of GB and tens of minutes, so parity at scale
// is established on the device by
//   * bfs_traditional — an independent level-synchronous queue BFS over the
//     CSR of ORIGINAL ids (no SlimSell layout, no bitmaps), with the
//     reference's parent rule: the smallest-id neighbour one level closer
//     (bfs.cpp:248-286 scans an ascending frontier, so the first discoverer is
//     that neighbour);
//   * validate_bfs — the checks of the reference's verify_against_oracle
//     (cli.cpp:73-112: unreached ⇒ no parent, root self-parented, parent is a
//     neighbour one level closer) plus the Graph500 edge checks that stand in
//     for the oracle's distances (every edge joins levels at most 1 apart and
//     never a reached and an unreached vertex; only the root has level 0).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include <cstdlib>
#include "ssb_internal.cuh"

namespace ssb {
namespace {

constexpr int32_t kInf32 = 0x7fffffff;

int grid_for(int64_t items, int threads = 256) {
  const int64_t want = (items + threads - 1) / threads;
  const int64_t cap = int64_t(num_sms()) * 32;
  return int(want < 1 ? 1 : (want > cap ? cap : want));
}

#define GRID_LOOP(i, count)                                                              \
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x, _s = int64_t(gridDim.x) * \
                                                                        blockDim.x;       \
       i < (count); i += _s)

__global__ void both_arcs_kernel(const uint64_t* __restrict__ keys, int64_t m, int bits,
                                 uint64_t* __restrict__ arcs) {
  const uint64_t mask = (uint64_t{1} << bits) - 1;
  GRID_LOOP(i, m) {
    const uint64_t u = keys[i] >> bits, v = keys[i] & mask;
    arcs[2 * i] = (u << bits) | v;
    arcs[2 * i + 1] = (v << bits) | u;
  }
}

__global__ void endpoint_degree_kernel(const uint64_t* __restrict__ keys, int64_t m, int bits,
                                       int64_t* __restrict__ deg) {
  const uint64_t mask = (uint64_t{1} << bits) - 1;
  GRID_LOOP(i, m) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&deg[keys[i] >> bits]), 1ull);
    atomicAdd(reinterpret_cast<unsigned long long*>(&deg[keys[i] & mask]), 1ull);
  }
}

// arcs (u, v) with u in [u0, u1), compacted through a warp-aggregated counter
__global__ void range_arcs_kernel(const uint64_t* __restrict__ keys, int64_t m, int bits, int64_t u0,
                                  int64_t u1, unsigned long long* __restrict__ count,
                                  uint64_t* __restrict__ arcs) {
  const uint64_t mask = (uint64_t{1} << bits) - 1;
  const int lane = threadIdx.x & 31;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < m; base += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    uint64_t u = 0, v = 0;
    bool a0 = false, a1 = false;
    if (i < m) {
      u = keys[i] >> bits;
      v = keys[i] & mask;
      a0 = int64_t(u) >= u0 && int64_t(u) < u1;
      a1 = int64_t(v) >= u0 && int64_t(v) < u1;
    }
    const int mine = int(a0) + int(a1);
    int incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long at = 0;
    if (lane == 31 && total) at = atomicAdd(count, (unsigned long long)total);
    at = __shfl_sync(0xffffffffu, at, 31) + uint64_t(incl - mine);
    if (a0) arcs[at++] = (u << bits) | v;
    if (a1) arcs[at] = (v << bits) | u;
  }
}

__global__ void low_bits_kernel(const uint64_t* __restrict__ arcs, int64_t na, int bits,
                                int32_t* __restrict__ col) {
  const uint64_t mask = (uint64_t{1} << bits) - 1;
  GRID_LOOP(i, na) col[i] = int32_t(arcs[i] & mask);
}

// ---- queue BFS -------------------------------------------------------------

__global__ void qbfs_init_kernel(int32_t* __restrict__ dist, int64_t n, int32_t root) {
  GRID_LOOP(v, n) dist[v] = v == root ? 0 : kInf32;
}

// One warp per frontier vertex: its neighbours are claimed with a CAS on dist.
__global__ void qbfs_level_kernel(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                                  int32_t* __restrict__ dist, const int32_t* __restrict__ q,
                                  int64_t qn, int32_t* __restrict__ next,
                                  unsigned long long* __restrict__ next_n, int32_t level) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; i < qn; i += warps) {
    const int32_t u = q[i];
    for (int64_t e = row[u] + lane; e < row[u + 1]; e += 32) {
      const int32_t w = col[e];
      if (dist[w] == kInf32 && atomicCAS(&dist[w], kInf32, level) == kInf32)
        next[atomicAdd(next_n, 1ull)] = w;
    }
  }
}

// parent[v] = the smallest neighbour one level closer (rows are ascending, so
// the first found); the root is its own parent; unreached: -1.
__global__ void qbfs_parent_kernel(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                                   const int32_t* __restrict__ dist, int64_t n, int32_t root,
                                   int64_t* __restrict__ dist_out, int64_t* __restrict__ parent) {
  GRID_LOOP(v, n) {
    const int32_t d = dist[v];
    int64_t p = -1;
    if (v == root) {
      p = root;
    } else if (d != kInf32) {
      for (int64_t e = row[v]; e < row[v + 1]; ++e)
        if (dist[col[e]] == d - 1) {
          p = col[e];
          break;
        }
    }
    dist_out[v] = d == kInf32 ? INT64_MAX : int64_t(d);
    if (parent) parent[v] = p;
  }
}

// ---- validator ---------------------------------------------------------------

enum : int32_t {
  kVRootLevel = 1,       // dist[root] != 0
  kVZeroNotRoot = 2,     // another vertex at level 0
  kVEdgeSpan = 3,        // an edge joins levels more than 1 apart
  kVEdgeReach = 4,       // an edge joins a reached and an unreached vertex
  kVUnreachedParent = 5, // unreached but parent set
  kVRootParent = 6,      // root not self-parented
  kVParentRange = 7,     // parent outside [0, n) or not a neighbour
  kVParentLevel = 8,     // parent not one level closer
  kVParentExact = 9,     // parent differs from the reference's deterministic rule
};

struct Violations {
  unsigned long long count;
  int64_t first_v[4];  // vertex (or edge index) of the first few violations
  int32_t first_code[4];
  int64_t first_x[4];  // the offending parent / other endpoint
};

__device__ void report(Violations* out, int32_t code, int64_t v, int64_t x) {
  const unsigned long long i = atomicAdd(&out->count, 1ull);
  if (i < 4) {
    out->first_v[i] = v;
    out->first_code[i] = code;
    out->first_x[i] = x;
  }
}

__global__ void check_edges_kernel(const uint64_t* __restrict__ keys, int64_t m, int bits,
                                   const int64_t* __restrict__ dist, Violations* out) {
  const uint64_t mask = (uint64_t{1} << bits) - 1;
  GRID_LOOP(i, m) {
    const int64_t u = int64_t(keys[i] >> bits), v = int64_t(keys[i] & mask);
    const int64_t du = dist[u], dv = dist[v];
    const bool ru = du != INT64_MAX, rv = dv != INT64_MAX;
    if (ru != rv) report(out, kVEdgeReach, u, v);
    else if (ru && (du - dv > 1 || dv - du > 1)) report(out, kVEdgeSpan, u, v);
  }
}

__device__ bool has_edge(const int64_t* row, const int32_t* col, int64_t p, int64_t v) {
  int64_t lo = row[p], hi = row[p + 1];
  while (lo < hi) {  // col is ascending within a row
    const int64_t mid = (lo + hi) >> 1;
    if (col[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo < row[p + 1] && col[lo] == v;
}

__global__ void check_vertices_kernel(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                                      int64_t n, int64_t root, const int64_t* __restrict__ dist,
                                      const int64_t* __restrict__ parent, int flags, Violations* out) {
  GRID_LOOP(v, n) {
    const int64_t d = dist[v];
    if (v == root && d != 0) report(out, kVRootLevel, v, d);
    if (v != root && d == 0) report(out, kVZeroNotRoot, v, d);
    if (!parent) continue;
    const int64_t p = parent[v];
    if (d == INT64_MAX) {
      if (p != -1) report(out, kVUnreachedParent, v, p);
      continue;
    }
    // the reference's sel-max root encoding gives the
    // root and its depth-1 vertices the parent perm[root]: not a tree edge
    // (exact_parent_kernel checks that value when asked to)
    if ((flags & SSB_VALIDATE_SELMAX_COMPAT) && d <= 1) continue;
    if (d == 0) {
      if (p != v) report(out, kVRootParent, v, p);
      continue;
    }
    if (p < 0 || p >= n || !has_edge(row, col, p, v)) {
      report(out, kVParentRange, v, p);
      continue;
    }
    if (dist[p] != d - 1) report(out, kVParentLevel, v, p);
  }
}

// The exact parent every reference variant returns (one warp per vertex,
// the neighbour list scanned 32 at a time — hub rows hold 1M neighbours):
//   min rule  (tropical / real / boolean, dp_transform semiring.cpp:159-187,
//             == bfs_traditional's first discoverer):
//             the smallest ORIGINAL-id neighbour one level closer;
//   sel-max   (selmax_parents bfs.cpp:94-101, App. A.3):
//             perm[max{inv_perm[u] : u ∈ N(v), d(u) = d(v) − 1}], and with
//             the reference's root encoding (compat) perm[root] at levels 0-1.
// The root is its own parent (min rule, sel-max without compat). Reached
// vertices only; unreached ones are checked by check_vertices_kernel.
__global__ void exact_parent_kernel(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                                    int64_t n, int64_t root, const int64_t* __restrict__ dist,
                                    const int64_t* __restrict__ parent, const int32_t* __restrict__ perm,
                                    const int32_t* __restrict__ inv_perm, int flags, Violations* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const bool sel = (flags & SSB_VALIDATE_SELMAX_EXACT) != 0;
  const bool compat = sel && (flags & SSB_VALIDATE_SELMAX_COMPAT) != 0;
  for (int64_t v = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    const int64_t d = dist[v];
    if (d == INT64_MAX) continue;
    int64_t want;
    if (compat && d <= 1) {
      want = perm[root];
    } else if (d == 0) {
      want = v;
    } else {
      // min rule: smallest id; sel-max: largest position (-1 = none found)
      int64_t best = sel ? -1 : INT64_MAX;
      for (int64_t e = row[v] + lane; e < row[v + 1]; e += 32) {
        const int32_t u = col[e];
        if (dist[u] != d - 1) continue;
        if (sel) best = max(best, int64_t(inv_perm[u]));
        else best = min(best, int64_t(u));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t b = __shfl_xor_sync(0xffffffffu, best, o);
        best = sel ? max(best, b) : min(best, b);
      }
      want = sel ? (best < 0 ? -2 : int64_t(perm[best])) : (best == INT64_MAX ? -2 : best);
    }
    if (lane == 0 && parent[v] != want) report(out, kVParentExact, v, want);
  }
}

}  // namespace

// Device CSR of the normalised edge set (original ids, rows ascending),
// cached on the handle: the validator and the queue BFS share it.
struct DevCsr {
  int64_t n = 0, na = 0;
  DevBuf<int64_t> row;  // n + 1
  DevBuf<int32_t> col;  // 2m
};

// Rows from the endpoint degrees, then the arcs sorted and written in passes
// over row ranges sized to the free memory (one pass up to ~S26; S28's 8.4e9
// arcs would need 135 GB of sort buffers at once).
static DevCsr& device_csr(ssb_edges& e) {
  if (e.csr) return *static_cast<DevCsr*>(e.csr.get());
  if (e.n >= (int64_t{1} << 31)) fail(SSB_EINVAL, "device CSR supports n < 2^31");
  auto c = std::make_shared<DevCsr>();
  cudaStream_t s = e.sc.s;
  c->n = e.n;
  c->na = 2 * e.m;
  c->row.alloc(size_t(e.n + 1));
  c->col.alloc(size_t(std::max<int64_t>(c->na, 1)));
  {
    DevBuf<int64_t> deg{size_t(std::max<int64_t>(e.n, 1))};
    SSB_CUDA(cudaMemsetAsync(deg.p, 0, deg.bytes(), s));
    if (e.m > 0) endpoint_degree_kernel<<<grid_for(e.m), 256, 0, s>>>(e.keys.p, e.m, e.bits, deg.p);
    SSB_CUDA(cudaGetLastError());
    SSB_CUDA(cudaMemsetAsync(c->row.p, 0, 8, s));
    if (e.n > 0) {
      size_t tb = 0;
      SSB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, deg.p, c->row.p + 1, e.n, s));
      DevBuf<uint8_t> tmp(tb);
      SSB_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, deg.p, c->row.p + 1, e.n, s));
    }
    e.sc.sync();
  }
  if (c->na > 0) {
    std::vector<int64_t> row(size_t(e.n + 1));
    SSB_CUDA(cudaMemcpy(row.data(), c->row.p, 8 * row.size(), cudaMemcpyDeviceToHost));
    size_t free_b = 0, tot_b = 0;
    SSB_CUDA(cudaMemGetInfo(&free_b, &tot_b));
    const char* ev = std::getenv("SSB_ARCS_PER_PASS");
    const int64_t per_pass = ev ? std::max<int64_t>(std::atoll(ev), 1)
                                : std::max<int64_t>(int64_t(double(free_b) * 0.6 / 20.0), 1 << 20);
    int64_t u0 = 0;
    while (u0 < e.n) {
      // the largest row range starting at u0 whose arcs fit a pass (>= 1 row)
      const int64_t lim = row[size_t(u0)] + per_pass;
      int64_t u1 = int64_t(std::upper_bound(row.begin() + u0 + 1, row.end(), lim) - row.begin()) - 1;
      u1 = std::max<int64_t>(u1, u0 + 1);
      const int64_t na = row[size_t(u1)] - row[size_t(u0)];
      if (na > 0) {
        DevBuf<uint64_t> arcs{size_t(na)}, alt{size_t(na)};
        if (u0 == 0 && u1 == e.n) {
          both_arcs_kernel<<<grid_for(e.m), 256, 0, s>>>(e.keys.p, e.m, e.bits, arcs.p);
        } else {
          DevBuf<unsigned long long> cnt(1);
          SSB_CUDA(cudaMemsetAsync(cnt.p, 0, 8, s));
          range_arcs_kernel<<<grid_for(e.m), 256, 0, s>>>(e.keys.p, e.m, e.bits, u0, u1, cnt.p, arcs.p);
        }
        SSB_CUDA(cudaGetLastError());
        cub::DoubleBuffer<uint64_t> db(arcs.p, alt.p);
        size_t tb = 0;
        SSB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, na, 0, 2 * e.bits, s));
        {
          DevBuf<uint8_t> tmp(tb);
          SSB_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, db, na, 0, 2 * e.bits, s));
          low_bits_kernel<<<grid_for(na), 256, 0, s>>>(db.Current(), na, e.bits, c->col.p + row[size_t(u0)]);
          SSB_CUDA(cudaGetLastError());
          e.sc.sync();
        }
      }
      u0 = u1;
    }
  }
  e.sc.sync();
  e.csr = c;
  return *c;
}

int64_t bfs_traditional(ssb_edges& e, int64_t root, int64_t* dist, int64_t* parent,
                        std::vector<ssb_iter_stats>& per_iter) {
  // bfs.cpp:250-253
  if (root < 0 || root >= e.n)
    fail(SSB_ERANGE, "root " + std::to_string(root) + " outside [0, " + std::to_string(e.n) + ")");
  DevCsr& c = device_csr(e);
  cudaStream_t s = e.sc.s;
  const int64_t n = e.n;
  DevBuf<int32_t> d{size_t(n)}, q0{size_t(n)}, q1{size_t(n)};
  DevBuf<unsigned long long> cnt(1);
  qbfs_init_kernel<<<grid_for(n), 256, 0, s>>>(d.p, n, int32_t(root));
  const int32_t r32 = int32_t(root);
  SSB_CUDA(cudaMemcpyAsync(q0.p, &r32, 4, cudaMemcpyHostToDevice, s));
  int64_t qn = 1, k = 0;
  int32_t *q = q0.p, *next = q1.p;
  cudaEvent_t t0, t1;
  SSB_CUDA(cudaEventCreate(&t0));
  SSB_CUDA(cudaEventCreate(&t1));
  while (qn > 0) {  // the reference's loop: k counts levels incl. the empty last one
    ++k;
    SSB_CUDA(cudaMemsetAsync(cnt.p, 0, 8, s));
    SSB_CUDA(cudaEventRecord(t0, s));
    const int64_t blocks = std::min<int64_t>((qn * 32 + 255) / 256, int64_t(num_sms()) * 16);
    qbfs_level_kernel<<<int(std::max<int64_t>(blocks, 1)), 256, 0, s>>>(c.row.p, c.col.p, d.p, q, qn,
                                                                        next, cnt.p, int32_t(k));
    SSB_CUDA(cudaGetLastError());
    SSB_CUDA(cudaEventRecord(t1, s));
    unsigned long long nn = 0;
    SSB_CUDA(cudaMemcpyAsync(&nn, cnt.p, 8, cudaMemcpyDeviceToHost, s));
    e.sc.sync();
    float ms = 0;
    SSB_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    ssb_iter_stats st{};
    st.iteration = k;
    st.frontier_size = int64_t(nn);
    st.elapsed_ns = int64_t(double(ms) * 1e6);
    per_iter.push_back(st);
    qn = int64_t(nn);
    std::swap(q, next);
  }
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  DevBuf<int64_t> dd{size_t(n)}, pp{parent ? size_t(n) : size_t(0)};
  qbfs_parent_kernel<<<grid_for(n), 256, 0, s>>>(c.row.p, c.col.p, d.p, n, int32_t(root), dd.p,
                                                 parent ? pp.p : nullptr);
  SSB_CUDA(cudaGetLastError());
  SSB_CUDA(cudaMemcpyAsync(dist, dd.p, 8 * n, cudaMemcpyDeviceToHost, s));
  if (parent) SSB_CUDA(cudaMemcpyAsync(parent, pp.p, 8 * n, cudaMemcpyDeviceToHost, s));
  e.sc.sync();
  return k;
}

int64_t validate_bfs(ssb_edges& e, int64_t root, const int64_t* dist, const int64_t* parent,
                     int flags, std::string& report_text, const ssb_graph* layout) {
  if (root < 0 || root >= e.n)
    fail(SSB_ERANGE, "root " + std::to_string(root) + " outside [0, " + std::to_string(e.n) + ")");
  DevCsr& c = device_csr(e);
  cudaStream_t s = e.sc.s;
  const int64_t n = e.n;
  DevBuf<int64_t> dd{size_t(n)}, pp{parent ? size_t(n) : size_t(0)};
  DevBuf<Violations> vv(1);
  SSB_CUDA(cudaMemcpyAsync(dd.p, dist, 8 * n, cudaMemcpyHostToDevice, s));
  if (parent) SSB_CUDA(cudaMemcpyAsync(pp.p, parent, 8 * n, cudaMemcpyHostToDevice, s));
  SSB_CUDA(cudaMemsetAsync(vv.p, 0, sizeof(Violations), s));
  if (e.m > 0) check_edges_kernel<<<grid_for(e.m), 256, 0, s>>>(e.keys.p, e.m, e.bits, dd.p, vv.p);
  check_vertices_kernel<<<grid_for(n), 256, 0, s>>>(c.row.p, c.col.p, n, root, dd.p,
                                                    parent ? pp.p : nullptr, flags, vv.p);
  SSB_CUDA(cudaGetLastError());
  if (parent && (flags & (SSB_VALIDATE_SELMAX_EXACT | SSB_VALIDATE_MIN_PARENT_EXACT))) {
    if ((flags & SSB_VALIDATE_SELMAX_EXACT) && (flags & SSB_VALIDATE_MIN_PARENT_EXACT))
      fail(SSB_EINVAL, "SSB_VALIDATE_SELMAX_EXACT and SSB_VALIDATE_MIN_PARENT_EXACT exclude each other");
    const int32_t *perm = nullptr, *inv = nullptr;
    if (flags & SSB_VALIDATE_SELMAX_EXACT) {
      if (!layout) fail(SSB_EINVAL, "SSB_VALIDATE_SELMAX_EXACT needs the layout (perm / inv_perm)");
      if (layout->n != n) fail(SSB_EINVAL, "layout and edge set have different vertex counts");
      perm = layout->perm.p;
      inv = layout->inv_perm.p;
    }
    exact_parent_kernel<<<grid_for(n * 32), 256, 0, s>>>(c.row.p, c.col.p, n, root, dd.p, pp.p, perm, inv,
                                                         flags, vv.p);
    SSB_CUDA(cudaGetLastError());
  }
  Violations h{};
  SSB_CUDA(cudaMemcpyAsync(&h, vv.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  e.sc.sync();
  report_text.clear();
  static const char* what[] = {"",
                               "root not at level 0",
                               "non-root vertex at level 0",
                               "edge joins levels more than 1 apart",
                               "edge joins a reached and an unreached vertex",
                               "unreached but parent set",
                               "root not self-parented",
                               "parent is not a neighbor",
                               "parent not one level closer",
                               "parent differs from the reference rule; expected"};
  for (int i = 0; i < int(std::min<unsigned long long>(h.count, 4)); ++i) {
    char buf[160];
    const int32_t code = h.first_code[i];
    if (code == kVEdgeSpan || code == kVEdgeReach)
      std::snprintf(buf, sizeof buf, "  edge (%lld, %lld): %s\n", (long long)h.first_v[i],
                    (long long)h.first_x[i], what[code]);
    else
      std::snprintf(buf, sizeof buf, "  vertex %lld: %s (%lld)\n", (long long)h.first_v[i],
                    what[code], (long long)h.first_x[i]);
    report_text += buf;
  }
  return int64_t(h.count);
}

}  // namespace ssb
