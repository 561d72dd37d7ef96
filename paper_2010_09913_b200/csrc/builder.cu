// SlimSell builder on the device (north_star subsystem 1).
//
// Reference: make_sort_plan (repr.cpp:62-82) and build_slimsell
// (repr.cpp:84-131). Same output bit for bit:
//   σ_eff = min(σ, max(n,1)); windows [w, w+σ_eff) sorted by (deg desc, id asc)
//   -> perm / inv_perm; cl[i] = max degree of chunk i's real rows;
//   cs = exclusive prefix of C·cl; col[cs[i] + k·C + lane] = k-th smallest
//   inv_perm[nbr] of row i·C+lane, else -1.
// B200 pipeline: degree histogram (atomics) -> one stable radix sort of
// (window, ~deg) keys carrying ids -> chunk max + scans -> one radix sort of
// the 2m arcs keyed (row position, neighbour position) -> rank-within-row
// scatter into the column-major chunk grid. Every stage streams HBM; nothing
// here is a GEMM.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <memory>

#include "ssb_internal.cuh"

namespace ssb {
namespace {

int bits_for_value(uint64_t v) {  // bits to hold values in [0, v]
  int b = 1;
  while (b < 64 && (uint64_t{1} << b) <= v) ++b;
  return b;
}

// SSB_ARCS_PER_PASS: arcs sorted per builder pass (tests force several passes)
int64_t env_arcs_per_pass() {
  const char* v = std::getenv("SSB_ARCS_PER_PASS");
  return v ? std::atoll(v) : 0;
}

int grid_for(int64_t items, int threads = 256) {
  const int64_t want = (items + threads - 1) / threads;
  const int64_t cap = int64_t(num_sms()) * 32;
  return int(want < 1 ? 1 : (want > cap ? cap : want));
}

#define GRID_STRIDE(i, count)                                                       \
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < (count); \
       i += int64_t(gridDim.x) * blockDim.x)

__global__ void degree_kernel(const uint64_t* __restrict__ keys, int64_t m, int bits,
                              int32_t* __restrict__ deg) {
  const uint64_t mask = (uint64_t{1} << bits) - 1;
  GRID_STRIDE(i, m) {
    atomicAdd(&deg[keys[i] >> bits], 1);
    atomicAdd(&deg[keys[i] & mask], 1);
  }
}

__global__ void max_reduce_kernel(const int32_t* __restrict__ v, int64_t n,
                                  int* __restrict__ out) {
  int mx = 0;
  GRID_STRIDE(i, n) mx = max(mx, v[i]);
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// make_sort_plan key: window in the high bits, (maxdeg - deg) below, so an
// ascending STABLE sort of ids 0..n-1 yields (window, deg desc, id asc).
__global__ void sort_keys_kernel(const int32_t* __restrict__ deg, int64_t n, int64_t sigma,
                                 int dbits, int32_t maxdeg, uint64_t* __restrict__ keys,
                                 int32_t* __restrict__ ids) {
  GRID_STRIDE(v, n) {
    const uint64_t w = uint64_t(v / sigma);
    keys[v] = (w << dbits) | uint64_t(maxdeg - deg[v]);
    ids[v] = int32_t(v);
  }
}

__global__ void iota_kernel(int32_t* __restrict__ a, int64_t n) {
  GRID_STRIDE(i, n) a[i] = int32_t(i);
}

__global__ void perm_derive_kernel(const int32_t* __restrict__ perm, int64_t n,
                                   int64_t n_padded, const int32_t* __restrict__ deg,
                                   int32_t* __restrict__ inv_perm,
                                   int32_t* __restrict__ deg_perm) {
  GRID_STRIDE(p, n_padded) {
    if (p < n) {
      const int32_t o = perm[p];
      inv_perm[o] = int32_t(p);
      deg_perm[p] = deg[o];
    } else {
      deg_perm[p] = 0;
    }
  }
}

// cl for every chunk; cells only for the chunks the handle holds (held[i],
// null = all): a shard of a multi-GPU layout holds just its own cells
//
__global__ void chunk_len_kernel(const int32_t* __restrict__ deg_perm, int64_t n_chunks,
                                 int64_t C, const uint8_t* __restrict__ held, int32_t* __restrict__ cl,
                                 int64_t* __restrict__ cells) {
  GRID_STRIDE(i, n_chunks) {
    int32_t mx = 0;
    for (int64_t l = 0; l < C; ++l) mx = max(mx, deg_perm[i * C + l]);
    cl[i] = mx;
    cells[i] = !held || held[i] ? int64_t(mx) * C : 0;
  }
}

// row degrees of the held rows in [r0, r1) (arc offsets of a pass), 0 elsewhere
__global__ void range_deg_kernel(const int32_t* __restrict__ deg_perm, int64_t n_padded, int64_t C,
                                 const uint8_t* __restrict__ held, int64_t r0, int64_t r1,
                                 int64_t* __restrict__ out) {
  GRID_STRIDE(p, n_padded)
    out[p] = p >= r0 && p < r1 && (!held || held[p / C]) ? int64_t(deg_perm[p]) : 0;
}

__global__ void arc_keys_kernel(const uint64_t* __restrict__ keys, int64_t m, int bits,
                                const int32_t* __restrict__ inv_perm, int pbits,
                                uint64_t* __restrict__ arcs) {
  const uint64_t mask = (uint64_t{1} << bits) - 1;
  GRID_STRIDE(i, m) {
    const uint64_t pu = uint64_t(inv_perm[keys[i] >> bits]);
    const uint64_t pv = uint64_t(inv_perm[keys[i] & mask]);
    arcs[2 * i] = (pu << pbits) | pv;
    arcs[2 * i + 1] = (pv << pbits) | pu;
  }
}

// Sorted arcs: arc a is the (a - rowptr[row])-th smallest neighbour of row.
// Arcs whose row (permuted) lies in [r0, r1) only, compacted through a
// warp-aggregated counter (their order does not matter: they are sorted).
__global__ void arc_keys_range_kernel(const uint64_t* __restrict__ keys, int64_t m, int bits,
                                      const int32_t* __restrict__ inv_perm, int pbits, int64_t C,
                                      const uint8_t* __restrict__ held, int64_t r0, int64_t r1,
                                      unsigned long long* __restrict__ count,
                                      uint64_t* __restrict__ arcs) {
  const uint64_t mask = (uint64_t{1} << bits) - 1;
  const int lane = threadIdx.x & 31;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < m; base += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    uint64_t k0 = 0, k1 = 0;
    bool a0 = false, a1 = false;
    if (i < m) {
      const int64_t pu = inv_perm[keys[i] >> bits];
      const int64_t pv = inv_perm[keys[i] & mask];
      a0 = pu >= r0 && pu < r1 && (!held || held[pu / C]);
      a1 = pv >= r0 && pv < r1 && (!held || held[pv / C]);
      k0 = (uint64_t(pu) << pbits) | uint64_t(pv);
      k1 = (uint64_t(pv) << pbits) | uint64_t(pu);
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
    if (a0) arcs[at++] = k0;
    if (a1) arcs[at] = k1;
  }
}

__global__ void scatter_kernel(const uint64_t* __restrict__ arcs, int64_t n_arcs, int pbits,
                               const int64_t* __restrict__ rowptr,
                               const int64_t* __restrict__ cs, int64_t C,
                               int32_t* __restrict__ col) {
  const uint64_t mask = (uint64_t{1} << pbits) - 1;
  GRID_STRIDE(a, n_arcs) {
    const uint64_t key = arcs[a];
    const int64_t row = int64_t(key >> pbits);
    const int64_t k = a - rowptr[row];
    col[cs[row / C] + k * C + row % C] = int32_t(key & mask);
  }
}

__global__ void narrow_col_kernel(const int64_t* __restrict__ in, int64_t count,
                                  int32_t* __restrict__ out) {
  GRID_STRIDE(i, count) out[i] = int32_t(in[i]);
}

__global__ void row_len_kernel(const int32_t* __restrict__ col, const int64_t* __restrict__ cs,
                               const int32_t* __restrict__ cl, int64_t n_padded, int64_t C,
                               int32_t* __restrict__ deg_perm) {
  GRID_STRIDE(p, n_padded) {
    const int64_t ch = p / C, lane = p % C;
    int32_t d = 0;
    for (int64_t j = 0; j < cl[ch]; ++j) d += col[cs[ch] + j * C + lane] >= 0;
    deg_perm[p] = d;
  }
}

template <typename T>
void exclusive_scan(const T* in, T* out, int64_t count, cudaStream_t s) {
  size_t tb = 0;
  SSB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, count, s));
  DevBuf<uint8_t> tmp(tb);
  SSB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, count, s));
}

struct I32ToI64 {
  __host__ __device__ int64_t operator()(int32_t v) const { return v; }
};

// Layout finishing shared by both builders: cl/cs/max from deg_perm.
void finish_chunks(ssb_graph& g, cudaStream_t s) {
  g.cl.alloc(std::max<int64_t>(g.n_chunks, 1));
  g.cs.alloc(g.n_chunks + 1);
  DevBuf<int64_t> cells(g.n_chunks + 1);
  SSB_CUDA(cudaMemsetAsync(cells.p, 0, 8 * (g.n_chunks + 1), s));
  if (g.n_chunks)
    chunk_len_kernel<<<grid_for(g.n_chunks), 256, 0, s>>>(g.deg.p, g.n_chunks, g.C,
                                                          g.partial() ? g.held.p : nullptr, g.cl.p,
                                                          cells.p);
  SSB_CUDA(cudaGetLastError());
  exclusive_scan(cells.p, g.cs.p, g.n_chunks + 1, s);
  SSB_CUDA(cudaMemcpyAsync(&g.n_cells, g.cs.p + g.n_chunks, 8, cudaMemcpyDeviceToHost, s));
  g.cl_host.resize(g.n_chunks);
  if (g.n_chunks)
    SSB_CUDA(cudaMemcpyAsync(g.cl_host.data(), g.cl.p, 4 * g.n_chunks, cudaMemcpyDeviceToHost, s));
  g.sc.sync();
  g.max_cl = 0;
  g.total_cells = 0;
  for (int32_t c : g.cl_host) {
    g.max_cl = std::max<int64_t>(g.max_cl, c);
    g.total_cells += int64_t(c) * g.C;
  }
}

}  // namespace

ssb_graph* build_from_edges(const ssb_edges& e, int64_t C, int64_t sigma) {
  return build_range_from_edges(e, C, sigma, {});
}

std::vector<int64_t> normalize_segments(const int64_t* bounds, int64_t nseg, int64_t n_chunks) {
  if (nseg < 0 || (nseg > 0 && !bounds)) fail(SSB_EINVAL, "bad segment list");
  std::vector<std::pair<int64_t, int64_t>> v;
  for (int64_t i = 0; i < nseg; ++i) {
    const int64_t b = bounds[2 * i], e = bounds[2 * i + 1];
    if (b < 0 || b > e || e > n_chunks) fail(SSB_EINVAL, "chunk range out of bounds");
    if (b < e) v.push_back({b, e});
  }
  std::sort(v.begin(), v.end());
  std::vector<int64_t> out;
  for (auto& x : v) {
    if (!out.empty() && x.first < out.back()) fail(SSB_EINVAL, "overlapping chunk segments");
    if (!out.empty() && x.first == out.back()) out.back() = x.second;  // merge adjacent
    else {
      out.push_back(x.first);
      out.push_back(x.second);
    }
  }
  return out;
}

// The layout's metadata (perm, inv_perm, row degrees, cl) for every chunk and
// the cells (cs, col) of the chunk segments `segs` only — one rank's share of
// a multi-GPU layout; empty segs = the whole layout.
ssb_graph* build_range_from_edges(const ssb_edges& e, int64_t C, int64_t sigma,
                                  const std::vector<int64_t>& segs_in) {
  // repr.cpp:63,85
  if (C <= 0) fail(SSB_EINVAL, "chunk height must be positive");
  if (sigma <= 0) fail(SSB_EINVAL, "sorting scope must be positive");
  auto g = std::make_unique<ssb_graph>();
  cudaStream_t s = g->sc.s;
  SSB_CUDA(cudaStreamSynchronize(e.sc.s));
  const int64_t n = e.n, m = e.m;
  g->C = C;
  g->n = n;
  g->sigma = std::min<int64_t>(sigma, std::max<int64_t>(n, 1));
  g->n_chunks = (n + C - 1) / C;
  g->n_padded = g->n_chunks * C;
  g->nonzeros = 2 * m;
  if (int64_t(g->n_padded) >= (int64_t{1} << 31)) fail(SSB_EINVAL, "n too large");
  {
    const std::vector<int64_t> sg =
        segs_in.empty() ? std::vector<int64_t>{}
                        : normalize_segments(segs_in.data(), int64_t(segs_in.size() / 2), g->n_chunks);
    const bool whole = segs_in.empty() || (sg.size() == 2 && sg[0] == 0 && sg[1] == g->n_chunks);
    if (!whole) {
      g->segs = sg.empty() ? std::vector<int64_t>{0, 0} : sg;  // {0, 0}: no cells (metadata only)
      std::vector<uint8_t> h(size_t(std::max<int64_t>(g->n_chunks, 1)), 0);
      for (size_t i = 0; i + 1 < sg.size(); i += 2)
        for (int64_t c = sg[i]; c < sg[i + 1]; ++c) h[size_t(c)] = 1;
      g->held.alloc(h.size());
      SSB_CUDA(cudaMemcpyAsync(g->held.p, h.data(), h.size(), cudaMemcpyHostToDevice, s));
    }
  }
  const bool partial = g->partial();
  const uint8_t* held = partial ? g->held.p : nullptr;
  const int64_t cb = 0, ce = g->n_chunks;  // passes walk every chunk; the mask keeps the held ones

  // 1. degrees
  DevBuf<int32_t> deg(std::max<int64_t>(n, 1));
  SSB_CUDA(cudaMemsetAsync(deg.p, 0, 4 * std::max<int64_t>(n, 1), s));
  if (m) degree_kernel<<<grid_for(m), 256, 0, s>>>(e.keys.p, m, e.bits, deg.p);
  SSB_CUDA(cudaGetLastError());
  DevBuf<int> dmax(1);
  SSB_CUDA(cudaMemsetAsync(dmax.p, 0, 4, s));
  if (n) max_reduce_kernel<<<grid_for(n), 256, 0, s>>>(deg.p, n, dmax.p);
  int maxdeg = 0;
  SSB_CUDA(cudaMemcpyAsync(&maxdeg, dmax.p, 4, cudaMemcpyDeviceToHost, s));
  g->sc.sync();

  // 2. sort plan (repr.cpp:62-82)
  g->perm.alloc(std::max<int64_t>(n, 1));
  g->inv_perm.alloc(std::max<int64_t>(n, 1));
  if (n > 0 && g->sigma > 1) {
    const int dbits = bits_for_value(uint64_t(maxdeg));
    const int64_t n_windows = (n + g->sigma - 1) / g->sigma;
    const int wbits = n_windows > 1 ? bits_for_value(uint64_t(n_windows - 1)) : 0;
    DevBuf<uint64_t> k0(n), k1(n);
    DevBuf<int32_t> v0(n);
    sort_keys_kernel<<<grid_for(n), 256, 0, s>>>(deg.p, n, g->sigma, dbits, maxdeg, k0.p, v0.p);
    SSB_CUDA(cudaGetLastError());
    cub::DoubleBuffer<uint64_t> dk(k0.p, k1.p);
    cub::DoubleBuffer<int32_t> dv(v0.p, g->perm.p);
    size_t tb = 0;
    SSB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, n, 0, dbits + wbits, s));
    DevBuf<uint8_t> tmp(tb);
    SSB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk, dv, n, 0, dbits + wbits, s));
    if (dv.Current() != g->perm.p)
      SSB_CUDA(cudaMemcpyAsync(g->perm.p, dv.Current(), 4 * n, cudaMemcpyDeviceToDevice, s));
    g->sc.sync();
  } else if (n > 0) {
    iota_kernel<<<grid_for(n), 256, 0, s>>>(g->perm.p, n);
  }
  g->deg.alloc(std::max<int64_t>(g->n_padded, 1));
  if (g->n_padded)
    perm_derive_kernel<<<grid_for(g->n_padded), 256, 0, s>>>(g->perm.p, n, g->n_padded, deg.p,
                                                             g->inv_perm.p, g->deg.p);
  SSB_CUDA(cudaGetLastError());
  deg.release();

  // 3. chunk lengths and offsets (repr.cpp:102-114)
  finish_chunks(*g, s);

  // 4. column-major scatter of the sorted, remapped neighbour lists
  //    (repr.cpp:116-128)
  g->col.alloc(std::max<int64_t>(g->n_cells, 1));
  SSB_CUDA(cudaMemsetAsync(g->col.p, 0xff, 4 * std::max<int64_t>(g->n_cells, 1), s));
  // Arcs (row, neighbour) of the built range, sorted and scattered in one or
  // more passes over row sub-ranges: a pass holds 2 x 8 B per arc (sort
  // double buffer), so a graph whose 2m arcs do not fit beside its col (S28:
  // 8.4e9 arcs, 135 GB) is built in several passes into the one col array.
  if (m > 0 && ce > cb) {
    const int pbits = bits_for_value(uint64_t(std::max<int64_t>(n - 1, 1)));
    // arcs per held chunk -> pass boundaries by cumulative arcs
    std::vector<int64_t> arcs_to(size_t(ce - cb) + 1, 0);
    {
      std::vector<int32_t> degp(size_t((ce - cb) * C));
      std::vector<uint8_t> h(partial ? size_t(g->n_chunks) : 0);
      SSB_CUDA(cudaMemcpyAsync(degp.data(), g->deg.p + cb * C, 4 * degp.size(), cudaMemcpyDeviceToHost, s));
      if (partial) SSB_CUDA(cudaMemcpyAsync(h.data(), g->held.p, h.size(), cudaMemcpyDeviceToHost, s));
      g->sc.sync();
      for (int64_t i = 0; i < ce - cb; ++i) {
        int64_t a = 0;
        if (!partial || h[size_t(i)])
          for (int64_t l = 0; l < C; ++l) a += degp[size_t(i * C + l)];
        arcs_to[size_t(i) + 1] = arcs_to[size_t(i)] + a;
      }
    }
    const int64_t total_arcs = arcs_to.back();
    size_t free_b = 0, tot_b = 0;
    SSB_CUDA(cudaMemGetInfo(&free_b, &tot_b));
    const int64_t cap_env = env_arcs_per_pass();
    // 16 B per arc for the sort's two buffers + ~25% for its temp storage
    const int64_t per_pass = cap_env > 0 ? cap_env : std::max<int64_t>(int64_t(double(free_b) * 0.6 / 20.0), 1 << 20);
    DevBuf<int64_t> rowptr(g->n_padded + 1);
    DevBuf<int64_t> rd(g->n_padded + 1);
    int64_t pc = cb;  // first chunk of the next pass
    while (pc < ce) {
      int64_t pe = pc + 1;
      while (pe < ce && arcs_to[size_t(pe + 1 - cb)] - arcs_to[size_t(pc - cb)] <= per_pass) ++pe;
      const int64_t r0 = pc * C, r1 = pe * C;
      // offsets over this pass's rows only; na = their arc count
      range_deg_kernel<<<grid_for(g->n_padded), 256, 0, s>>>(g->deg.p, g->n_padded, C, held, r0, r1,
                                                             rd.p);
      SSB_CUDA(cudaGetLastError());
      SSB_CUDA(cudaMemsetAsync(rd.p + g->n_padded, 0, 8, s));
      exclusive_scan(rd.p, rowptr.p, g->n_padded + 1, s);
      const int64_t na = arcs_to[size_t(pe - cb)] - arcs_to[size_t(pc - cb)];
      if (na > 0) {
        DevBuf<uint64_t> arcs(na), alt(na);
        if (!partial && pc == 0 && pe == g->n_chunks) {
          arc_keys_kernel<<<grid_for(m), 256, 0, s>>>(e.keys.p, m, e.bits, g->inv_perm.p, pbits, arcs.p);
        } else {
          DevBuf<unsigned long long> cnt(1);
          SSB_CUDA(cudaMemsetAsync(cnt.p, 0, 8, s));
          arc_keys_range_kernel<<<grid_for(m), 256, 0, s>>>(e.keys.p, m, e.bits, g->inv_perm.p, pbits,
                                                            C, held, r0, r1, cnt.p, arcs.p);
          g->sc.sync();
        }
        SSB_CUDA(cudaGetLastError());
        cub::DoubleBuffer<uint64_t> db(arcs.p, alt.p);
        size_t tb = 0;
        SSB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, na, 0, 2 * pbits, s));
        {
          DevBuf<uint8_t> tmp(tb);
          SSB_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, db, na, 0, 2 * pbits, s));
          g->sc.sync();
        }
        (db.Current() == arcs.p ? alt : arcs).release();
        scatter_kernel<<<grid_for(na), 256, 0, s>>>(db.Current(), na, pbits, rowptr.p, g->cs.p,
                                                    g->C, g->col.p);
        SSB_CUDA(cudaGetLastError());
        g->sc.sync();
      }
      g->build_passes += 1;
      pc = pe;
    }
    (void)total_arcs;
  }
  g->padding = g->total_cells - g->nonzeros;
  g->sc.sync();
  return g.release();
}

ssb_graph* graph_from_host_layout(int64_t n, int64_t C, int64_t sigma, int64_t nonzeros,
                                  const int64_t* col, int64_t n_cells, const int64_t* cs,
                                  const int64_t* cl, int64_t n_chunks, const int64_t* perm) {
  if (C <= 0) fail(SSB_EINVAL, "chunk height must be positive");
  if (n < 0 || n_chunks != (n + C - 1) / C) fail(SSB_EINVAL, "inconsistent layout sizes");
  if (n_chunks * C >= (int64_t{1} << 31)) fail(SSB_EINVAL, "n too large");
  auto g = std::make_unique<ssb_graph>();
  cudaStream_t s = g->sc.s;
  g->C = C;
  g->sigma = sigma;
  g->n = n;
  g->n_chunks = n_chunks;
  g->n_padded = n_chunks * C;
  g->nonzeros = nonzeros;
  // Validate the host layout (repr.hpp:33-55 invariants) before trusting it.
  int64_t total = 0;
  for (int64_t i = 0; i < n_chunks; ++i) {
    if (cl[i] < 0 || cs[i] != total) fail(SSB_EINVAL, "cs/cl inconsistent");
    total += C * cl[i];
  }
  if (total != n_cells) fail(SSB_EINVAL, "n_cells != sum of C*cl");
  std::vector<int32_t> p32(std::max<int64_t>(n, 1)), inv(std::max<int64_t>(n, 1), -1);
  for (int64_t p = 0; p < n; ++p) {
    if (perm[p] < 0 || perm[p] >= n || inv[perm[p]] != -1) fail(SSB_EINVAL, "perm is not a permutation");
    p32[p] = int32_t(perm[p]);
    inv[perm[p]] = int32_t(p);
  }
  g->perm.alloc(std::max<int64_t>(n, 1));
  g->inv_perm.alloc(std::max<int64_t>(n, 1));
  SSB_CUDA(cudaMemcpyAsync(g->perm.p, p32.data(), 4 * n, cudaMemcpyHostToDevice, s));
  SSB_CUDA(cudaMemcpyAsync(g->inv_perm.p, inv.data(), 4 * n, cudaMemcpyHostToDevice, s));
  {
    std::vector<int64_t> cs1(cs, cs + n_chunks);
    cs1.push_back(n_cells);
    std::vector<int32_t> cl32(cl, cl + n_chunks);
    g->cs.alloc(n_chunks + 1);
    g->cl.alloc(std::max<int64_t>(n_chunks, 1));
    SSB_CUDA(cudaMemcpyAsync(g->cs.p, cs1.data(), 8 * (n_chunks + 1), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(g->cl.p, cl32.data(), 4 * n_chunks, cudaMemcpyHostToDevice, s));
    g->sc.sync();
    g->cl_host = std::move(cl32);
  }
  g->n_cells = n_cells;
  g->col.alloc(std::max<int64_t>(n_cells, 1));
  {
    // bounded staging: convert int64 -> int32 on the device in slabs
    const int64_t slab = int64_t{1} << 26;
    DevBuf<int64_t> st(std::min<int64_t>(slab, std::max<int64_t>(n_cells, 1)));
    for (int64_t off = 0; off < n_cells; off += slab) {
      const int64_t cnt = std::min<int64_t>(slab, n_cells - off);
      SSB_CUDA(cudaMemcpyAsync(st.p, col + off, 8 * cnt, cudaMemcpyHostToDevice, s));
      narrow_col_kernel<<<grid_for(cnt), 256, 0, s>>>(st.p, cnt, g->col.p + off);
      SSB_CUDA(cudaGetLastError());
      g->sc.sync();
    }
  }
  g->deg.alloc(std::max<int64_t>(g->n_padded, 1));
  if (g->n_padded)
    row_len_kernel<<<grid_for(g->n_padded), 256, 0, s>>>(g->col.p, g->cs.p, g->cl.p, g->n_padded,
                                                         C, g->deg.p);
  SSB_CUDA(cudaGetLastError());
  g->max_cl = 0;
  for (int32_t c : g->cl_host) g->max_cl = std::max<int64_t>(g->max_cl, c);
  g->total_cells = n_cells;
  g->padding = n_cells - nonzeros;
  g->sc.sync();
  return g.release();
}

}  // namespace ssb
