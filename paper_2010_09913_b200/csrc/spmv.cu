// Generic int64 semiring product over the SlimSell layout — the kernel-level
// form of the reference's public spmv_step / spmv_segment (repr.hpp:79-98,
// repr.cpp:20-35, 153-217) with the reference's literal scalar algebra
// (semiring.hpp:56-87). The BFS engine (bfs.cu) does not use it: under BFS
// initial conditions the product reduces to 1-bit state,
// but the API multiplies arbitrary int64 vectors.
//
// Schedule: one warp per WORK UNIT — a chunk's column range of at most
// kUnitCols columns (the hub chunks of a power-law layout, up to 1M columns at
// S26, split into many units, SlimChunk-style). Lane l holds row l of the
// chunk (rows in groups of 32 for C > 32); each column is one coalesced
// C·4-byte load of col plus one 8-byte gather of x per lane. A unit that
// covers its whole chunk writes plus(x_prev[row], acc) directly; the units of
// a split chunk fold into rows seeded with x_prev by 64-bit atomics (min /
// add / or / max — every semiring plus is associative and commutative on
// int64, so the order of the folds cannot change the result).
#include <algorithm>
#include <climits>
#include <memory>
#include <vector>

#include "ssb_internal.cuh"

namespace ssb {
namespace {

constexpr int64_t kInf = INT64_MAX;
constexpr int32_t kUnitCols = 1024;

template <int V>
struct Ops;
template <>
struct Ops<SSB_TROPICAL> {
  static constexpr int64_t zero = kInf, edge = 1, pad = kInf, ident = kInf;
  __device__ static int64_t plus(int64_t a, int64_t b) { return a < b ? a : b; }
  __device__ static int64_t times(int64_t a, int64_t b) {
    return (a == kInf || b == kInf) ? kInf : a + b;
  }
  __device__ static void fold(int64_t* p, int64_t v) {
    atomicMin(reinterpret_cast<long long*>(p), static_cast<long long>(v));
  }
};
template <>
struct Ops<SSB_REAL> {
  static constexpr int64_t zero = 0, edge = 1, pad = 0, ident = 0;
  // two's-complement wrap, as the reference's int64 add/mul on x86-64
  __device__ static int64_t plus(int64_t a, int64_t b) {
    return int64_t(uint64_t(a) + uint64_t(b));
  }
  __device__ static int64_t times(int64_t a, int64_t b) {
    return int64_t(uint64_t(a) * uint64_t(b));
  }
  __device__ static void fold(int64_t* p, int64_t v) {
    atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
  }
};
template <>
struct Ops<SSB_BOOLEAN> {
  static constexpr int64_t zero = 0, edge = 1, pad = 0, ident = 0;
  __device__ static int64_t plus(int64_t a, int64_t b) { return a | b; }
  __device__ static int64_t times(int64_t a, int64_t b) { return a & b; }
  __device__ static void fold(int64_t* p, int64_t v) {
    atomicOr(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
  }
};
template <>
struct Ops<SSB_SELMAX> {
  // zero = 0 is the semiring's (non-negative) zero; a unit's partial starts
  // at the true identity of max so arbitrary int64 inputs fold exactly
  static constexpr int64_t zero = 0, edge = 1, pad = 0, ident = INT64_MIN;
  __device__ static int64_t plus(int64_t a, int64_t b) { return a > b ? a : b; }
  __device__ static int64_t times(int64_t a, int64_t b) {
    return int64_t(uint64_t(a) * uint64_t(b));
  }
  __device__ static void fold(int64_t* p, int64_t v) {
    atomicMax(reinterpret_cast<long long*>(p), static_cast<long long>(v));
  }
};

enum : int32_t { kSplit = 0, kWhole = 1, kSegment = 2 };
struct Unit {
  int32_t chunk, col_begin, col_len, mode;
};

// rows of the chunks the units do not write in full (split or cell-less):
// out = x_prev (repr.cpp:206's seed)
__global__ void seed_rows_kernel(const int32_t* __restrict__ chunks, int64_t nchunks, int64_t C,
                                 const int64_t* __restrict__ x, int64_t* __restrict__ out) {
  const int64_t total = nchunks * C;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = int64_t(chunks[i / C]) * C + i % C;
    out[r] = x[r];
  }
}

// One warp per unit. Padding cells gather x[0] with pad_value (repr.cpp:30-32).
template <int V>
__global__ void __launch_bounds__(256) spmv_units_kernel(const int32_t* __restrict__ col,
                                                         const int64_t* __restrict__ cs, int64_t C,
                                                         const Unit* __restrict__ units, int64_t n_units,
                                                         const int64_t* __restrict__ x,
                                                         int64_t* __restrict__ out,
                                                         int64_t* __restrict__ seg_acc) {
  using O = Ops<V>;
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_units; w += warps) {
    const Unit u = units[w];
    const int32_t* base = col + cs[u.chunk] + int64_t(u.col_begin) * C;
    for (int64_t l0 = 0; l0 < C; l0 += 32) {
      const int64_t l = l0 + lane;
      if (l >= C) break;
      const int32_t* cells = base + l;
      int64_t acc = O::ident;
      int32_t j = 0;
      for (; j + 4 <= u.col_len; j += 4) {  // four columns' loads in flight
        int32_t c[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = __ldg(cells + int64_t(j + q) * C);
        int64_t xv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) xv[q] = __ldg(x + (c[q] < 0 ? 0 : c[q]));
#pragma unroll
        for (int q = 0; q < 4; ++q) acc = O::plus(acc, O::times(xv[q], c[q] < 0 ? O::pad : O::edge));
      }
      for (; j < u.col_len; ++j) {
        const int32_t c = __ldg(cells + int64_t(j) * C);
        acc = O::plus(acc, O::times(__ldg(x + (c < 0 ? 0 : c)), c < 0 ? O::pad : O::edge));
      }
      const int64_t r = int64_t(u.chunk) * C + l;
      if (u.mode == kWhole) out[r] = O::plus(x[r], acc);
      else if (u.mode == kSplit) O::fold(out + r, acc);
      else O::fold(seg_acc + l, acc);  // a segment's units fold into acc
    }
  }
}

// The unit plan of a chunk range, cached on the handle (host-built from cl).
struct SpmvPlan {
  int64_t cb = -1, ce = -1;
  DevBuf<Unit> units;
  DevBuf<int32_t> seed_chunks;
  int64_t n_units = 0, n_seed = 0, cells = 0;
};

SpmvPlan& plan_for(ssb_graph& g, int64_t cb, int64_t ce) {
  auto* p = static_cast<SpmvPlan*>(g.spmv_plan.get());
  if (p && p->cb == cb && p->ce == ce) return *p;
  auto np = std::make_shared<SpmvPlan>();
  std::vector<Unit> units;
  std::vector<int32_t> seed;
  for (int64_t i = cb; i < ce; ++i) {
    const int32_t len = g.cl_host[size_t(i)];
    if (len == 0) {
      seed.push_back(int32_t(i));
      continue;
    }
    if (len <= kUnitCols) {
      units.push_back({int32_t(i), 0, len, kWhole});
    } else {
      seed.push_back(int32_t(i));
      for (int32_t c = 0; c < len; c += kUnitCols) units.push_back({int32_t(i), c, std::min(kUnitCols, len - c), kSplit});
    }
    np->cells += int64_t(len) * g.C;
  }
  // longest units first: the hub chunks' pieces do not trail the launch
  std::stable_sort(units.begin(), units.end(), [](const Unit& a, const Unit& b) { return a.col_len > b.col_len; });
  np->cb = cb;
  np->ce = ce;
  np->n_units = int64_t(units.size());
  np->n_seed = int64_t(seed.size());
  np->units.alloc(std::max<size_t>(units.size(), 1));
  np->seed_chunks.alloc(std::max<size_t>(seed.size(), 1));
  if (!units.empty())
    SSB_CUDA(cudaMemcpy(np->units.p, units.data(), units.size() * sizeof(Unit), cudaMemcpyHostToDevice));
  if (!seed.empty())
    SSB_CUDA(cudaMemcpy(np->seed_chunks.p, seed.data(), seed.size() * 4, cudaMemcpyHostToDevice));
  g.spmv_plan = np;
  return *np;
}

template <int V>
void launch_units(ssb_graph& g, const Unit* units, int64_t n_units, const int64_t* x, int64_t* out,
                  int64_t* seg_acc, cudaStream_t s) {
  if (n_units == 0) return;
  const int64_t want = (n_units * 32 + 255) / 256;
  const int grid = int(std::min<int64_t>(want, int64_t(num_sms()) * 8));
  spmv_units_kernel<V><<<grid, 256, 0, s>>>(g.col.p, g.cs.p, g.C, units, n_units, x, out, seg_acc);
  SSB_CUDA(cudaGetLastError());
}

void dispatch(int variant, ssb_graph& g, const Unit* units, int64_t n_units, const int64_t* x,
              int64_t* out, int64_t* seg_acc, cudaStream_t s) {
  switch (variant) {
    case SSB_TROPICAL: launch_units<SSB_TROPICAL>(g, units, n_units, x, out, seg_acc, s); break;
    case SSB_REAL: launch_units<SSB_REAL>(g, units, n_units, x, out, seg_acc, s); break;
    case SSB_BOOLEAN: launch_units<SSB_BOOLEAN>(g, units, n_units, x, out, seg_acc, s); break;
    default: launch_units<SSB_SELMAX>(g, units, n_units, x, out, seg_acc, s); break;
  }
}

void check_range(const ssb_graph& g, int variant, int64_t chunk_begin, int64_t chunk_end) {
  if (variant < 0 || variant > 3) fail(SSB_EINVAL, "bad variant");
  if (chunk_begin < 0 || chunk_end > g.n_chunks || chunk_begin > chunk_end)
    fail(SSB_EINVAL, "chunk range out of bounds");
  if (!g.holds(chunk_begin, chunk_end))
    fail(SSB_EINVAL, "chunk range outside the segments this handle holds");
}

}  // namespace

// Device-resident operands: x_prev / out are n_padded int64 in device memory.
void spmv_step_device(const ssb_graph& cg, int variant, const int64_t* x_prev, int64_t* out,
                      int64_t chunk_begin, int64_t chunk_end, double* device_ms) {
  ssb_graph& g = const_cast<ssb_graph&>(cg);
  check_range(g, variant, chunk_begin, chunk_end);
  if (g.n_padded == 0 || chunk_end == chunk_begin) {
    if (device_ms) *device_ms = 0;
    return;
  }
  SpmvPlan& P = plan_for(g, chunk_begin, chunk_end);
  cudaStream_t s = g.sc.s;
  SSB_CUDA(cudaEventRecord(g.sc.e0, s));
  if (P.n_seed) {
    const int64_t total = P.n_seed * g.C;
    const int grid = int(std::min<int64_t>((total + 255) / 256, int64_t(num_sms()) * 16));
    seed_rows_kernel<<<grid, 256, 0, s>>>(P.seed_chunks.p, P.n_seed, g.C, x_prev, out);
    SSB_CUDA(cudaGetLastError());
  }
  dispatch(variant, g, P.units.p, P.n_units, x_prev, out, nullptr, s);
  SSB_CUDA(cudaEventRecord(g.sc.e1, s));
  g.sc.sync();
  if (device_ms) {
    float ms = 0;
    SSB_CUDA(cudaEventElapsedTime(&ms, g.sc.e0, g.sc.e1));
    *device_ms = ms;
  }
}

void spmv_step(const ssb_graph& cg, int variant, const int64_t* x_prev, int64_t* out,
               int64_t chunk_begin, int64_t chunk_end) {
  ssb_graph& g = const_cast<ssb_graph&>(cg);
  check_range(g, variant, chunk_begin, chunk_end);
  const int64_t np = g.n_padded;
  if (np == 0) return;
  cudaStream_t s = g.sc.s;
  DevBuf<int64_t> dx(np), dout(np);
  SSB_CUDA(cudaMemcpyAsync(dx.p, x_prev, 8 * np, cudaMemcpyHostToDevice, s));
  SSB_CUDA(cudaMemcpyAsync(dout.p, out, 8 * np, cudaMemcpyHostToDevice, s));  // rows outside: untouched
  spmv_step_device(g, variant, dx.p, dout.p, chunk_begin, chunk_end, nullptr);
  SSB_CUDA(cudaMemcpyAsync(out, dout.p, 8 * np, cudaMemcpyDeviceToHost, s));
  g.sc.sync();
}

// spmv_segment (repr.hpp:79-81, repr.cpp:153-170): acc[lane] = plus(acc[lane],
// times(x[c], edge/pad)) over columns [col_begin, col_begin + col_len) of one
// chunk; acc holds C values.
void spmv_segment(const ssb_graph& cg, int variant, const int64_t* x_prev, int64_t* acc, int64_t chunk,
                  int64_t col_begin, int64_t col_len) {
  ssb_graph& g = const_cast<ssb_graph&>(cg);
  if (variant < 0 || variant > 3) fail(SSB_EINVAL, "bad variant");
  if (chunk < 0 || chunk >= g.n_chunks) fail(SSB_EINVAL, "chunk out of bounds");
  if (!g.holds(chunk, chunk + 1)) fail(SSB_EINVAL, "chunk outside the segments this handle holds");
  const int64_t cl = g.cl_host[size_t(chunk)];
  if (col_begin < 0 || col_len < 0 || col_begin + col_len > cl)
    fail(SSB_EINVAL, "column range [" + std::to_string(col_begin) + ", " + std::to_string(col_begin + col_len) +
                         ") outside chunk " + std::to_string(chunk) + " of length " + std::to_string(cl));
  if (col_len == 0) return;
  cudaStream_t s = g.sc.s;
  const int64_t np = g.n_padded;
  DevBuf<int64_t> dx(np), dacc(g.C);
  SSB_CUDA(cudaMemcpyAsync(dx.p, x_prev, 8 * np, cudaMemcpyHostToDevice, s));
  SSB_CUDA(cudaMemcpyAsync(dacc.p, acc, 8 * g.C, cudaMemcpyHostToDevice, s));
  // one unit per kUnitCols columns, all folding into acc (atomics, any order)
  std::vector<Unit> units;
  for (int64_t c = col_begin; c < col_begin + col_len; c += kUnitCols)
    units.push_back({int32_t(chunk), int32_t(c), int32_t(std::min<int64_t>(kUnitCols, col_begin + col_len - c)),
                     kSegment});
  DevBuf<Unit> du(units.size());
  SSB_CUDA(cudaMemcpyAsync(du.p, units.data(), units.size() * sizeof(Unit), cudaMemcpyHostToDevice, s));
  dispatch(variant, g, du.p, int64_t(units.size()), dx.p, nullptr, dacc.p, s);
  SSB_CUDA(cudaMemcpyAsync(acc, dacc.p, 8 * g.C, cudaMemcpyDeviceToHost, s));
  g.sc.sync();
}

}  // namespace ssb
