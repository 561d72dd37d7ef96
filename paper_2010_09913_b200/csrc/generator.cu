// Graph input stage on the device: Kronecker generation and Graph::from_pairs
// normalisation (orient, drop self-loops, sort, dedup), plus to_csr.
//
// Reference: generator.hpp:14-35 (SplitMix64), generator.cpp:60-89
// (gen_kronecker), graph.cpp:65-86 (Graph::from_pairs), graph.cpp:212-232
// (to_csr). The reference draws its Kronecker bits from ONE sequential
// SplitMix64 stream; the stream is counter-based (state += γ per draw), so draw
// i of edge e at level l is mix64(s0 + (e·scale + l + 1)·γ) and every edge is
// generated independently — bit-exact with the serial loop.
#include <cub/cub.cuh>

#include <cmath>
#include <thread>
#include <vector>

#include "ssb_internal.cuh"

namespace ssb {
namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

int bits_for(int64_t n) {  // bits to hold ids in [0, n)
  int b = 1;
  while ((int64_t{1} << b) < n) ++b;
  return b;
}

// r >= t  <=>  (draw >> 11) >= ceil(t · 2^53) for r = (draw >> 11) · 2^-53, so
// the double comparisons of generator.cpp:81-82 become exact integer ones.
uint64_t unit_threshold(double t) {
  if (!(t > 0.0)) return 0;
  const double s = std::ldexp(t, 53);
  if (s > 9007199254740992.0) return (uint64_t{1} << 53) + 1;  // never reached
  return static_cast<uint64_t>(std::ceil(s));
}

// One thread per candidate edge; emits the normalised key of the pair, or the
// self-loop sentinel (n-1, n-1), which sorts last and is dropped after dedup.
__global__ void kron_keys_kernel(uint64_t* __restrict__ keys, int64_t cand, int scale,
                                 uint64_t s0, uint64_t t_a, uint64_t t_ab, uint64_t t_abc,
                                 int bits, uint64_t sentinel) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < cand; e += stride) {
    uint64_t st = s0 + (uint64_t(e) * uint64_t(scale)) * kGamma;
    uint64_t u = 0, v = 0;
    for (int l = 0; l < scale; ++l) {
      st += kGamma;
      const uint64_t m = mix64(st) >> 11;
      const uint64_t ub = m >= t_ab;
      const uint64_t vb = ub ? (m >= t_abc) : (m >= t_a);
      u = (u << 1) | ub;
      v = (v << 1) | vb;
    }
    const uint64_t lo = u < v ? u : v, hi = u < v ? v : u;
    keys[e] = lo == hi ? sentinel : ((lo << bits) | hi);
  }
}

__global__ void pairs_minmax_kernel(const int64_t* __restrict__ uv, int64_t count,
                                    unsigned long long* __restrict__ max_id,
                                    int* __restrict__ negative) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  unsigned long long mx = 0;
  bool any = false, neg = false;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const int64_t a = uv[2 * i], b = uv[2 * i + 1];
    if (a < 0 || b < 0) neg = true;
    else {
      const unsigned long long h = static_cast<unsigned long long>(a > b ? a : b);
      mx = any ? (h > mx ? h : mx) : h;
      any = true;
    }
  }
  if (neg) atomicOr(negative, 1);
  if (any) atomicMax(max_id, mx + 1);  // stored +1 so that 0 means "no pair"
}

__global__ void pairs_keys_kernel(const int64_t* __restrict__ uv, int64_t count,
                                  uint64_t* __restrict__ keys, int bits, uint64_t sentinel) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint64_t a = uint64_t(uv[2 * i]), b = uint64_t(uv[2 * i + 1]);
    const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
    keys[i] = lo == hi ? sentinel : ((lo << bits) | hi);
  }
}

__global__ void keys_to_pairs_kernel(const uint64_t* __restrict__ keys, int64_t m, int bits,
                                     int64_t* __restrict__ uv) {
  const uint64_t mask = (uint64_t{1} << bits) - 1;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    uv[2 * i] = int64_t(keys[i] >> bits);
    uv[2 * i + 1] = int64_t(keys[i] & mask);
  }
}

// Both arcs of every edge, keyed (row, neighbour) for the CSR sort.
__global__ void arcs_kernel(const uint64_t* __restrict__ keys, int64_t m, int bits,
                            uint64_t* __restrict__ arcs) {
  const uint64_t mask = (uint64_t{1} << bits) - 1;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint64_t u = keys[i] >> bits, v = keys[i] & mask;
    arcs[2 * i] = (u << bits) | v;
    arcs[2 * i + 1] = (v << bits) | u;
  }
}

__global__ void arc_rows_kernel(const uint64_t* __restrict__ arcs, int64_t n_arcs, int bits,
                                int64_t* __restrict__ col, unsigned int* __restrict__ deg) {
  const uint64_t mask = (uint64_t{1} << bits) - 1;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_arcs; i += stride) {
    col[i] = int64_t(arcs[i] & mask);
    atomicAdd(&deg[arcs[i] >> bits], 1u);
  }
}

int grid_for(int64_t items, int threads = 256) {
  const int64_t want = (items + threads - 1) / threads;
  const int64_t cap = int64_t(num_sms()) * 32;
  return int(want < 1 ? 1 : (want > cap ? cap : want));
}

// Sort + unique + drop the self-loop sentinel. keys holds `count` keys and is
// replaced by the m normalised keys.
void normalise(ssb_edges& e, DevBuf<uint64_t>& keys, int64_t count, uint64_t sentinel) {
  cudaStream_t s = e.sc.s;
  if (count == 0) {
    e.m = 0;
    e.keys = DevBuf<uint64_t>();
    return;
  }
  DevBuf<uint64_t> alt(count);
  cub::DoubleBuffer<uint64_t> db(keys.p, alt.p);
  size_t tmp_bytes = 0;
  const int end_bit = 2 * e.bits;
  SSB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, db, count, 0, end_bit, s));
  DevBuf<uint8_t> tmp(tmp_bytes);
  SSB_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, db, count, 0, end_bit, s));
  uint64_t* sorted = db.Current();
  uint64_t* other = db.Alternate();
  DevBuf<int64_t> nsel(1);
  size_t tmp2 = 0;
  SSB_CUDA(cub::DeviceSelect::Unique(nullptr, tmp2, sorted, other, nsel.p, count, s));
  if (tmp2 > tmp.n) tmp.alloc(tmp2);
  SSB_CUDA(cub::DeviceSelect::Unique(tmp.p, tmp2, sorted, other, nsel.p, count, s));
  int64_t m = 0;
  SSB_CUDA(cudaMemcpyAsync(&m, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  e.sc.sync();
  uint64_t last = 0;
  if (m > 0) {
    SSB_CUDA(cudaMemcpyAsync(&last, other + (m - 1), 8, cudaMemcpyDeviceToHost, s));
    e.sc.sync();
    if (last == sentinel) --m;
  }
  DevBuf<uint64_t> out(m);
  if (m) SSB_CUDA(cudaMemcpyAsync(out.p, other, m * 8, cudaMemcpyDeviceToDevice, s));
  e.sc.sync();
  e.m = m;
  e.keys = std::move(out);
}

}  // namespace

ssb_edges* edges_from_pairs(const int64_t* uv, int64_t count, int64_t n) {
  if (count < 0) fail(SSB_EINVAL, "negative pair count");
  auto e = std::make_unique<ssb_edges>();
  cudaStream_t s = e->sc.s;
  DevBuf<int64_t> duv(2 * count);
  if (count) SSB_CUDA(cudaMemcpyAsync(duv.p, uv, 16 * count, cudaMemcpyHostToDevice, s));
  DevBuf<unsigned long long> mx(1);
  DevBuf<int> neg(1);
  SSB_CUDA(cudaMemsetAsync(mx.p, 0, 8, s));
  SSB_CUDA(cudaMemsetAsync(neg.p, 0, 4, s));
  if (count) pairs_minmax_kernel<<<grid_for(count), 256, 0, s>>>(duv.p, count, mx.p, neg.p);
  SSB_CUDA(cudaGetLastError());
  unsigned long long maxp1 = 0;
  int negative = 0;
  SSB_CUDA(cudaMemcpyAsync(&maxp1, mx.p, 8, cudaMemcpyDeviceToHost, s));
  SSB_CUDA(cudaMemcpyAsync(&negative, neg.p, 4, cudaMemcpyDeviceToHost, s));
  e->sc.sync();
  // graph.cpp:67-79
  if (negative) fail(SSB_ERANGE, "negative vertex id");
  const int64_t max_id = int64_t(maxp1) - 1;
  if (n < 0) n = max_id + 1;
  else if (max_id >= n)
    fail(SSB_ERANGE, "vertex id " + std::to_string(max_id) +
                         " exceeds declared vertex count " + std::to_string(n));
  if (n >= (int64_t{1} << 31)) fail(SSB_EINVAL, "device layout supports n < 2^31");
  e->n = n;
  e->bits = bits_for(n);
  const uint64_t sentinel = n > 0 ? ((uint64_t(n - 1) << e->bits) | uint64_t(n - 1)) : 0;
  DevBuf<uint64_t> keys(count);
  if (count)
    pairs_keys_kernel<<<grid_for(count), 256, 0, s>>>(duv.p, count, keys.p, e->bits, sentinel);
  SSB_CUDA(cudaGetLastError());
  duv.release();
  normalise(*e, keys, count, sentinel);
  return e.release();
}

ssb_edges* gen_kronecker(int64_t scale, int64_t ef, uint64_t seed, const double init[4]) {
  // generator.cpp:62-68
  if (scale < 1) fail(SSB_EINVAL, "scale must be >= 1");
  if (ef < 1) fail(SSB_EINVAL, "edgefactor must be >= 1");
  const double sum = init[0] + init[1] + init[2] + init[3];
  if (std::abs(sum - 1.0) > 1e-9) fail(SSB_EINVAL, "initiator probabilities must sum to 1");
  if (scale > 30) fail(SSB_EINVAL, "device layout supports scale <= 30");
  auto e = std::make_unique<ssb_edges>();
  const int64_t n = int64_t{1} << scale;
  const int64_t cand = ef * n;
  e->n = n;
  e->bits = int(scale);
  const double ab = init[0] + init[1];
  const double abc = ab + init[2];
  // SplitMix64(seed).split(0x4b) (generator.cpp:74, generator.hpp:29-31)
  const uint64_t s0 = mix64(seed ^ mix64(0x4bULL + 0x6a09e667f3bcc909ULL));
  const uint64_t sentinel = (uint64_t(n - 1) << e->bits) | uint64_t(n - 1);
  DevBuf<uint64_t> keys(cand);
  kron_keys_kernel<<<grid_for(cand), 256, 0, e->sc.s>>>(
      keys.p, cand, int(scale), s0, unit_threshold(init[0]), unit_threshold(ab),
      unit_threshold(abc), e->bits, sentinel);
  SSB_CUDA(cudaGetLastError());
  normalise(*e, keys, cand, sentinel);
  return e.release();
}

namespace {
// Pair index t of the upper triangle (row-major, pairs (u, u+1+v)) -> key.
// Row u starts at S(u) = u(n-1) - u(u-1)/2; exact integer binary search.
__global__ void er_decode_kernel(const int64_t* __restrict__ t, int64_t count, int64_t n,
                                 int bits, uint64_t* __restrict__ keys) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const int64_t x = t[i];
    int64_t lo = 0, hi = n - 2;  // largest u with S(u) <= x
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      const int64_t s = mid * (n - 1) - mid * (mid - 1) / 2;
      if (s <= x) lo = mid;
      else hi = mid - 1;
    }
    const int64_t u = lo;
    const int64_t v = u + 1 + (x - (u * (n - 1) - u * (u - 1) / 2));
    keys[i] = (uint64_t(u) << bits) | uint64_t(v);
  }
}
}  // namespace

// gen_erdos_renyi (generator.cpp:15-58). The reference walks the pair index
// space [0, n(n-1)/2) with geometric skips drawn from ONE SplitMix64 stream
// (split(0xe5)); the stream is counter-based, so the skips are computed by all
// host threads at once with the same libm log/log1p as the reference
// (bit-exact — a device log could differ in the last ulp and move a floor),
// their prefix sums give the pair indices, and the device decodes them to
// (u, v). The pairs come out sorted and unique, i.e. already normalised.
ssb_edges* gen_erdos_renyi(int64_t n, double p, uint64_t seed) {
  if (n < 0) fail(SSB_EINVAL, "vertex count must be >= 0");
  if (!(p >= 0.0 && p <= 1.0)) fail(SSB_EINVAL, "edge probability must be in [0, 1]");
  if (n >= (int64_t{1} << 31)) fail(SSB_EINVAL, "device layout supports n < 2^31");
  std::vector<int64_t> pos;  // pair indices, ascending
  const int64_t total = n > 1 ? n * (n - 1) / 2 : 0;
  if (p > 0.0 && n > 1) {
    if (p == 1.0) {
      pos.resize(size_t(total));
      for (int64_t i = 0; i < total; ++i) pos[size_t(i)] = i;
    } else {
      const uint64_t s0 = mix64(seed ^ mix64(0xe5ULL + 0x6a09e667f3bcc909ULL));
      const double denom = std::log1p(-p);
      const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
      // draw i (0-based) -> geometric skip, generator.cpp:48-53
      auto skip_of = [&](int64_t i) -> int64_t {
        const uint64_t x = mix64(s0 + uint64_t(i + 1) * kGamma);
        const double unit = 1.0 - double(x >> 11) * 0x1.0p-53;
        return int64_t(std::floor(std::log(unit) / denom));
      };
      const double mean = double(total) * p;
      int64_t drawn = 0, cursor = -1;  // cursor: last pair index (t_{-1} = -1)
      bool first = true;
      std::vector<int64_t> sk;
      pos.reserve(size_t(std::min<double>(mean + 10.0 * std::sqrt(mean + 1.0) + 1024.0, double(total))));
      while (true) {
        // first batch: the expected pair count + 10 sigma; then 1M draws at a time
        const int64_t batch = drawn == 0 ? int64_t(mean + 10.0 * std::sqrt(mean + 1.0)) + 1024
                                         : int64_t{1} << 20;
        sk.resize(size_t(std::max<int64_t>(batch, 1 << 16)));
        const int64_t b = int64_t(sk.size());
        std::vector<std::thread> th;
        for (unsigned w = 0; w < nt; ++w)
          th.emplace_back([&, w] {
            for (int64_t i = b * w / nt; i < b * (w + 1) / nt; ++i) sk[size_t(i)] = skip_of(drawn + i);
          });
        for (auto& x : th) x.join();
        bool done = false;
        for (int64_t i = 0; i < b; ++i) {
          // advance(first ? skip : 1 + skip) from the cursor (generator.cpp:35-53)
          cursor += (first ? sk[size_t(i)] + 1 : 1 + sk[size_t(i)]);
          first = false;
          if (cursor >= total || cursor < 0) {
            done = true;
            break;
          }
          pos.push_back(cursor);
        }
        drawn += b;
        if (done) break;
      }
    }
  }
  auto e = std::make_unique<ssb_edges>();
  e->n = n;
  e->bits = bits_for(std::max<int64_t>(n, 1));
  const int64_t m = int64_t(pos.size());
  e->m = m;
  e->keys.alloc(size_t(std::max<int64_t>(m, 1)));
  if (m) {
    DevBuf<int64_t> dt{static_cast<size_t>(m)};
    SSB_CUDA(cudaMemcpyAsync(dt.p, pos.data(), 8 * m, cudaMemcpyHostToDevice, e->sc.s));
    er_decode_kernel<<<grid_for(m), 256, 0, e->sc.s>>>(dt.p, m, n, e->bits, e->keys.p);
    SSB_CUDA(cudaGetLastError());
    e->sc.sync();
  }
  return e.release();
}

void edges_to_csr(const ssb_edges& ce, int64_t* row, int64_t* col) {
  ssb_edges& e = const_cast<ssb_edges&>(ce);
  cudaStream_t s = e.sc.s;
  const int64_t n = e.n, m = e.m, na = 2 * m;
  std::vector<unsigned int> deg(n > 0 ? n : 1, 0);
  if (na > 0) {
    DevBuf<uint64_t> arcs(na), alt(na);
    arcs_kernel<<<grid_for(m), 256, 0, s>>>(e.keys.p, m, e.bits, arcs.p);
    SSB_CUDA(cudaGetLastError());
    cub::DoubleBuffer<uint64_t> db(arcs.p, alt.p);
    size_t tb = 0;
    SSB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, na, 0, 2 * e.bits, s));
    DevBuf<uint8_t> tmp(tb);
    SSB_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, db, na, 0, 2 * e.bits, s));
    DevBuf<int64_t> dcol(na);
    DevBuf<unsigned int> ddeg(n);
    SSB_CUDA(cudaMemsetAsync(ddeg.p, 0, 4 * n, s));
    arc_rows_kernel<<<grid_for(na), 256, 0, s>>>(db.Current(), na, e.bits, dcol.p, ddeg.p);
    SSB_CUDA(cudaGetLastError());
    SSB_CUDA(cudaMemcpyAsync(col, dcol.p, 8 * na, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaMemcpyAsync(deg.data(), ddeg.p, 4 * n, cudaMemcpyDeviceToHost, s));
    e.sc.sync();
  }
  row[0] = 0;
  for (int64_t v = 0; v < n; ++v) row[v + 1] = row[v] + (na > 0 ? deg[v] : 0);
}

}  // namespace ssb
