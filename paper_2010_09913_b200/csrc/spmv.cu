// Generic int64 semiring product over the SlimSell layout — the kernel-level
// form of the reference's public spmv_step (repr.hpp:90-92, repr.cpp:193-217)
// with the reference's literal scalar algebra (semiring.hpp:56-87). The BFS
// engine (bfs.cu) does not use it: under BFS initial conditions the product
// reduces to 1-bit state, but the API must still multiply
// arbitrary int64 vectors, e.g. for kernel-level parity tests.
#include <climits>

#include "ssb_internal.cuh"

namespace ssb {
namespace {

constexpr int64_t kInf = INT64_MAX;

template <int V>
struct Ops;
template <>
struct Ops<SSB_TROPICAL> {
  static constexpr int64_t zero = kInf, edge = 1, pad = kInf;
  __device__ static int64_t plus(int64_t a, int64_t b) { return a < b ? a : b; }
  __device__ static int64_t times(int64_t a, int64_t b) {
    return (a == kInf || b == kInf) ? kInf : a + b;
  }
};
template <>
struct Ops<SSB_REAL> {
  static constexpr int64_t zero = 0, edge = 1, pad = 0;
  // two's-complement wrap, as the reference's int64 add/mul on x86-64
  __device__ static int64_t plus(int64_t a, int64_t b) {
    return int64_t(uint64_t(a) + uint64_t(b));
  }
  __device__ static int64_t times(int64_t a, int64_t b) {
    return int64_t(uint64_t(a) * uint64_t(b));
  }
};
template <>
struct Ops<SSB_BOOLEAN> {
  static constexpr int64_t zero = 0, edge = 1, pad = 0;
  __device__ static int64_t plus(int64_t a, int64_t b) { return a | b; }
  __device__ static int64_t times(int64_t a, int64_t b) { return a & b; }
};
template <>
struct Ops<SSB_SELMAX> {
  static constexpr int64_t zero = 0, edge = 1, pad = 0;
  __device__ static int64_t plus(int64_t a, int64_t b) { return a > b ? a : b; }
  __device__ static int64_t times(int64_t a, int64_t b) {
    return int64_t(uint64_t(a) * uint64_t(b));
  }
};

// One thread per row; the accumulator is seeded with x_prev[row]
// (repr.cpp:206) and padding cells gather x[0] with pad_value (repr.cpp:30-32).
template <int V>
__global__ void spmv_rows_kernel(const int32_t* __restrict__ col, const int64_t* __restrict__ cs,
                                 const int32_t* __restrict__ cl, int64_t C, int64_t row_begin,
                                 int64_t row_end, const int64_t* __restrict__ x,
                                 int64_t* __restrict__ out) {
  using O = Ops<V>;
  for (int64_t r = row_begin + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < row_end;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t ch = r / C, lane = r % C;
    const int32_t* cells = col + cs[ch] + lane;
    int64_t acc = x[r];
    const int32_t len = cl[ch];
    for (int32_t j = 0; j < len; ++j) {
      const int32_t c = cells[int64_t(j) * C];
      acc = O::plus(acc, O::times(x[c < 0 ? 0 : c], c < 0 ? O::pad : O::edge));
    }
    out[r] = acc;
  }
}

}  // namespace

void spmv_step(const ssb_graph& cg, int variant, const int64_t* x_prev, int64_t* out,
               int64_t chunk_begin, int64_t chunk_end) {
  ssb_graph& g = const_cast<ssb_graph&>(cg);
  if (variant < 0 || variant > 3) fail(SSB_EINVAL, "bad variant");
  if (chunk_begin < 0 || chunk_end > g.n_chunks || chunk_begin > chunk_end)
    fail(SSB_EINVAL, "chunk range out of bounds");
  if (!g.holds(chunk_begin, chunk_end))
    fail(SSB_EINVAL, "chunk range outside the segments this handle holds");
  const int64_t np = g.n_padded;
  if (np == 0) return;
  cudaStream_t s = g.sc.s;
  DevBuf<int64_t> dx(np), dout(np);
  SSB_CUDA(cudaMemcpyAsync(dx.p, x_prev, 8 * np, cudaMemcpyHostToDevice, s));
  SSB_CUDA(cudaMemcpyAsync(dout.p, out, 8 * np, cudaMemcpyHostToDevice, s));
  const int64_t r0 = chunk_begin * g.C, r1 = chunk_end * g.C;
  if (r1 > r0) {
    const int threads = 256;
    const int64_t want = (r1 - r0 + threads - 1) / threads;
    const int grid = int(want > int64_t(num_sms()) * 16 ? int64_t(num_sms()) * 16 : want);
    switch (variant) {
      case SSB_TROPICAL:
        spmv_rows_kernel<SSB_TROPICAL><<<grid, threads, 0, s>>>(g.col.p, g.cs.p, g.cl.p, g.C, r0, r1, dx.p, dout.p);
        break;
      case SSB_REAL:
        spmv_rows_kernel<SSB_REAL><<<grid, threads, 0, s>>>(g.col.p, g.cs.p, g.cl.p, g.C, r0, r1, dx.p, dout.p);
        break;
      case SSB_BOOLEAN:
        spmv_rows_kernel<SSB_BOOLEAN><<<grid, threads, 0, s>>>(g.col.p, g.cs.p, g.cl.p, g.C, r0, r1, dx.p, dout.p);
        break;
      default:
        spmv_rows_kernel<SSB_SELMAX><<<grid, threads, 0, s>>>(g.col.p, g.cs.p, g.cl.p, g.C, r0, r1, dx.p, dout.p);
        break;
    }
    SSB_CUDA(cudaGetLastError());
  }
  SSB_CUDA(cudaMemcpyAsync(out, dout.p, 8 * np, cudaMemcpyDeviceToHost, s));
  g.sc.sync();
}

}  // namespace ssb
