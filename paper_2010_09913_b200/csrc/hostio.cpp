// Host side of the result fetch (ssb_bfs_spmv / ssb_bfs_fetch with host
// outputs): the device packs each BFS result in original-id order as a
// narrow wire format — uint8 levels (255 = unreached) and int32 parents —
// which crosses PCIe in chunks; a persistent pool of host threads widens
// every chunk into the caller's int64 dist / parent arrays (the reference's
// BfsResult layout, bfs.hpp:36-42) while the next chunk is in flight.
// 5 instead of 16 bytes per vertex over PCIe, the bound of the e2e path.
#include <immintrin.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "ssb_internal.cuh"

namespace ssb {
namespace {

class Pool {
 public:
  explicit Pool(int n) {
    for (int i = 1; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return int(th_.size()) + 1; }
  // f(w) on every worker w in [0, size()); the caller runs w = 0. One job at
  // a time: concurrent callers (e.g. one host thread per GPU, ctypes drops
  // the GIL) queue on run_mu_ instead of overwriting each other's job.
  void run(const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> serial(run_mu_);
    {
      std::lock_guard<std::mutex> l(mu_);
      job_ = &f;
      pending_ = int(th_.size());
      ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> l(mu_);
    done_.wait(l, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int w) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        f = job_;
      }
      (*f)(w);
      std::lock_guard<std::mutex> l(mu_);
      if (--pending_ == 0) done_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex run_mu_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

Pool& pool() {
  static Pool p([] {
    const int hw = int(std::thread::hardware_concurrency());
    const char* e = std::getenv("SSB_HOST_THREADS");
    const int want = e ? std::atoi(e) : 16;  // enough to outrun PCIe (scripts/widen_bw.c)
    return std::max(1, std::min(want, std::max(hw, 1)));
  }());
  return p;
}

bool has_avx2() {
  static const bool v = __builtin_cpu_supports("avx2");
  return v;
}

// dist[i] = lev[i] == 255 ? INT64_MAX : lev[i]
__attribute__((target("avx2"))) void widen_levels_avx2(const uint8_t* lev, int64_t* dist, int64_t b,
                                                      int64_t e) {
  int64_t i = b;
  for (; i < e && (reinterpret_cast<uintptr_t>(dist + i) & 31); ++i)
    dist[i] = lev[i] == 255 ? INT64_MAX : int64_t(lev[i]);
  const __m256i ff = _mm256_set1_epi64x(255), mx = _mm256_set1_epi64x(INT64_MAX);
  for (; i + 4 <= e; i += 4) {
    int32_t four;
    __builtin_memcpy(&four, lev + i, 4);
    __m256i l = _mm256_cvtepu8_epi64(_mm_cvtsi32_si128(four));
    l = _mm256_blendv_epi8(l, mx, _mm256_cmpeq_epi64(l, ff));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dist + i), l);
  }
  for (; i < e; ++i) dist[i] = lev[i] == 255 ? INT64_MAX : int64_t(lev[i]);
}

__attribute__((target("avx2"))) void widen_parents_avx2(const int32_t* par, int64_t* parent, int64_t b,
                                                       int64_t e) {
  int64_t i = b;
  for (; i < e && (reinterpret_cast<uintptr_t>(parent + i) & 31); ++i) parent[i] = par[i];
  for (; i + 4 <= e; i += 4) {
    const __m256i p = _mm256_cvtepi32_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i*>(par + i)));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(parent + i), p);
  }
  for (; i < e; ++i) parent[i] = par[i];
}

// Packed wire (sel-max results with dist and parents wanted, ids < 2^bits,
// levels < 2^(32-bits) - 1): one 32-bit word per vertex, level << bits | id,
// all ones where unreached — 4 instead of 5 bytes per vertex DMA-written and
// read back by the host, whose memory traffic bounds the e2e path.
__attribute__((target("avx2"))) void widen_packed_avx2(const uint32_t* w, int64_t* dist, int64_t* parent,
                                                      int64_t b, int64_t e, int bits) {
  const uint32_t lmax = 0xffffffffu >> bits;
  const uint32_t idmask = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
  auto one = [&](int64_t i) {
    const uint32_t x = w[i], l = x >> bits;
    dist[i] = l == lmax ? INT64_MAX : int64_t(l);
    parent[i] = l == lmax ? -1 : int64_t(x & idmask);
  };
  const __m128i sh = _mm_cvtsi32_si128(bits);
  const __m256i vl = _mm256_set1_epi64x(int64_t(lmax)), vm = _mm256_set1_epi64x(int64_t(idmask));
  const __m256i mx = _mm256_set1_epi64x(INT64_MAX), neg = _mm256_set1_epi64x(-1);
  // (a macro, not a lambda: lambdas do not inherit the avx2 target)
#define SSB_PACKED_FOUR(i, d, p)                                                                     \
  do {                                                                                               \
    const __m256i x_ = _mm256_cvtepu32_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i*>(w + (i)))); \
    const __m256i l_ = _mm256_srl_epi64(x_, sh);                                                     \
    const __m256i un_ = _mm256_cmpeq_epi64(l_, vl);                                                  \
    d = _mm256_blendv_epi8(l_, mx, un_);                                                             \
    p = _mm256_blendv_epi8(_mm256_and_si256(x_, vm), neg, un_);                                      \
  } while (0)
  int64_t i = b;
  __m256i d, p;
  if ((reinterpret_cast<uintptr_t>(dist) ^ reinterpret_cast<uintptr_t>(parent)) & 31) {
    // the two outputs never align together: plain unaligned stores
    for (; i + 4 <= e; i += 4) {
      SSB_PACKED_FOUR(i, d, p);
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(dist + i), d);
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(parent + i), p);
    }
  } else {
    for (; i < e && (reinterpret_cast<uintptr_t>(dist + i) & 31); ++i) one(i);
    for (; i + 4 <= e; i += 4) {
      SSB_PACKED_FOUR(i, d, p);
      _mm256_stream_si256(reinterpret_cast<__m256i*>(dist + i), d);
      _mm256_stream_si256(reinterpret_cast<__m256i*>(parent + i), p);
    }
  }
  for (; i < e; ++i) one(i);
#undef SSB_PACKED_FOUR
}

void widen(const uint8_t* lev, const int32_t* par, int64_t* dist, int64_t* parent, int64_t b, int64_t e,
           int packed_bits) {
  if (packed_bits > 0) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(par);
    if (has_avx2()) {
      widen_packed_avx2(w, dist, parent, b, e, packed_bits);
      _mm_sfence();
      return;
    }
    const uint32_t lmax = 0xffffffffu >> packed_bits, idmask = (1u << packed_bits) - 1u;
    for (int64_t i = b; i < e; ++i) {
      const uint32_t l = w[i] >> packed_bits;
      dist[i] = l == lmax ? INT64_MAX : int64_t(l);
      parent[i] = l == lmax ? -1 : int64_t(w[i] & idmask);
    }
    return;
  }
  if (has_avx2()) {
    if (dist) widen_levels_avx2(lev, dist, b, e);
    if (parent) widen_parents_avx2(par, parent, b, e);
    _mm_sfence();
    return;
  }
  for (int64_t i = b; i < e; ++i) {
    if (dist) dist[i] = lev[i] == 255 ? INT64_MAX : int64_t(lev[i]);
    if (parent) parent[i] = par[i];
  }
}

}  // namespace

// chunk c = entries [bounds[c], bounds[c+1]) of the host wire buffers, ready
// once ready[c] has completed; every worker widens its share of every chunk.
void widen_chunks(const std::vector<int64_t>& bounds, const std::vector<cudaEvent_t>& ready,
                  const uint8_t* lev, const int32_t* par, int64_t* dist, int64_t* parent,
                  int packed_bits) {
  Pool& p = pool();
  // Pieces of 64K entries (multiples of 64: the workers' stores stay in
  // separate cache lines) handed out in order through one counter, so a
  // worker slowed down by another thread on its core delays only its piece.
  constexpr int64_t kPiece = 1 << 16;
  std::vector<int64_t> first(bounds.size(), 0);  // first piece of chunk c
  for (size_t c = 0; c + 1 < bounds.size(); ++c)
    first[c + 1] = first[c] + (bounds[c + 1] - bounds[c] + kPiece - 1) / kPiece;
  std::atomic<int64_t> next{0};
  const int64_t total = first.back();
  p.run([&](int) {
    size_t c = 0;
    bool waited = false;
    for (int64_t q = next.fetch_add(1); q < total; q = next.fetch_add(1)) {
      while (q >= first[c + 1]) {
        ++c;
        waited = false;
      }
      if (!waited) {
        cudaEventSynchronize(ready[c]);
        waited = true;
      }
      const int64_t lo = bounds[c] + (q - first[c]) * kPiece;
      const int64_t hi = std::min(lo + kPiece, bounds[c + 1]);
      widen(lev, par, dist, parent, lo, hi, packed_bits);
    }
  });
}

int host_threads() { return pool().size(); }

}  // namespace ssb
