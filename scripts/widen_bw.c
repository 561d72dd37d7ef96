// Host widening bandwidth probe: uint8 levels -> int64 dist and int32 parents
// -> int64 parent, multi-threaded, regular vs non-temporal stores. Decides
// whether a narrow PCIe wire format + host widening beats int64 zero-copy.
// gcc -O3 -mavx2 -pthread widen_bw.c -o widen_bw
#include <immintrin.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
static int64_t N = 1 << 26;
static uint8_t* lev;
static int32_t* par;
static int64_t *dist, *parent;
static int nt_mode = 0, T = 1;
static double now(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + 1e-9 * t.tv_nsec; }
static void* work(void* arg) {
  int64_t id = (int64_t)arg, b = N * id / T, e = N * (id + 1) / T;
  b &= ~7LL; if (id == T - 1) e = N; else e &= ~7LL;
  if (!nt_mode) {
    for (int64_t i = b; i < e; ++i) { uint8_t l = lev[i]; dist[i] = l == 255 ? INT64_MAX : l; parent[i] = par[i]; }
  } else {
    const __m256i ff = _mm256_set1_epi64x(255), mx = _mm256_set1_epi64x(INT64_MAX);
    for (int64_t i = b; i < e; i += 4) {
      __m256i l = _mm256_cvtepu8_epi64(_mm_cvtsi32_si128(*(const int32_t*)(lev + i)));
      l = _mm256_blendv_epi8(l, mx, _mm256_cmpeq_epi64(l, ff));
      _mm256_stream_si256((__m256i*)(dist + i), l);
      __m256i p = _mm256_cvtepi32_epi64(_mm_loadu_si128((const __m128i*)(par + i)));
      _mm256_stream_si256((__m256i*)(parent + i), p);
    }
    _mm_sfence();
  }
  return 0;
}
int main(void) {
  lev = malloc(N); par = malloc(4 * N);
  dist = aligned_alloc(64, 8 * N); parent = aligned_alloc(64, 8 * N);
  for (int64_t i = 0; i < N; ++i) { lev[i] = i % 7 == 0 ? 255 : i % 9; par[i] = (int32_t)(i * 7); }
  memset(dist, 1, 8 * N); memset(parent, 1, 8 * N);
  int ts[] = {1, 4, 8, 16, 32};
  for (nt_mode = 0; nt_mode < 2; ++nt_mode)
    for (int k = 0; k < 5; ++k) {
      T = ts[k];
      double best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        pthread_t th[64];
        double t0 = now();
        for (int i = 0; i < T; ++i) pthread_create(&th[i], 0, work, (void*)(int64_t)i);
        for (int i = 0; i < T; ++i) pthread_join(th[i], 0);
        double dt = now() - t0; if (dt < best) best = dt;
      }
      printf("%s T=%2d: %.2f ms, %.1f GB/s written\n", nt_mode ? "stream" : "plain ", T, best * 1e3, 16.0 * N / best / 1e9);
    }
  return 0;
}
