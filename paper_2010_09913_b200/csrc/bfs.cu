// The BFS-SpMV engine on the device (north_star subsystems 2-4).
//
// Reference: bfs_spmv / BfsEngine (bfs.cpp:53-155, 222-246), the kernel
// slim_segment_impl (repr.cpp:20-35), post_process_rows (semiring.cpp:90-124),
// should_skip_chunk (semiring.cpp:130-150), is_converged (semiring.cpp:152-157),
// plan_subchunks / combine_chunks (bfs.cpp:10-22, 205-220), selmax_parents
// (bfs.cpp:94-101), dp_transform (semiring.cpp:159-187).
//
// State encoding: under BFS initial conditions every value
// that reaches an output is a function of 1-bit state, so the engine keeps
//   visited  — 1 bit per padded row (chunk i <-> word i when C = 32),
//   F[2]     — the frontier of the previous / current iteration,
//   S[3]     — a coarse summary of F (1 bit per 2^gshift words) for the part
//              of F that does not fit in shared memory,
//   level / parent — int32 per row, written once when the row is reached.
// The per-semiring product for an unvisited row becomes
//   tropical  min_u (d_u + 1)  -> "some frontier neighbour" -> d = k
//   real      Σ f_u ≠ 0        -> "some frontier neighbour"
//   boolean   ∨ f_u            -> "some frontier neighbour"
//   sel-max   max_u (pos_u+1)  -> the largest frontier-neighbour position,
//             i.e. the LAST hit of the row's ascending column list.
// Visited rows never change any output, SlimWork skips chunks whose real rows
// are all visited, and convergence is "no row newly reached" for every variant.
//
// Two engines:
//  * C = 32 (warp width): one persistent cooperative kernel runs all
//    iterations. Each CTA stages the frontier prefix + summary in shared
//    memory, warps pull SlimChunk tasks (≤ 32 work units) from a per-iteration
//    atomic counter, and each 8-lane group streams one unit column-major with
//    128-bit loads (lane = 4 rows of one column), gathering frontier bits from
//    shared memory. Split chunks combine through global atomics; the last unit
//    finalises. Iterations are separated by grid.sync().
//  * any other C: a straightforward row-per-thread engine driven from the
//    host (the reference's small-C parity configurations).
#include <cooperative_groups.h>

#include <algorithm>
#include <future>
#include <chrono>
#include <mutex>
#include <climits>
#include <cstdlib>
#include <memory>
#include <cstdio>
#include <cstring>
#include <thread>
#include <type_traits>
#include <unistd.h>

#include "ssb_internal.cuh"

namespace cg = cooperative_groups;

namespace ssb {
namespace {

#ifndef SSB_BFS_THREADS
#define SSB_BFS_THREADS 1024
#endif
constexpr int kThreads = SSB_BFS_THREADS;  // 32 warps, 64 registers (spills: a few words of per-task bookkeeping, none in the column loops)
constexpr int kUnitsPerTask = 32;
constexpr int kStatW = 8;  // int64 per iteration record
// record: 0 frontier_size, 1 chunks_processed, 2 chunks_skipped,
//         3 subchunks_processed, 4 columns_processed, 5 elapsed_ns
#ifndef SSB_ITERS_PER_LAUNCH
#define SSB_ITERS_PER_LAUNCH 1024  // (1: one launch per iteration, for per-iteration profiles)
#endif
constexpr int kItersPerLaunch = SSB_ITERS_PER_LAUNCH;
constexpr int64_t kRecFirst = 64;  // records returned with every launch (a BFS rarely needs more)

int env_int(const char* name, int def) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : def;
}

int grid_for(int64_t items, int threads = 256) {
  const int64_t want = (items + threads - 1) / threads;
  const int64_t cap = int64_t(num_sms()) * 32;
  return int(want < 1 ? 1 : (want > cap ? cap : want));
}

#define GRID_STRIDE(i, count)                                                       \
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < (count); \
       i += int64_t(gridDim.x) * blockDim.x)

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0;" : "=l"(p));
  return p;
}

// Streaming 128-bit load of col: read-only for the kernel, not kept in L1,
// marked evict-first in L2 so the 8.5 GB stream does not push the frontier
// bitmap out of the 126 MB L2.
__device__ __forceinline__ int4 ld_stream(const int4* p, uint64_t pol) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// Bulk L2 prefetch (no registers, no completion tracking): keeps more of the
// col stream in flight than the four-step register ring alone can. bytes is a
// multiple of 16, p 16-byte aligned.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
#ifndef SSB_LAST_GRAB_SKIP
#define SSB_LAST_GRAB_SKIP 1  // no counter round trip after the first task when n_tasks <= warps
#endif
#ifndef SSB_BCAST
#define SSB_BCAST 1  // per-iteration totals read by one thread per CTA and broadcast in shared memory
#endif
#ifndef SSB_LAZY_STAGE
#define SSB_LAZY_STAGE 1  // warps wait for the staged image at their first probe, not before their first task
#endif
// The wait for an iteration's staged frontier image, taken once per warp
// (warp-uniform: every lane of the warp calls it together).
struct ImgWait {
  unsigned long long* bar;
  uint32_t phase;
  bool ok;
  __device__ __forceinline__ void operator()() {
    if (!ok) {
      mbar_wait(bar, phase);
      ok = true;
    }
  }
};
// TMA bulk copy global -> this CTA's shared memory in <= 32 KB pieces
// (bytes and both addresses 16-byte aligned), completing on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  for (uint32_t off = 0; off < bytes; off += 32768u) {
    const uint32_t sz = min(32768u, bytes - off);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(static_cast<char*>(dst) + off)),
        "l"(static_cast<const char*>(src) + off), "r"(sz), "r"(smem_u32(bar))
        : "memory");
  }
}

#ifndef SSB_PF_AHEAD
#define SSB_PF_AHEAD 1  // in-loop prefetch distance, in 2 KB loop iterations (A/B: 1 best)
#endif
constexpr int32_t kPfAhead = SSB_PF_AHEAD;
#ifndef SSB_TLIST64
#define SSB_TLIST64 1
#endif
// SSB_TLIST64: a list entry carries its task's unit range (first unit | count
// << 32), so a kept task's walk starts without the dependent task_begin load;
// the skip flags are then indexed by the task's first unit.
#if SSB_TLIST64
typedef int64_t ssb_tentry;
#else
typedef int32_t ssb_tentry;
#endif
#ifndef SSB_PF_HEAD
#define SSB_PF_HEAD 0  // steps (512 B) of each unit prefetched when its task starts
#endif
constexpr int32_t kPfHeadSteps = SSB_PF_HEAD;

struct Args32 {
  const int32_t* col;
  const int64_t* cs;
  const int32_t* cl;
  const ssb_unit* units;
  const int32_t* task_begin;
  const int32_t* split_units;
  uint32_t* split_hit;
  int32_t* split_best;
  uint32_t* split_count;
  uint32_t* visited;
  uint32_t* F0;
  uint32_t* F1;
  uint32_t* S0;
  uint32_t* S1;
  uint32_t* S2;
  int32_t* level;
  int32_t* parent;
  int64_t* stats;      // [kItersPerLaunch][kStatW]
  uint32_t* task_ctr;  // [kItersPerLaunch] tasks grabbed per iteration
  uint32_t* task_out;  // [kItersPerLaunch] tasks kept for the next iteration
  ssb_tentry* tlist0;  // active task lists (ping-pong by iteration parity)
  ssb_tentry* tlist1;
  uint8_t* tskip;      // per task (SSB_TLIST64: per first unit): every unit skipped in its last sweep
  unsigned long long* gone_chunks;  // chunks of retired tasks (skipped forever)
  int32_t retire_once; // retire a task the first time all its units are skipped (see run_tasks)
  int32_t hash_on;     // sparse iterations also build the hashed summary (Probe kHash), used next
  uint32_t HB;         // summary bits (SW * 32)
  uint32_t hash_arg;   // summary_hash's shift: 32 - log2 of the hashed bits (a power of two <= HB)
  int64_t hash_thr;    // early-exit iterations probe the hashed summary while |F_{k-1}| <= this
  int32_t hash_prev_in; // iteration k_begin - 1 (a previous launch) built the hashed summary
  uint32_t* H0;        // hashed summaries, rotating like S0..S2
  uint32_t* H1;
  uint32_t* H2;
  int32_t n_tasks;     // active tasks entering iteration k_begin
  unsigned long long gone_base;  // chunks of tasks retired before k_begin
  int64_t front_in;    // frontier size entering iteration k_begin
  int64_t dense_thr;   // frontiers above this use the early-exit sweeps
  int64_t direct_thr;  // ... and above this the summary-free direct probes
  int32_t n_chunks;
  int32_t PW;      // frontier prefix words staged in shared memory
  int32_t SW;      // summary words staged in shared memory
  int32_t gshift;  // summary granularity: 2^gshift frontier words per bit
  int32_t L;       // slimchunk_len for the subchunk counter (0 = off)
  int32_t slimwork;
  int32_t root_code;  // sel-max parent position recorded at iteration 1
  uint32_t last_real;  // real-row mask of the last chunk
  int32_t k_begin;
  int32_t k_end;
  int* trace;  // debug progress words in mapped host memory (SSB_TRACE), or null
  // Device-resident carry between launches (asynchronous shard stepping), or
  // null: {|F| entering k_begin, active tasks, retired chunks}. Read at launch
  // start instead of n_tasks / front_in / gone_base, written back at the end;
  // a launch entering with |F| = 0 (the BFS already converged) does nothing.
  int64_t* carry;
  // Mapped pinned host memory receiving the first min(k_end - k_begin,
  // kRecFirst) records when the launch ends (CTA 0), or null: the host reads
  // them after the launch without a copy on the stream.
  int64_t* rec_host;
};

// Fused multi-GPU exchange (chunk-range shards): every rank's
// frontier F0/F1 and summaries S0..S2 live in a WINDOW that the other ranks
// map (CUDA IPC over NVLink, or plain device memory when the ranks are
// emulated inside one cooperative launch). After each iteration's sweep the
// rank stores its owned frontier words and ORs its owned summary words
// straight into every peer's window, publishes |newly| in a slot ring, and
// meets the others at a counter barrier in its own window — the reference's
// per-iteration all-gather + is_converged without leaving the kernel.
constexpr int kMaxRanks = 8;
constexpr int kSlotRing = 64;  // generations of |newly| slots kept in a window
constexpr int kMaxSeg = 8;     // owned chunk segments per rank
struct P2PArgs {
  uint32_t* win[kMaxRanks];    // every rank's window base (peer-mapped)
  int64_t offF[2];             // word offsets of F0 / F1 in a window
  int64_t offS[3];             // ... of S0 / S1 / S2
  int64_t offSlots;            // int64 [kSlotRing][kMaxRanks]
  int64_t offArrive;           // uint64 arrival counter (cumulative)
  unsigned long long gen_base; // barrier generations completed before this launch
  unsigned long long arrivals; // CTAs per generation over all ranks
  unsigned long long timeout_ns; // a peer missing for this long traps the kernel (0: wait forever)
  int32_t rank, world;
  int32_t nseg;                // owned chunk segments (round-robin partitions)
  int32_t wseg[2 * kMaxSeg];   // their frontier words [b, e) (= chunks, C = 32)
  int32_t sseg[2 * kMaxSeg];   // their summary words [b, e) (shared at the ends)
};
constexpr int kMaxVRanks = 8;  // ranks emulated in one launch (single-GPU tests, config 5 shape)
struct GroupArgs {
  Args32 a[kMaxVRanks];
  P2PArgs x[kMaxVRanks];
  int32_t nvb;  // CTAs per (virtual) rank
};

#define TRACE(slot, v)                                           \
  do {                                                           \
    if (a.trace) *reinterpret_cast<volatile int*>(&a.trace[slot]) = (v); \
  } while (0)

// Shared-memory image of the frontier F_{k-1} as ONE virtual bit array:
//   bits [0, P)      fine frontier bits of vertices [0, P), P = 32·PW (the
//                    hubs: the σ = n sort puts high degrees first)
//   bits [P, P+G)    summary of the rest: bit P + t says vertices
//                    [P + 256t, P + 256t + 256) hold a frontier vertex
// preceded by 4 zero words, the target of padding cells (c = -1). Cell c maps
// to virtual bit v = min(c, (c >> S) + P - (P >> S)) — c itself in the prefix,
// the bit of its absolute 2^S-vertex group in the tail (P is a multiple of
// 2^S and x - (x >> S) is monotone, so the min picks the right branch) — so
// every probe is the same shared load; only a set summary bit needs the exact
// word from global memory (L2-resident).
// S is chosen per graph (geometry32): 8 when the prefix holds most cell
// targets (hub-heavy graphs), 6 — a 4x finer summary at the cost of prefix —
// when it does not (low-skew graphs such as Erdős–Rényi).
//
// kHash (hub-heavy graphs, iterations after a sparse one): the summary holds
// one bit per tail frontier VERTEX at a multiplicative hash of its position
// instead of one bit per 2^S-vertex group. Frontier vertices and cell targets
// crowd the same low tail positions (both degree-weighted), so group bits are
// set where the probes land: at S26 iteration 3 a hashed summary of the same
// size is set for 5-9x fewer open tail cells (scripts/summary_fp.py). A set
// bit still only sends the cell to its exact word: no false negatives.
// Fibonacci hash: the top log2(bits) bits of pos · 2^32/φ, `shift` = 32 -
// log2(bits) for the largest power of two of bits within the summary (a
// shift, not a high multiply: A/B at S26 4.301 -> 4.279 ms per BFS, iteration
// 3 -21 µs, `profiles/r2v_ab_hash_shift.txt`)
__device__ __forceinline__ uint32_t summary_hash(int32_t pos, uint32_t shift) {
  return (uint32_t(pos) * 0x9E3779B1u) >> shift;
}

template <int kS, bool kHash = false>
struct Probe {
  static constexpr int kShift = kS;
  const uint32_t* sm;  // word 0 = first prefix word; sm[-4..-1] are zero
  const uint32_t* Fc;  // the full frontier in global memory
  int32_t P;           // prefix vertices (multiple of 2^S)
  int32_t Pt;          // P - (P >> S); kHash: summary_hash's shift

  // virtual bit of cell target c (padding c = -1 maps to a zero word)
  __device__ __forceinline__ int32_t vidx(int32_t c) const {
    if constexpr (kHash) return c < P ? c : P + int32_t(summary_hash(c, uint32_t(Pt)));
    else return min(c, (c >> kS) + Pt);
  }
  // the probe's word rotated so that its bit sits at bit 0
  __device__ __forceinline__ uint32_t vrot(int32_t c) const {
    const int32_t v = vidx(c);
    const uint32_t word = sm[v >> 5];
    return __funnelshift_r(word, word, v);  // bit (v mod 32) -> bit 0
  }
  __device__ __forceinline__ uint32_t exact(int32_t c) const {
    return (Fc[c >> 5] >> (c & 31)) & 1u;  // L1 is invalidated by every grid.sync fence
  }
  // The four probes of one int4 as one batch: four shared loads issued back to
  // back (one shared-memory round trip instead of four dependent ones).
  __device__ __forceinline__ uint32_t vbits4(const int32_t (&c)[4]) const {
    int32_t v[4];
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = vidx(c[q]);
    const uint32_t base = uint32_t(__cvta_generic_to_shared(sm));
    asm volatile(
        "ld.shared.u32 %0, [%4];\n\t"
        "ld.shared.u32 %1, [%5];\n\t"
        "ld.shared.u32 %2, [%6];\n\t"
        "ld.shared.u32 %3, [%7];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
        : "r"(base + 4u * uint32_t(v[0] >> 5)), "r"(base + 4u * uint32_t(v[1] >> 5)),
          "r"(base + 4u * uint32_t(v[2] >> 5)), "r"(base + 4u * uint32_t(v[3] >> 5)));
    uint32_t b = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) b |= (__funnelshift_r(w[q], w[q], v[q]) & 1u) << q;
    return b;
  }
  // Exact frontier bits of the cells flagged in `need`, the four global loads
  // in flight together (unflagged lanes re-read word 0: one shared sector).
  __device__ __forceinline__ uint32_t exact4(const int32_t (&c)[4], uint32_t need) const {
    uint32_t w[4];
    const uint32_t* p[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) p[q] = Fc + (((need >> q) & 1u) ? (c[q] >> 5) : 0);
    asm volatile(
        "ld.global.u32 %0, [%4];\n\t"
        "ld.global.u32 %1, [%5];\n\t"
        "ld.global.u32 %2, [%6];\n\t"
        "ld.global.u32 %3, [%7];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
        : "l"(p[0]), "l"(p[1]), "l"(p[2]), "l"(p[3]));
    uint32_t b = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) b |= ((w[q] >> (c[q] & 31)) & 1u) << q;
    return b & need;
  }
};

// Four cells of one column (rows 4·lg .. 4·lg+3). `hit` bit q says row q is
// decided: for the "any" semirings the first frontier neighbour decides the
// row (columns are swept forward), for sel-max the first one met sweeping the
// columns BACKWARD is the largest position (rows are ascending), i.e. the
// reference's max. Decided rows skip their remaining probes — the reduction
// short-circuits, the column stream itself is still read in full. Prefix hits
// are final; a set summary bit is resolved against the global frontier before
// the next column, so each row still sees its cells in sweep order.
// kEarly = false (sparse frontiers, where hits are rare): no masking, every
// column is probed in ascending order and sel-max keeps the LAST hit — the
// cheapest instruction stream. kEarly = true (dense frontiers, where the exact
// lookups dominate): decided rows are masked out as described above.
// Early-exit cells without the summary, for iterations whose previous
// frontier sets most summary bits anyway (|F| above the summary's bit count):
// each open cell is ONE generic load of its exact frontier word — from the
// shared image for c < P, from the global frontier (L1/L2) otherwise — so
// tail cells skip the summary probe and its dependent second load. Decided
// rows and padding cells read a zero word of the image.
template <bool kSelMax, class Probe>
__device__ __forceinline__ void take_cells_direct(const int4 v, const Probe& pr, uint32_t& hit,
                                                  int32_t (&best)[4]) {
  const int32_t c[4] = {v.x, v.y, v.z, v.w};
  const uint32_t* p[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool open = !((hit >> q) & 1u) && c[q] >= 0;
    p[q] = !open ? pr.sm - 4 : (c[q] < pr.P ? pr.sm : pr.Fc) + (c[q] >> 5);
  }
  uint32_t w[4];
  asm volatile(
      "ld.u32 %0, [%4];\n\t"
      "ld.u32 %1, [%5];\n\t"
      "ld.u32 %2, [%6];\n\t"
      "ld.u32 %3, [%7];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
      : "l"(p[0]), "l"(p[1]), "l"(p[2]), "l"(p[3]));
  uint32_t b = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t bit = (w[q] >> (c[q] & 31)) & 1u;
    if (kSelMax) best[q] = bit ? c[q] : best[q];
    b |= bit << q;
  }
  hit |= b;
}

#ifdef SSB_COUNT
// debug counters (SSB_COUNT builds, one launch per iteration): open probes,
// tail probes, exact lookups, exact hits, warp steps with a lookup
__device__ unsigned long long g_cnt[8];
#endif
#ifndef SSB_LEAN_DENSE
#define SSB_LEAN_DENSE 2  // A/B: S26 4.548 -> 4.470 (1) -> 4.439 (2) ms per BFS, S22 0.443 -> 0.434, ER flat
#endif
// The summary-probe early-exit step with mask arithmetic instead of per-cell
// selects: one rotate-and-mask per probe puts its bit at position q, the
// prefix test is a 4-bit mask, prefix hits and exact hits meet in ONE mask
// and one round of best updates. (The mid-size-frontier iterations of
// hub-heavy graphs are ALU-bound in this step.)
template <bool kSelMax, class Probe>
__device__ __forceinline__ void take_cells_lean(const int4 v, const Probe& pr, uint32_t& hit,
                                                int32_t (&best)[4]) {
  const int32_t c[4] = {v.x, v.y, v.z, v.w};
  int32_t vq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) vq[q] = pr.vidx(c[q]);
  uint32_t w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) w[q] = pr.sm[vq[q] >> 5];  // shared image (padding: the zero words)
  uint32_t vb = 0, pm = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    vb |= __funnelshift_r(w[q], w[q], vq[q] - q) & (1u << q);  // bit vq -> bit q
    pm |= uint32_t(c[q] < pr.P) << q;
  }
  vb &= ~hit;
  const uint32_t need = vb & ~pm;  // set summary bit: the exact word decides
  uint32_t e = vb & pm;            // prefix bits are exact
  if (__any_sync(0xffffffffu, need)) {
    uint32_t x[4];
#if SSB_LEAN_DENSE >= 2
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      x[q] = 0u;
      if ((need >> q) & 1u) x[q] = pr.Fc[uint32_t(c[q]) >> 5];
    }
#else
#pragma unroll
    for (int q = 0; q < 4; ++q) x[q] = pr.Fc[((need >> q) & 1u) ? (uint32_t(c[q]) >> 5) : 0u];
#endif
#pragma unroll
    for (int q = 0; q < 4; ++q) e |= __funnelshift_r(x[q], x[q], c[q] - q) & (need & (1u << q));
  }
  hit |= e;
  if (kSelMax && (SSB_LEAN_DENSE < 2 || __any_sync(0xffffffffu, e))) {
#pragma unroll
    for (int q = 0; q < 4; ++q) best[q] = ((e >> q) & 1u) ? c[q] : best[q];
  }
}

template <bool kSelMax, bool kEarly, bool kDirect, class Probe>
__device__ __forceinline__ void take_cells(const int4 v, const Probe& pr, uint32_t& hit,
                                           int32_t (&best)[4]) {
  if constexpr (kDirect) {
    take_cells_direct<kSelMax>(v, pr, hit, best);
    return;
  }
  if constexpr (kEarly && SSB_LEAN_DENSE) {
    take_cells_lean<kSelMax>(v, pr, hit, best);
    return;
  }
  const int32_t c[4] = {v.x, v.y, v.z, v.w};
  const uint32_t open = kEarly ? ~hit : 0xffffffffu;
  // Sparse sweeps are instruction-issue bound and their probes almost always
  // miss: test the four probe bits together and leave the per-cell bookkeeping
  // to the (warp-uniform) rare path. Dense sweeps batch the four shared loads.
  uint32_t rot[4];
  if (!kEarly) {
#pragma unroll
    for (int q = 0; q < 4; ++q) rot[q] = pr.vrot(c[q]);
    if (!__any_sync(0xffffffffu, (rot[0] | rot[1] | rot[2] | rot[3]) & 1u)) return;
  }
  const uint32_t vb = kEarly ? pr.vbits4(c) & open : 0u;
  uint32_t need = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t b = kEarly ? (vb >> q) & 1u : rot[q] & 1u;
    const bool def = b && c[q] < pr.P;
    if (kSelMax) best[q] = def ? c[q] : best[q];
    // sel-max without early exit derives its row mask from best afterwards
    if (!kSelMax || kEarly) hit |= uint32_t(def) << q;
    need |= uint32_t(b && c[q] >= pr.P) << q;
  }
#ifdef SSB_COUNT
  {
    uint32_t probes = 0, tail = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool o = (open >> q) & 1u;
      probes += o;
      tail += o && c[q] >= pr.P;
    }
    const uint32_t pw = __reduce_add_sync(0xffffffffu, probes), tw = __reduce_add_sync(0xffffffffu, tail),
                   nw = __reduce_add_sync(0xffffffffu, uint32_t(__popc(need)));
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&g_cnt[0], (unsigned long long)pw);
      atomicAdd(&g_cnt[1], (unsigned long long)tw);
      atomicAdd(&g_cnt[2], (unsigned long long)nw);
      if (nw) atomicAdd(&g_cnt[4], 1ull);
    }
  }
#endif
  if (__any_sync(0xffffffffu, need)) {  // warp-uniform: no reconvergence bookkeeping
    if (kEarly) {  // (A/B: the batched form does not help the sparse sweeps; ER 2^26 k = 4-5 +5% slower)
      const uint32_t e = pr.exact4(c, need);
#ifdef SSB_COUNT
      {
        const uint32_t ew = __reduce_add_sync(0xffffffffu, uint32_t(__popc(e)));
        if ((threadIdx.x & 31) == 0) atomicAdd(&g_cnt[3], (unsigned long long)ew);
      }
#endif
      hit |= e;
      if (kSelMax) {
#pragma unroll
        for (int q = 0; q < 4; ++q) best[q] = ((e >> q) & 1u) ? c[q] : best[q];
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (((need >> q) & 1u) && pr.exact(c[q])) {
          hit |= 1u << q;
          if (kSelMax) best[q] = c[q];
        }
      }
    }
  }
}

// One 128-byte column of padding cells: the load target of groups without a
// unit, so the sweep needs no per-load predicates.
__device__ __align__(16) int32_t g_pad_column[32] = {
    -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1,
    -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};

#ifndef SSB_WARP_UNIT_COLS
#define SSB_WARP_UNIT_COLS 32  // A/B at S26: 16 -> 32 gives Kronecker +1-2%, Erdős–Rényi +13%
#endif
constexpr int32_t kWarpUnitCols = SSB_WARP_UNIT_COLS;  // units at least this long use the warp-wide sweep

#ifndef SSB_KEEP_BUF
#define SSB_KEEP_BUF 1  // kept tasks appended 32 per atomic (0: one atomic per task)
#endif
#ifndef SSB_GRAB
#define SSB_GRAB 1  // tasks taken per counter atomic in early-exit iterations
#endif
#ifndef SSB_SPLIT_X
#define SSB_SPLIT_X 1  // tasks are shared by D ≤ 8 warps while n_tasks · D · X ≤ warps (0: never)
#endif

// Completes one work unit; called by all 32 lanes, `valid` per 8-lane group.
// m = the unit's 32-row hit mask, best[q] = last hit of row 4·lg+q (sel-max).
// SlimChunk combine (bfs.cpp:205-220): partial results of a split chunk meet
// in a scratch slot and the unit that arrives last finalises the chunk —
// post_process_rows (semiring.cpp:90-124) in 1-bit form.
template <bool kSelMax, bool kEarly, bool kHash>
__device__ __forceinline__ void finish_unit(const Args32& a, int32_t k, uint32_t* Fn, uint32_t* Sn,
                                            bool valid, int32_t chunk, int32_t split, uint32_t uvis,
                                            uint32_t ureal, uint32_t m, int32_t (&best)[4], int grp,
                                            int lg, uint32_t gmask, uint32_t& c_front) {
  bool fin = valid && split < 0;
  const bool sp = valid && split >= 0;
  if (sp) {
    if (lg == 0 && m) atomicOr(&a.split_hit[split], m);
    if (kSelMax) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (best[q] >= 0) atomicMax(&a.split_best[split * 32 + 4 * lg + q], best[q]);
    }
    __threadfence();
  }
  __syncwarp();
  uint32_t last = 0;
  if (sp && lg == 0) {
    const uint32_t arrived = atomicAdd(&a.split_count[split], 1u) + 1u;
    last = arrived == uint32_t(a.split_units[split]);
  }
  last = __shfl_sync(0xffffffffu, last, grp * 8);
  if (sp && last) {
    __threadfence();
    fin = true;
    if (lg == 0) {
      m = atomicExch(&a.split_hit[split], 0u);
      a.split_count[split] = 0u;
    }
    m = __shfl_sync(gmask, m, grp * 8, 32);
    if (kSelMax) {
#pragma unroll
      for (int q = 0; q < 4; ++q) best[q] = atomicExch(&a.split_best[split * 32 + 4 * lg + q], -1);
    }
  }
  if (fin) {
    const uint32_t newly = m & ~uvis & ureal;
    if (lg == 0) {
      Fn[chunk] = newly;
      if (newly) {
        a.visited[chunk] = uvis | newly;
        if (chunk >= a.PW) {
          const int32_t gi = (chunk - a.PW) >> a.gshift;
          atomicOr(&Sn[gi >> 5], 1u << (gi & 31));
        }
        c_front += __popc(newly);
      }
    }
    if (newly) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int32_t r = 4 * lg + q;
        if ((newly >> r) & 1u) {
          const int64_t row = int64_t(chunk) * 32 + r;
          a.level[row] = k;
          if (kSelMax) a.parent[row] = k == 1 ? a.root_code : best[q];
          // sparse iterations also build the hashed summary of the tail
          // frontier (the pointer comes from the parameter space: nothing
          // extra stays live through the sweep)
          if (kHash && !kEarly && chunk >= a.PW) {
            uint32_t* Hn = (k % 3) == 0 ? a.H0 : ((k % 3) == 1 ? a.H1 : a.H2);
            const uint32_t h = summary_hash(int32_t(row), a.hash_arg);
            atomicOr(&Hn[h >> 5], 1u << (h & 31));
          }
        }
      }
    }
  }
}

// Whole-warp sweep of one long unit starting at `base` (len columns). int4 i
// of the unit = column i/8, rows 4(i%8)..+3; lane l takes i = 32s + l, so lg
// (rows) is fixed per lane and grp picks the column within each 4-column
// step. Out-of-range indices re-read the lane's own rows of the last column
// (idempotent). Loads run four steps ahead of the probes. On return `hit` and
// `best` are combined over the four lanes that share rows. Early-exit sweeps
// stop the unit once all 32 rows are decided (the semiring "plus" has
// short-circuited for every row, so the remaining columns cannot change the
// result). Returns the number of columns swept.
template <bool kSelMax, bool kEarly, bool kDirect, class Probe>
__device__ __forceinline__ int32_t sweep_long(const int4* base, int32_t len, int lane, int lg,
                                           const Probe& pr, uint64_t pol, uint32_t& hit,
                                           int32_t (&best)[4], ImgWait& iw) {
  const int32_t nv = len * 8, imax = nv - 8 + lg;
  const int32_t nsteps = (nv + 31) >> 5;
  // lanes sharing rows exchange decided-row bits after every 4 steps
  // ... and report whether every row of the unit is decided (warp-uniform)
  auto share = [&]() -> bool {
    if (kEarly) {
      hit |= __shfl_xor_sync(0xffffffffu, hit, 8);
      hit |= __shfl_xor_sync(0xffffffffu, hit, 16);
      return __all_sync(0xffffffffu, hit == 0xfu);
    }
    return false;
  };
  int32_t swept = len;
  if (!(kSelMax && kEarly)) {
    // forward sweep: step s = 0, 1, ...
    int4 v0 = ld_stream(base + min(lane, imax), pol);
    int4 v1 = ld_stream(base + min(32 + lane, imax), pol);
    int4 v2 = ld_stream(base + min(64 + lane, imax), pol);
    int4 v3 = ld_stream(base + min(96 + lane, imax), pol);
    iw();  // the image is needed from the first probe on
    // Steps s+4..s+7 are all full (no clamping) while s + 9 <= nsteps; the
    // prefetch pointer then advances by 2 KB per 4 steps, offsets immediate.
    const int4* pf = base + 128 + lane;
    int32_t s = 0;
    bool done = false;
    for (; s + 9 <= nsteps; s += 4, pf += 128) {
      if (kPfAhead > 0 && lane == 0 && s + 9 + 4 * kPfAhead <= nsteps)
        prefetch_l2(pf - lane + 128 * kPfAhead, 2048);
      take_cells<kSelMax, kEarly, kDirect>(v0, pr, hit, best);
      v0 = ld_stream(pf, pol);
      take_cells<kSelMax, kEarly, kDirect>(v1, pr, hit, best);
      v1 = ld_stream(pf + 32, pol);
      take_cells<kSelMax, kEarly, kDirect>(v2, pr, hit, best);
      v2 = ld_stream(pf + 64, pol);
      take_cells<kSelMax, kEarly, kDirect>(v3, pr, hit, best);
      v3 = ld_stream(pf + 96, pol);
      if (share()) {
        done = true;
        swept = 4 * (s + 4);
        break;
      }
    }
    for (; !done && s < nsteps; s += 4) {
      const bool more = s + 4 < nsteps;  // warp-uniform
      const int32_t i0 = (s + 4) * 32 + lane;
      take_cells<kSelMax, kEarly, kDirect>(v0, pr, hit, best);
      if (more) v0 = ld_stream(base + min(i0, imax), pol);
      take_cells<kSelMax, kEarly, kDirect>(v1, pr, hit, best);
      if (more) v1 = ld_stream(base + min(i0 + 32, imax), pol);
      take_cells<kSelMax, kEarly, kDirect>(v2, pr, hit, best);
      if (more) v2 = ld_stream(base + min(i0 + 64, imax), pol);
      take_cells<kSelMax, kEarly, kDirect>(v3, pr, hit, best);
      if (more) v3 = ld_stream(base + min(i0 + 96, imax), pol);
      if (share()) {
        swept = min(len, 4 * (s + 4));
        break;
      }
    }
  } else {
    // backward sweep (sel-max, early exit): steps nsteps-1 .. 0, clamped at 0
    const int32_t top = nsteps - 1;
    auto at = [&](int32_t st) { return base + min(32 * max(st, 0) + lane, imax); };
    int4 v0 = ld_stream(at(top), pol);
    int4 v1 = ld_stream(at(top - 1), pol);
    int4 v2 = ld_stream(at(top - 2), pol);
    int4 v3 = ld_stream(at(top - 3), pol);
    iw();
    // steps top-r-4 .. top-r-7 are all full and >= 0 while r + 8 <= nsteps
    const int4* pf = base + 32 * (top - 4) + lane;
    int32_t r = 0;
    bool done = false;
    // columns in the top r steps (the top step may be partial)
    auto cols_of = [&](int32_t st) { return max(0, len - 4 * (nsteps - st)); };
    for (; r + 8 <= nsteps; r += 4, pf -= 128) {
      // steps top-r-4-4A .. top-r-7-4A: int4 [32(top-r-7-4A), +128)
      if (kPfAhead > 0 && lane == 0 && r + 8 + 4 * kPfAhead <= nsteps)
        prefetch_l2(pf - lane - 96 - 128 * kPfAhead, 2048);
      take_cells<kSelMax, kEarly, kDirect>(v0, pr, hit, best);
      v0 = ld_stream(pf, pol);
      take_cells<kSelMax, kEarly, kDirect>(v1, pr, hit, best);
      v1 = ld_stream(pf - 32, pol);
      take_cells<kSelMax, kEarly, kDirect>(v2, pr, hit, best);
      v2 = ld_stream(pf - 64, pol);
      take_cells<kSelMax, kEarly, kDirect>(v3, pr, hit, best);
      v3 = ld_stream(pf - 96, pol);
      if (share()) {
        done = true;
        swept = cols_of(r + 4);
        break;
      }
    }
    for (; !done && r < nsteps; r += 4) {
      const bool more = r + 4 < nsteps;  // warp-uniform
      take_cells<kSelMax, kEarly, kDirect>(v0, pr, hit, best);
      if (more) v0 = ld_stream(at(top - r - 4), pol);
      take_cells<kSelMax, kEarly, kDirect>(v1, pr, hit, best);
      if (more) v1 = ld_stream(at(top - r - 5), pol);
      take_cells<kSelMax, kEarly, kDirect>(v2, pr, hit, best);
      if (more) v2 = ld_stream(at(top - r - 6), pol);
      take_cells<kSelMax, kEarly, kDirect>(v3, pr, hit, best);
      if (more) v3 = ld_stream(at(top - r - 7), pol);
      if (share()) {
        swept = cols_of(min(nsteps, r + 4));
        break;
      }
    }
  }
  // combine the four column groups
  if (kSelMax) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      best[q] = max(best[q], __shfl_xor_sync(0xffffffffu, best[q], 8));
      best[q] = max(best[q], __shfl_xor_sync(0xffffffffu, best[q], 16));
      hit |= uint32_t(best[q] >= 0) << q;
    }
  }
  hit |= __shfl_xor_sync(0xffffffffu, hit, 8);
  hit |= __shfl_xor_sync(0xffffffffu, hit, 16);
  return swept;
}

// One short unit per 8-lane group: column j of the unit is int4 p[8j] (lane
// lg: rows 4lg..4lg+3). Groups shorter than maxlen re-read their last (or,
// backward, first) column — idempotent for both reductions; groups without a
// unit read a padding column. Loads run 4 columns ahead of the probes.
// Early-exit sweeps stop once every row of the four units is decided. Returns
// the number of column steps run (the group's unit swept min(len, that)).
template <bool kSelMax, bool kEarly, bool kDirect, class Probe>
__device__ __forceinline__ int32_t sweep_group(const int4* p, int32_t jlast, int64_t stride,
                                            int32_t maxlen, const Probe& pr, uint64_t pol,
                                            uint32_t& hit, int32_t (&best)[4], ImgWait& iw) {
  constexpr bool kBack = kSelMax && kEarly;
  auto at = [&](int32_t j) { return p + (kBack ? max(jlast - j, 0) : min(j, jlast)) * stride; };
  int4 v0 = ld_stream(at(0), pol);
  int4 v1 = ld_stream(at(1), pol);
  int4 v2 = ld_stream(at(2), pol);
  int4 v3 = ld_stream(at(3), pol);
  iw();
  int32_t j = 0;
  while (j < maxlen) {
    const bool more = j + 4 < maxlen;  // warp-uniform
    take_cells<kSelMax, kEarly, kDirect>(v0, pr, hit, best);
    if (more) v0 = ld_stream(at(j + 4), pol);
    take_cells<kSelMax, kEarly, kDirect>(v1, pr, hit, best);
    if (more) v1 = ld_stream(at(j + 5), pol);
    take_cells<kSelMax, kEarly, kDirect>(v2, pr, hit, best);
    if (more) v2 = ld_stream(at(j + 6), pol);
    take_cells<kSelMax, kEarly, kDirect>(v3, pr, hit, best);
    if (more) v3 = ld_stream(at(j + 7), pol);
    j += 4;
    if (kEarly && __all_sync(0xffffffffu, hit == 0xfu)) break;
  }
  if (kSelMax) {
#pragma unroll
    for (int q = 0; q < 4; ++q) hit |= uint32_t(best[q] >= 0) << q;
  }
  return min(j, maxlen);
}

#ifdef SSB_PHASES
__device__ unsigned long long g_phase[4];  // debug: staging, tasks, barrier ns; iterations
#endif

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Cross-rank barrier of generation `gen` (called by every CTA of every rank):
// this CTA's prior stores (local and peer) are released to all ranks, then
// thread 0 waits until every CTA of every rank has arrived.
__device__ __forceinline__ void p2p_barrier(const P2PArgs& x, unsigned long long gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int r = 0; r < x.world; ++r)
      atomicAdd_system(reinterpret_cast<unsigned long long*>(x.win[r] + x.offArrive), 1ull);
    const unsigned long long* mine =
        reinterpret_cast<const unsigned long long*>(x.win[x.rank] + x.offArrive);
    const uint64_t t0 = x.timeout_ns ? globaltimer() : 0;
    while (ld_acquire_sys(mine) < gen * x.arrivals) {
      __nanosleep(64);
      // a rank that never arrives (died, or never launched) would hang every
      // peer forever: fail the launch instead (the host sees an error)
      if (x.timeout_ns && globaltimer() - t0 > x.timeout_ns) asm volatile("trap;");
    }
  }
  __syncthreads();
  __threadfence();  // no stale L1 lines of the peers' words past this point
}

// One iteration's exchange; returns the global |newly| (every rank's count).
// Fn / Sn are this rank's window regions of the iteration just swept.
__device__ __forceinline__ int64_t p2p_exchange(const P2PArgs& x, int32_t k, const uint32_t* Fn,
                                                const uint32_t* Sn, int64_t local_front,
                                                unsigned long long gen, int vb, int nvb) {
  const int tid = vb * kThreads + threadIdx.x, nth = nvb * kThreads;
  for (int r = 0; r < x.world; ++r) {
    if (r == x.rank) continue;
    uint32_t* pf = x.win[r] + x.offF[k & 1];
    uint32_t* ps = x.win[r] + x.offS[k % 3];
    for (int q = 0; q < x.nseg; ++q) {
      for (int32_t w = x.wseg[2 * q] + tid; w < x.wseg[2 * q + 1]; w += nth) pf[w] = __ldcg(Fn + w);
      // summary words at the segment ends are shared with other ranks
      for (int32_t w = x.sseg[2 * q] + tid; w < x.sseg[2 * q + 1]; w += nth) {
        const uint32_t v = __ldcg(Sn + w);
        if (v) atomicOr_system(&ps[w], v);
      }
    }
  }
  const int slot = int(gen % kSlotRing) * kMaxRanks;
  if (vb == 0 && threadIdx.x == 0)
    for (int r = 0; r < x.world; ++r)
      *reinterpret_cast<volatile int64_t*>(reinterpret_cast<int64_t*>(x.win[r] + x.offSlots) + slot +
                                           x.rank) = local_front;
  p2p_barrier(x, gen);
  const volatile int64_t* sl = reinterpret_cast<const int64_t*>(x.win[x.rank] + x.offSlots) + slot;
  int64_t front = 0;
  for (int r = 0; r < x.world; ++r) front += sl[r];
  return front;
}

// The BFS loop of one rank. vb / nvb: this CTA's index and the CTA count of
// the rank (the whole grid, except when ranks are emulated in one launch).
template <bool kSelMax, int kS, bool kP2P, bool kHash>
__device__ __forceinline__ void bfs32_body(const Args32& a, const P2PArgs& x, const int vb,
                                           const int nvb) {
  extern __shared__ uint4 smem_v4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem_v4);
  uint32_t* summ = sm + 4 + a.PW;
  __shared__ __align__(8) unsigned long long stage_bar_storage;
  unsigned long long* stage_bar = &stage_bar_storage;
  uint32_t stage_phase = 0;
  __shared__ unsigned long long blk[6];  // stats slots 0-4 and 6
  __shared__ int64_t bcast[3];           // the iteration's |newly|, kept tasks, retired chunks
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(stage_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    smem_v4[0] = make_uint4(0u, 0u, 0u, 0u);  // the zero words in front of the image (never staged over)
  }
  if (threadIdx.x < 6) blk[threadIdx.x] = 0ull;
  __syncthreads();

  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int grp = lane >> 3;  // 8-lane group: one work unit
  const int lg = lane & 7;    // rows 4*lg .. 4*lg+3 of the unit's chunk
  const uint32_t gmask = 0xffu << (grp * 8);
  const uint64_t pol = evict_first_policy();
  uint64_t t_prev = 0;
  if (vb == 0 && threadIdx.x == 0) t_prev = globaltimer();
  int32_t n_in = a.n_tasks;                  // active tasks entering iteration k
  int64_t front_in = a.front_in;             // |F_{k-1}|
  unsigned long long gone = a.gone_base;     // chunks of tasks retired before k
  if (a.carry) {  // grid-uniform: every CTA reads the words the previous kernels wrote
    front_in = a.carry[0];
    n_in = int32_t(a.carry[1]);
    gone = static_cast<unsigned long long>(a.carry[2]);
    if (front_in == 0) return;
  }
  // every rank has reset its window before anyone stores into it
  if (kP2P) p2p_barrier(x, x.gen_base + 1);
  bool hash_prev = kHash && a.hash_prev_in;  // the previous iteration built the hashed summary

  for (int32_t k = a.k_begin; k < a.k_end; ++k) {
    const int32_t rec = k - a.k_begin;
#ifdef SSB_PHASES
    uint64_t ph0 = 0, ph1 = 0, ph2 = 0;
    if (vb == 0 && threadIdx.x == 0) ph0 = globaltimer();
#endif
    const uint32_t* Fc = ((k - 1) & 1) ? a.F1 : a.F0;
    uint32_t* Fn = (k & 1) ? a.F1 : a.F0;
    const int32_t km3 = (k - 1) % 3;
    const uint32_t* Sc = km3 == 0 ? a.S0 : (km3 == 1 ? a.S1 : a.S2);
    uint32_t* Sn = (k % 3) == 0 ? a.S0 : ((k % 3) == 1 ? a.S1 : a.S2);
    uint32_t* Sx = ((k + 1) % 3) == 0 ? a.S0 : (((k + 1) % 3) == 1 ? a.S1 : a.S2);
    const uint32_t* Hc = km3 == 0 ? a.H0 : (km3 == 1 ? a.H1 : a.H2);
    uint32_t* Hx = ((k + 1) % 3) == 0 ? a.H0 : (((k + 1) % 3) == 1 ? a.H1 : a.H2);

    // sweep mode of this iteration (grid-uniform, from |F_{k-1}|): dense ->
    // early exit; dense and direct -> summary-free probes, whose image is the
    // prefix alone, so the summary's words extend the prefix instead
    const bool dense = front_in > a.dense_thr;
    const bool direct = dense && front_in > a.direct_thr;
    const int32_t img_words = direct ? a.PW + a.SW : a.PW;
    // hashed summary (hub-heavy graphs): built by sparse iterations (whose
    // output frontier is small enough for one atomic per tail vertex), probed
    // by the next one unless it probes exactly; the block summary is always
    // built, so a launch starting mid-BFS simply uses it
    const bool use_hash = kHash && hash_prev && dense && !direct && front_in <= a.hash_thr;
    // -- stage the frontier prefix and the summary into shared memory -------
    // One thread issues TMA bulk copies (global -> shared, completion on an
    // mbarrier); everyone else goes on to the per-iteration setup and then
    // waits on the barrier's phase.
    {
      if (threadIdx.x == 0) {
        // prior generic accesses (reads of the previous image, other CTAs'
        // frontier stores ordered by grid.sync) before the async-proxy copies
        asm volatile("fence.proxy.async;" ::: "memory");
        const uint32_t bytes_p = uint32_t(img_words) * 4u, bytes_s = direct ? 0u : uint32_t(a.SW) * 4u;
        mbar_arrive_expect_tx(stage_bar, bytes_p + bytes_s);
        bulk_g2s(sm + 4, Fc, bytes_p, stage_bar);
        if (bytes_s) bulk_g2s(summ, use_hash ? Hc : Sc, bytes_s, stage_bar);
      }
      // clear the summary buffers of iteration k+1 (last read at k-1)
      for (int i = vb * kThreads + threadIdx.x; i < a.SW; i += nvb * kThreads) {
        Sx[i] = 0u;
        if (kHash) Hx[i] = 0u;
      }
    }
#if SSB_LAZY_STAGE
    // The copies land while the warps take their first tasks (task entry,
    // unit, cs and visited loads, the first col loads): each warp waits at
    // its first probe. blk was cleared at the end of the previous iteration.
    ImgWait iw{stage_bar, stage_phase, false};
#else
    mbar_wait(stage_bar, stage_phase);
    __syncthreads();
    ImgWait iw{stage_bar, stage_phase, true};
#endif
    stage_phase ^= 1u;
#ifdef SSB_PHASES
    if (vb == 0 && threadIdx.x == 0) ph1 = globaltimer();
#endif
    if (vb == 0 && threadIdx.x == 0) { TRACE(0, k); TRACE(1, 1); }

    // per-warp counters of this iteration (a warp's share fits 32 bits)
    uint32_t c_front = 0, c_proc = 0, c_skip = 0, c_sub = 0, c_cols = 0, c_swept = 0;
    const Probe<kS> prb{sm + 4, Fc, img_words * 32, a.PW * 32 - ((a.PW * 32) >> kS)};

    // Active task list: iteration 1 walks every task; later iterations only the
    // tasks kept by the previous one. A task whose units were all skipped
    // (a.retire_once; else: in two consecutive iterations, so both frontier
    // buffers hold zeros for its chunks) is retired: SlimWork would skip it
    // forever, and its chunks are counted as skipped through gone_chunks.
    const ssb_tentry* list_in = ((k - 1) & 1) ? a.tlist1 : a.tlist0;
    ssb_tentry* list_out = (k & 1) ? a.tlist1 : a.tlist0;
    auto run_tasks = [&](auto early_tag, auto direct_tag, const auto& pr) {
    constexpr bool kEarly = decltype(early_tag)::value;
    constexpr bool kDirect = decltype(direct_tag)::value;
    // each warp's first task is its global warp id; the rest come from the
    // atomic counter (late iterations with few tasks then cost no atomics)
    const int32_t n_warps = int32_t(nvb) * (kThreads / 32);
    // Few active tasks (late iterations): each task is shared by D warps, the
    // d-th non-skipped unit going to sub-task d mod D, so a task's units are
    // not swept four per round by one warp while the others idle. Sub-task 0
    // does the task's bookkeeping (counters, retirement).
    int32_t dsh = 0;
    while (SSB_SPLIT_X > 0 && dsh < 3 && int64_t(n_in) * SSB_SPLIT_X << (dsh + 1) <= n_warps) ++dsh;
    const int32_t n_v = n_in << dsh;
    int32_t t_first = int32_t(vb) * (kThreads / 32) + int32_t(threadIdx.x >> 5);
    // Kept tasks are buffered one per lane and appended to list_out with one
    // atomic per 32 (a per-task append on one counter stalled every task on
    // its round trip: 13% of k = 4-5's stall samples at S26). Only in the
    // early-exit iterations: buffering groups the list by warp, and the
    // sparse iterations' lists must keep the heavy (hub) tasks first for the
    // dense sweep that follows (A/B: buffering there slowed S22 k = 3 by 20%).
    constexpr bool kBuf = SSB_KEEP_BUF && kEarly;
    ssb_tentry keep_t = 0;
    int32_t keep_n = 0;  // warp-uniform
    auto flush_kept = [&]() {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&a.task_out[rec], uint32_t(keep_n));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (lane < keep_n) list_out[base + lane] = keep_t;
      keep_n = 0;
    };
    // early-exit iterations grab kGrab tasks per atomic (their tasks are
    // mostly skip-only walks, where the counter's round trip dominated)
    constexpr int32_t kGrab = kEarly ? SSB_GRAB : 1;
    int32_t t_pend = 0, n_pend = 0;  // warp-uniform: grabbed, not yet started
    for (;;) {
      int32_t t = t_first;
      if (SSB_LAST_GRAB_SKIP && t < 0 && n_v <= n_warps) {  // every task was some warp's first: nothing to grab
        if (kBuf && keep_n) flush_kept();
        break;
      }
      if (t < 0) {
        if (n_pend == 0) {
          if (lane == 0) t_pend = int32_t(atomicAdd(&a.task_ctr[rec], uint32_t(kGrab))) + n_warps;
          t_pend = __shfl_sync(0xffffffffu, t_pend, 0);
          n_pend = kGrab;
        }
        t = t_pend++;
        --n_pend;
      }
      t_first = -1;
      if (t >= n_v) {
        if (kBuf && keep_n) flush_kept();
        break;
      }
      const int32_t sub = t & ((1 << dsh) - 1);
      t >>= dsh;
#if SSB_TLIST64
      int32_t ub, ue;
      if (k > 1) {
        const int64_t e = list_in[t];
        ub = int32_t(e);
        ue = ub + int32_t(e >> 32);
      } else {
        ub = a.task_begin[t];
        ue = a.task_begin[t + 1];
      }
      const ssb_tentry t_entry = int64_t(uint32_t(ub)) | (int64_t(ue - ub) << 32);
      const int32_t t_skip = ub;  // tskip index
#else
      if (k > 1) t = list_in[t];
      const int32_t ub = a.task_begin[t], ue = a.task_begin[t + 1];
      const ssb_tentry t_entry = t;
      const int32_t t_skip = t;
#endif

      // window: lane l owns unit ub + l
      const int32_t u = ub + lane;
      const bool has = u < ue;
      ssb_unit U = {0, 0, 0, -1};
      uint32_t vis = 0, realm = 0;
      int64_t ubase = 0;  // the unit's first cell in col (loaded once per task)
      bool skip = false;
      // A shared task (dsh > 0) is walked by 2^dsh warps at once; sub-task d
      // owns the units in lanes l with l mod 2^dsh == d. Ownership must not
      // depend on visited: a sibling may finalise a chunk (and rewrite its
      // visited word) before this warp reads it. Only the owner reads
      // visited for its decisions — it does so before its own unit can
      // arrive, so it always sees the value the iteration started with.
      const bool mine = dsh == 0 || (lane & ((1 << dsh) - 1)) == sub;
      if (has) {
        U = a.units[u];
        ubase = a.cs[U.chunk] + int64_t(U.col_begin) * 32;
        vis = a.visited[U.chunk];
        realm = U.chunk == a.n_chunks - 1 ? a.last_real : 0xffffffffu;
        skip = a.slimwork && vis == realm;  // should_skip_chunk
        if (U.col_begin == 0 && mine) {
          if (skip) {
            ++c_skip;
            Fn[U.chunk] = 0u;
          } else {
            const int32_t len = U.split < 0 ? U.col_len : a.cl[U.chunk];
            ++c_proc;
            c_cols += uint32_t(len);
            if (a.L > 0 && len > 0) c_sub += uint32_t((len + a.L - 1) / a.L);
          }
        }
      }
      const uint32_t open_all = __ballot_sync(0xffffffffu, has && !skip);
      if (!mine) skip = true;
      // every lane prefetches the head (in sweep order) of its unit into L2
      if (kPfHeadSteps > 0 && has && !skip && U.col_len > 0) {
        const int32_t hc = min(U.col_len, 4 * kPfHeadSteps);  // columns
        const int32_t first = (kSelMax && kEarly) ? U.col_len - hc : 0;
        prefetch_l2(a.col + a.cs[U.chunk] + int64_t(U.col_begin + first) * 32, uint32_t(hc) * 128u);
      }
#ifndef SSB_PF_SHORT
#define SSB_PF_SHORT 0
#endif
      // SSB_PF_SHORT: prefetch the whole columns of short units into L2 when
      // the task starts, so later group rounds hit L2 (paid off with 16-column
      // short units; with 32 it over-fetches: A/B S26 Kronecker +0.3%, ER +2%
      // without it)
      if (SSB_PF_SHORT && has && !skip && U.col_len > 0 && U.col_len < kWarpUnitCols)
        prefetch_l2(a.col + ubase, uint32_t(U.col_len) * 128u);
      // Long units (≥ kWarpUnitCols columns) are swept by the whole warp as one
      // contiguous 128-bit stream; short ones four at a time, one per group.
      const bool is_long = has && !skip && U.col_len >= kWarpUnitCols;
      uint32_t longs = __ballot_sync(0xffffffffu, is_long);
      uint32_t active = __ballot_sync(0xffffffffu, has && !skip && !is_long);
      {
        // Retirement needs every unit's skip state, which only the unit's
        // owner reads reliably: shared tasks (few active tasks, late
        // iterations) are never retired; they mark themselves "not skipped".
        const bool all_skipped = dsh == 0 && open_all == 0u;
        const uint32_t firsts = __ballot_sync(0xffffffffu, has && U.col_begin == 0);
        if (!kBuf) {
          if (lane == 0 && sub == 0) {
            if (a.slimwork && all_skipped && (a.retire_once || a.tskip[t_skip])) {
              atomicAdd(&a.gone_chunks[rec], (unsigned long long)__popc(firsts));
            } else {
              list_out[atomicAdd(&a.task_out[rec], 1u)] = t_entry;
              a.tskip[t_skip] = all_skipped;
            }
          }
        } else if (sub == 0) {
          const bool retire = a.slimwork && all_skipped &&
                              (a.retire_once ||
                               __shfl_sync(0xffffffffu, lane == 0 ? a.tskip[t_skip] : 0, 0));
          if (retire) {
            if (lane == 0) atomicAdd(&a.gone_chunks[rec], (unsigned long long)__popc(firsts));
          } else {
            if (lane == 0) a.tskip[t_skip] = all_skipped;
            if (lane == keep_n) keep_t = t_entry;
            if (++keep_n == 32) flush_kept();
          }
        }
      }

      while (longs) {
        const int32_t sl = __ffs(longs) - 1;
        longs &= longs - 1;
#ifndef SSB_PF_NEXT_LONG
#define SSB_PF_NEXT_LONG 16  // columns of the next long unit prefetched (A/B: +0.2-0.6%)
#endif
        if (SSB_PF_NEXT_LONG > 0 && longs) {
          // head (in sweep order) of the next long unit goes to L2 now
          const int32_t nx = __ffs(longs) - 1;
          const int32_t nl = __shfl_sync(0xffffffffu, U.col_len, nx);
          const int64_t nb = __shfl_sync(0xffffffffu, ubase, nx);
          const int32_t hc = min(nl, SSB_PF_NEXT_LONG);
          const int32_t first = (kSelMax && kEarly) ? nl - hc : 0;
          if (lane == 0) prefetch_l2(a.col + nb + int64_t(first) * 32, uint32_t(hc) * 128u);
        }
        const int32_t chunk = __shfl_sync(0xffffffffu, U.chunk, sl);
        const int32_t len = __shfl_sync(0xffffffffu, U.col_len, sl);
        const int32_t split = __shfl_sync(0xffffffffu, U.split, sl);
        const uint32_t uvis = __shfl_sync(0xffffffffu, vis, sl);
        const uint32_t ureal = __shfl_sync(0xffffffffu, realm, sl);
        // int4 i of the unit = column i/8, rows 4(i%8)..+3; lane l takes
        // i = 32s + l, so lg (rows) is fixed per lane and grp picks the column
        // within each 4-column step. Out-of-range indices re-read the lane's
        // own rows of the last column (idempotent).
        const int4* base = reinterpret_cast<const int4*>(a.col + __shfl_sync(0xffffffffu, ubase, sl));
        // early-exit sweeps start with the rows already settled (visited or
        // padding) marked decided: their probes are skipped
        uint32_t hit = kEarly ? ((uvis | ~ureal) >> (4 * lg)) & 0xfu : 0u;
        int32_t best[4] = {-1, -1, -1, -1};
        const int32_t sw = sweep_long<kSelMax, kEarly, kDirect>(base, len, lane, lg, pr, pol, hit, best, iw);
        if (lane == 0) c_swept += uint32_t(sw);
        uint32_t m = hit << (4 * lg);
        m |= __shfl_xor_sync(0xffffffffu, m, 1);
        m |= __shfl_xor_sync(0xffffffffu, m, 2);
        m |= __shfl_xor_sync(0xffffffffu, m, 4);
        finish_unit<kSelMax, kEarly, kHash>(a, k, Fn, Sn, grp == 0, chunk, split, uvis, ureal, m, best, grp, lg,
                             gmask, c_front);
      }

      bool first_round = true;
      while (active) {
        // the next (up to) four active units, one per 8-lane group
        int32_t src = -1;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int32_t f = active ? __ffs(active) - 1 : -1;
          if (g == grp) src = f;
          if (active) active &= active - 1;
        }
        const int32_t sl = src < 0 ? 0 : src;
#ifndef SSB_PF_NEXT
#define SSB_PF_NEXT 1  // rounds ahead whose units are prefetched (A/B S26 ER: 0 -> 1 +7%)
#endif
        if (SSB_PF_NEXT > 0) {
          // this group's unit of round +SSB_PF_NEXT (and, in the first round,
          // of the rounds before it) goes to L2 while this round runs
          uint32_t rest = active;
#pragma unroll
          for (int d = 1; d <= SSB_PF_NEXT; ++d) {
            int32_t nsrc = -1;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const int32_t f = rest ? __ffs(rest) - 1 : -1;
              if (g == grp) nsrc = f;
              if (rest) rest &= rest - 1;
            }
            if (d == SSB_PF_NEXT || first_round) {
              const int32_t nl = __shfl_sync(0xffffffffu, U.col_len, nsrc < 0 ? 0 : nsrc);
              const int64_t nb = __shfl_sync(0xffffffffu, ubase, nsrc < 0 ? 0 : nsrc);
              if (lg == 0 && nsrc >= 0 && nl > 0) prefetch_l2(a.col + nb, uint32_t(nl) * 128u);
            }
          }
          first_round = false;
        }
        const int32_t chunk = __shfl_sync(0xffffffffu, U.chunk, sl);
        const int32_t ulen = __shfl_sync(0xffffffffu, U.col_len, sl);  // all lanes shuffle
        const int32_t len = src < 0 ? 0 : ulen;
        const int32_t split = __shfl_sync(0xffffffffu, U.split, sl);
        const uint32_t uvis = __shfl_sync(0xffffffffu, vis, sl);
        const uint32_t ureal = __shfl_sync(0xffffffffu, realm, sl);
        int32_t maxlen = len;
        maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, 8));
        maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, 16));

        // Column j of the unit is int4 p[8j] (lane lg: rows 4lg..4lg+3). Groups
        // shorter than maxlen re-read their last column (idempotent for both
        // the "any" and the "last hit" reduction); groups without a unit read
        // a padding column. Loads run 4 columns ahead of the probes.
        const int64_t gbase = __shfl_sync(0xffffffffu, ubase, sl);  // all lanes shuffle
        const int4* p = len > 0 ? reinterpret_cast<const int4*>(a.col + gbase) + lg
                                : reinterpret_cast<const int4*>(g_pad_column) + (lg & 7);
        const int32_t jlast = len > 0 ? len - 1 : 0;
        const int64_t stride = len > 0 ? 8 : 0;
        // (a group without a unit counts as decided)
        uint32_t hit = kEarly ? (src < 0 ? 0xfu : ((uvis | ~ureal) >> (4 * lg)) & 0xfu) : 0u;
        int32_t best[4] = {-1, -1, -1, -1};
        const int32_t ran = sweep_group<kSelMax, kEarly, kDirect>(p, jlast, stride, maxlen, pr, pol, hit, best, iw);
        if (lg == 0) c_swept += uint32_t(min(len, ran));
        // 32-bit row mask of the unit (rows 4*lg+q)
        uint32_t m = hit << (4 * lg);
        m |= __shfl_xor_sync(0xffffffffu, m, 1);
        m |= __shfl_xor_sync(0xffffffffu, m, 2);
        m |= __shfl_xor_sync(0xffffffffu, m, 4);

        finish_unit<kSelMax, kEarly, kHash>(a, k, Fn, Sn, src >= 0, chunk, split, uvis, ureal, m, best, grp, lg,
                             gmask, c_front);
      }
    }
    };  // run_tasks
    if (direct) {
      run_tasks(std::true_type{}, std::true_type{}, prb);
    } else if (use_hash) {
      if constexpr (kHash) {
        const Probe<kS, true> prh{sm + 4, Fc, img_words * 32, int32_t(a.hash_arg)};
        run_tasks(std::true_type{}, std::false_type{}, prh);  // (use_hash implies dense)
      }
    } else if (dense) {
      run_tasks(std::true_type{}, std::false_type{}, prb);
    } else {
      run_tasks(std::false_type{}, std::false_type{}, prb);
    }
    // this (sparse) iteration built the hashed summary (recomputed here from
    // loop state rather than kept live through the sweep)
    hash_prev = kHash && !(front_in > a.dense_thr);
    // every warp has seen this phase complete before thread 0 re-arms the
    // barrier for the next iteration (warps without a sweep wait here)
    iw();

    // -- iteration counters: warp -> block -> grid --------------------------
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      c_front += __shfl_xor_sync(0xffffffffu, c_front, o);
      c_proc += __shfl_xor_sync(0xffffffffu, c_proc, o);
      c_skip += __shfl_xor_sync(0xffffffffu, c_skip, o);
      c_sub += __shfl_xor_sync(0xffffffffu, c_sub, o);
      c_cols += __shfl_xor_sync(0xffffffffu, c_cols, o);
      c_swept += __shfl_xor_sync(0xffffffffu, c_swept, o);
    }
    if (lane == 0) {
      atomicAdd(&blk[0], (unsigned long long)c_front);
      atomicAdd(&blk[1], (unsigned long long)c_proc);
      atomicAdd(&blk[2], (unsigned long long)c_skip);
      atomicAdd(&blk[3], (unsigned long long)c_sub);
      atomicAdd(&blk[4], (unsigned long long)c_cols);
      atomicAdd(&blk[5], (unsigned long long)c_swept);
    }
    __syncthreads();
    if (threadIdx.x < 6) {
      atomicAdd(reinterpret_cast<unsigned long long*>(
                    &a.stats[rec * kStatW + (threadIdx.x < 5 ? threadIdx.x : 6)]),
                blk[threadIdx.x]);
      blk[threadIdx.x] = 0ull;  // the next adds come after grid.sync
    }
    if (threadIdx.x == 0 && a.trace) atomicAdd(&a.trace[2], 1);
#ifdef SSB_PHASES
    if (vb == 0 && threadIdx.x == 0) ph2 = globaltimer();
#endif
    grid.sync();
#ifdef SSB_PHASES
    if (vb == 0 && threadIdx.x == 0) {
      const uint64_t ph3 = globaltimer();
      g_phase[0] += ph1 - ph0;
      g_phase[1] += ph2 - ph1;
      g_phase[2] += ph3 - ph2;
      g_phase[3] += 1;
    }
#endif
    if (vb == 0 && threadIdx.x == 0) TRACE(1, 4);
#if SSB_BCAST
    // the iteration's totals are read once per CTA and broadcast: uniform
    // volatile loads from every warp of the grid would queue 4736 requests
    // per word at one L2 slice
    if (threadIdx.x == 0) {
      bcast[0] = *reinterpret_cast<volatile int64_t*>(&a.stats[rec * kStatW]);
      bcast[1] = int64_t(*reinterpret_cast<volatile uint32_t*>(&a.task_out[rec]));
      bcast[2] = int64_t(*reinterpret_cast<volatile unsigned long long*>(&a.gone_chunks[rec]));
    }
    __syncthreads();
    int64_t front = bcast[0];
#else
    int64_t front = *reinterpret_cast<volatile int64_t*>(&a.stats[rec * kStatW]);
#endif
    if (kP2P) {
      if (vb == 0 && threadIdx.x == 0) TRACE(1, 5);
      front = p2p_exchange(x, k, Fn, Sn, front, x.gen_base + 2 + uint32_t(rec), vb, nvb);
      if (vb == 0 && threadIdx.x == 0) { TRACE(1, 6); TRACE(3, int(front)); }
      if (vb == 0 && threadIdx.x == 0) a.stats[rec * kStatW + 7] = front;  // global |newly|
    }
    front_in = front;
#if SSB_BCAST
    n_in = int32_t(bcast[1]);
#else
    n_in = int32_t(*reinterpret_cast<volatile uint32_t*>(&a.task_out[rec]));
#endif
    if (vb == 0 && threadIdx.x == 0) {
      const uint64_t t = globaltimer();
      a.stats[rec * kStatW + 5] = int64_t(t - t_prev);
      a.stats[rec * kStatW + 2] += int64_t(gone);  // retired tasks' chunks: skipped
      t_prev = t;
    }
#if SSB_BCAST
    gone += static_cast<unsigned long long>(bcast[2]);
#else
    gone += *reinterpret_cast<volatile unsigned long long*>(&a.gone_chunks[rec]);
#endif
    if (front == 0) break;  // is_converged: no row newly reached
  }
  if (a.rec_host && vb == 0) {  // every CTA's counters landed before the last grid.sync
    __syncthreads();
    const int32_t nw = min(a.k_end - a.k_begin, int32_t(kRecFirst)) * kStatW;
    for (int32_t i = threadIdx.x; i < nw; i += blockDim.x) a.rec_host[i] = __ldcg(a.stats + i);
  }
  // every CTA read the carry at launch start, before the first grid.sync
  if (a.carry && vb == 0 && threadIdx.x == 0) {
    a.carry[0] = front_in;
    a.carry[1] = n_in;
    a.carry[2] = static_cast<int64_t>(gone);
  }
}

struct ResetArgs {
  uint4* reg[5];      // visited, F0, S0..S2, stats, control words
  int64_t n16[5];
  uint8_t* tskip;
  int64_t n_tasks;
  uint32_t* visited;
  uint32_t* F0;
  uint32_t* S0;       // null without a summary
  int32_t root_pos, root_code, PW, gshift;
  int32_t* level;
  int32_t* parent;
  int32_t active;     // bfs32_kernel: reset before the first iteration
};

// init_state (semiring.cpp:56-88) in 1-bit form over the whole grid: the
// state regions zeroed, the root's visited / frontier / summary bits set, its
// level and parent seeded.
__device__ __forceinline__ void reset_body(const ResetArgs& r) {
  const int32_t rw = r.root_pos >> 5;
  const uint32_t rbit = 1u << (r.root_pos & 31);
  const int32_t sgi = r.S0 && rw >= r.PW ? (rw - r.PW) >> r.gshift : -1;
  for (int q = 0; q < 5; ++q) {
    uint4* p = r.reg[q];
    GRID_STRIDE(i, r.n16[q]) {
      uint4 z = make_uint4(0u, 0u, 0u, 0u);
      uint32_t* zw = reinterpret_cast<uint32_t*>(&z);
      uint32_t* base = reinterpret_cast<uint32_t*>(p + i);
      for (int t = 0; t < 4; ++t) {
        const uint32_t* w = base + t;
        if (w == r.visited + rw || w == r.F0 + rw) zw[t] = rbit;
        if (sgi >= 0 && w == r.S0 + (sgi >> 5)) zw[t] = 1u << (sgi & 31);
      }
      p[i] = z;
    }
  }
  GRID_STRIDE(i, r.n_tasks) r.tskip[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    r.level[r.root_pos] = 0;
    r.parent[r.root_pos] = r.root_code;
  }
}

__global__ void reset32_kernel(const ResetArgs r) { reset_body(r); }

// One single-GPU BFS launch; the first launch of a BFS also does init_state
// (one launch less per BFS than a separate reset kernel).
template <bool kSelMax, int kS, bool kHash>
__global__ void __launch_bounds__(kThreads, 1) bfs32_kernel(const Args32 a, const ResetArgs r) {
  if (r.active) {
    reset_body(r);
    cg::this_grid().sync();
  }
  bfs32_body<kSelMax, kS, false, kHash>(a, P2PArgs{}, int(blockIdx.x), int(gridDim.x));
}

// Chunk-range shard of a multi-GPU BFS with the frontier exchange fused in:
// one launch per rank (bfs32x_kernel), or all ranks of an emulated group in
// one cooperative launch (bfs32p_kernel, rank = blockIdx.x / nvb).
template <bool kSelMax, int kS>
__global__ void __launch_bounds__(kThreads, 1) bfs32x_kernel(const Args32 a, const P2PArgs x) {
  bfs32_body<kSelMax, kS, true, false>(a, x, int(blockIdx.x), int(gridDim.x));
}
template <bool kSelMax, int kS>
__global__ void __launch_bounds__(kThreads, 1) bfs32p_kernel(const __grid_constant__ GroupArgs ga) {
  const int vr = int(blockIdx.x) / ga.nvb;
  bfs32_body<kSelMax, kS, true, false>(ga.a[vr], ga.x[vr], int(blockIdx.x) - vr * ga.nvb, ga.nvb);
}

// ---- generic engine (any C) ------------------------------------------------

struct GenUnit {
  int32_t chunk, col_begin, col_len;
};
constexpr int32_t kGenUnitCols = 256;

// The C != 32 engine (the reference's small-C parity configurations, e.g.
// config 1's C = 8): byte-per-row state, one cooperative launch for the whole
// BFS, three grid-wide phases per iteration:
//   A  should_skip_chunk (semiring.cpp:130-150) per chunk + the counters;
//   B  one warp per work unit (a chunk's column range of <= kGenUnitCols
//      columns, so hub chunks are split across warps); lane l (and l + 32,
//      ... for C > 32) owns row l of the chunk and folds its largest
//      frontier-neighbour position into hitbest[row] with atomicMax — the
//      sel-max max (bfs.cpp:94-101), any hit for the other semirings;
//   C  post_process_rows (semiring.cpp:90-124) per row, the next frontier,
//      |newly|; hitbest is reset for the next iteration.
// Convergence (semiring.cpp:152-157) and the per-iteration records stay on
// the device.
struct ArgsG {
  const int32_t* col;
  const int64_t* cs;
  const int32_t* cl;
  int64_t C, n, n_chunks;
  uint8_t* vis;    // n_padded
  uint8_t* f0;     // n_padded: frontier of even iterations' input
  uint8_t* f1;     // n_padded
  uint8_t* skip;   // n_chunks
  int32_t* level;
  int32_t* parent;
  const GenUnit* units;
  int64_t n_units;
  int32_t* hitbest;          // n_padded, -1 between iterations
  unsigned long long* stats; // [kItersPerLaunch][kStatW]
  int32_t L, slimwork, root_code, selmax;
  int32_t k_begin, k_end;
};

__global__ void __launch_bounds__(1024, 1) genc_kernel(const ArgsG a) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  const int64_t np = a.n_chunks * a.C;
  uint64_t t_prev = 0;
  if (tid == 0) t_prev = globaltimer();
  for (int32_t k = a.k_begin; k < a.k_end; ++k) {
    unsigned long long* st = a.stats + int64_t(k - a.k_begin) * kStatW;
    const uint8_t* fcur = (k & 1) ? a.f0 : a.f1;  // F_{k-1}: k = 1 reads f0 (the root)
    uint8_t* fnext = (k & 1) ? a.f1 : a.f0;
    // A: SlimWork skip flags + processed / skipped / subchunk / column counters
    {
      unsigned long long proc = 0, skp = 0, sub = 0, cols = 0;
      for (int64_t i = tid; i < a.n_chunks; i += nth) {
        bool sk = false;
        if (a.slimwork) {
          sk = true;
          const int64_t r1 = min((i + 1) * a.C, a.n);
          for (int64_t r = i * a.C; r < r1 && sk; ++r) sk = a.vis[r] != 0;
        }
        a.skip[i] = sk;
        if (sk) {
          ++skp;
        } else {
          ++proc;
          cols += uint32_t(a.cl[i]);
          if (a.L > 0 && a.cl[i] > 0) sub += uint32_t((a.cl[i] + a.L - 1) / a.L);
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        proc += __shfl_xor_sync(0xffffffffu, proc, o);
        skp += __shfl_xor_sync(0xffffffffu, skp, o);
        sub += __shfl_xor_sync(0xffffffffu, sub, o);
        cols += __shfl_xor_sync(0xffffffffu, cols, o);
      }
      if (lane == 0) {
        if (proc) atomicAdd(&st[1], proc);
        if (skp) atomicAdd(&st[2], skp);
        if (sub) atomicAdd(&st[3], sub);
        if (cols) atomicAdd(&st[4], cols);
      }
    }
    grid.sync();
    // B: the sweep, one warp per unit. For C <= 32 the warp holds G = 32 / C
    // column groups: lane l takes row l % C and columns l / C, l / C + G, ...
    // (four in flight), so a C = 8 unit keeps every lane busy; each lane
    // folds its own largest hit (the row's max over groups by atomicMax).
    {
      const int64_t C = a.C;
      const int32_t G = C <= 32 ? int32_t(32 / C) : 1;
      const int32_t grp = C <= 32 ? int32_t(lane / C) : 0;
      for (int64_t w = tid >> 5; w < a.n_units; w += nth >> 5) {
        const GenUnit u = a.units[w];
        if (a.skip[u.chunk]) continue;
        const int32_t* base = a.col + a.cs[u.chunk] + int64_t(u.col_begin) * C;
        if (grp >= G) continue;  // lanes beyond G·C (C not a divisor of 32)
        for (int64_t l = C <= 32 ? lane % C : lane; l < C; l += 32) {
          int32_t best = -1;
          int32_t j = grp;
          for (; j + 3 * G < u.col_len; j += 4 * G) {
            int32_t c[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) c[q] = base[int64_t(j + q * G) * C + l];
            uint8_t f[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) f[q] = c[q] >= 0 ? fcur[c[q]] : uint8_t(0);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (f[q]) best = max(best, c[q]);
          }
          for (; j < u.col_len; j += G) {
            const int32_t c = base[int64_t(j) * C + l];
            if (c >= 0 && fcur[c]) best = max(best, c);  // columns ascend within a row
          }
          if (best >= 0) atomicMax(&a.hitbest[int64_t(u.chunk) * C + l], best);
        }
      }
    }
    grid.sync();
    // C: post-process, next frontier, |newly|
    {
      unsigned long long front = 0;
      for (int64_t r = tid; r < np; r += nth) {
        const int32_t best = a.hitbest[r];
        uint8_t nw = 0;
        if (best >= 0) {
          a.hitbest[r] = -1;
          if (r < a.n && !a.vis[r]) {
            nw = 1;
            a.vis[r] = 1;
            a.level[r] = k;
            if (a.selmax) a.parent[r] = k == 1 ? a.root_code : best;
            ++front;
          }
        }
        fnext[r] = nw;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) front += __shfl_xor_sync(0xffffffffu, front, o);
      if (lane == 0 && front) atomicAdd(&st[0], front);
    }
    grid.sync();
    if (tid == 0) {
      const uint64_t t = globaltimer();
      st[5] = t - t_prev;
      t_prev = t;
    }
    if (*reinterpret_cast<volatile unsigned long long*>(&st[0]) == 0) break;  // is_converged
  }
}

// ---- shared init / epilogue kernels ---------------------------------------

// init_state for the C=32 engine in ONE launch (one host call instead of five):
// zero the 16-byte-aligned regions (visited+F0, the summaries, the stats and
// control words), the per-task skip flags, and set the root's bits; the
// thread that zeroes the root's words writes them with the root bit instead.
__global__ void bytes_to_bits_kernel(const uint8_t* __restrict__ vis, int64_t n_padded,
                                     uint32_t* __restrict__ bits) {
  GRID_STRIDE(w, (n_padded + 31) / 32) {
    uint32_t v = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t r = w * 32 + b;
      if (r < n_padded && vis[r]) v |= 1u << b;
    }
    bits[w] = v;
  }
}

// permute_out (repr.cpp:247-253) + selmax_parents (bfs.cpp:94-101): results in
// original ids; sel-max positions decode through perm exactly like the
// reference, including its root encoding when compat is on.
// Summary of a full frontier bitmap (after a shard exchange): bit t of the
// summary <-> frontier words [PW + 8t, PW + 8t + 8) hold a set bit.
// |F| of a full frontier bitmap (the exchanged words of every rank): the global
// newly-reached count is_converged (semiring.cpp:152-157) needs, on the device.
// Only chunks with cells count: a newly reached row has a neighbour, and the
// words of cell-less chunks (isolated rows, never swept) are not maintained.
__global__ void front_count_kernel(const uint32_t* __restrict__ F, const int32_t* __restrict__ cl, int64_t nw,
                                   int64_t* __restrict__ out) {
  unsigned long long c = 0;
  GRID_STRIDE(w, nw) c += cl[w] > 0 ? __popc(F[w]) : 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(reinterpret_cast<unsigned long long*>(out), c);
}

__global__ void summary_from_words_kernel(const uint32_t* __restrict__ F, int64_t PW, int64_t NW,
                                          uint32_t* __restrict__ S, int64_t SW, int gshift) {
  GRID_STRIDE(sw, SW) {
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t w0 = PW + ((sw * 32 + b) << gshift);
      uint32_t any = 0;
      for (int64_t w = w0; w < w0 + (int64_t{1} << gshift) && w < NW; ++w) any |= F[w];
      bits |= uint32_t(any != 0) << b;
    }
    S[sw] = bits;
  }
}

// Gather form (one thread per ORIGINAL id, so the int64 outputs are written
// coalesced — straight into pinned host memory over PCIe when the caller's
// buffers allow it).
__global__ void unpermute_kernel(const uint32_t* __restrict__ visited,
                                 const int32_t* __restrict__ level,
                                 const int32_t* __restrict__ parent,
                                 const int32_t* __restrict__ perm,
                                 const int32_t* __restrict__ inv_perm, int64_t n,
                                 int selmax_parents, int64_t* __restrict__ dist,
                                 int64_t* __restrict__ par, const uint8_t* __restrict__ owned) {
  GRID_STRIDE(o, n) {
    const int32_t p = inv_perm[o];
    if (owned && !owned[p >> 5]) continue;  // another shard's row (C = 32: chunk = p / 32)
    const bool reached = (visited[p >> 5] >> (p & 31)) & 1u;
    if (dist) dist[o] = reached ? int64_t(level[p]) : INT64_MAX;
    if (selmax_parents) par[o] = reached ? int64_t(perm[parent[p]]) : -1;
  }
}

// dp_transform (semiring.cpp:159-187) on the layout: the smallest ORIGINAL id
// among the row's neighbours one level closer; root self-parented.
template <class T>
__global__ void dp_parent_kernel(const int32_t* __restrict__ col, const int64_t* __restrict__ cs,
                                 const int32_t* __restrict__ cl, int64_t C,
                                 const uint32_t* __restrict__ visited,
                                 const int32_t* __restrict__ level,
                                 const int32_t* __restrict__ perm,
                                 const int32_t* __restrict__ inv_perm, int64_t n,
                                 T* __restrict__ par, int* __restrict__ bad,
                                 const uint8_t* __restrict__ owned, int64_t o0 = 0) {
  GRID_STRIDE(i, n - o0) {
    const int64_t o = o0 + i;
    const int32_t p = inv_perm[o];
    if (owned && !owned[p / C]) continue;  // another shard's row
    if (!((visited[p >> 5] >> (p & 31)) & 1u)) {
      par[o] = -1;
      continue;
    }
    const int32_t lv = level[p];
    if (lv == 0) {
      par[o] = int64_t(o);
      continue;
    }
    const int64_t ch = p / C, lane = p % C;
    const int32_t* cells = col + cs[ch] + lane;
    int32_t bestp = INT_MAX;
    for (int32_t j = 0; j < cl[ch]; ++j) {
      const int32_t c = cells[int64_t(j) * C];
      if (c < 0) break;
      if (((visited[c >> 5] >> (c & 31)) & 1u) && level[c] == lv - 1) bestp = min(bestp, perm[c]);
    }
    if (bestp == INT_MAX) atomicOr(bad, 1);
    par[o] = bestp == INT_MAX ? T(-1) : T(bestp);
  }
}

// The result in original ids as the PCIe wire format of the fetch: uint8
// levels (255 = unreached) and int32 sel-max parents (-1 = unreached);
// hostio.cpp widens them into the caller's int64 arrays.
__global__ void pack_wire_kernel(const uint32_t* __restrict__ visited,
                                 const int32_t* __restrict__ level,
                                 const int32_t* __restrict__ parent,
                                 const int32_t* __restrict__ perm,
                                 const int32_t* __restrict__ inv_perm, int64_t o0, int64_t o1,
                                 uint8_t* __restrict__ lev8, int32_t* __restrict__ par32) {
  GRID_STRIDE(i, o1 - o0) {
    const int64_t o = o0 + i;
    const int32_t p = inv_perm[o];
    const bool reached = (visited[p >> 5] >> (p & 31)) & 1u;
    if (lev8) lev8[o] = reached ? uint8_t(level[p]) : uint8_t(255);
    if (par32) par32[o] = reached ? perm[parent[p]] : -1;
  }
}

// Packed wire (sel-max, dist and parents wanted): one 32-bit word per vertex,
// level << bits | parent's original id, all ones where unreached.
__global__ void pack_wire32_kernel(const uint32_t* __restrict__ visited, const int32_t* __restrict__ level,
                                   const int32_t* __restrict__ parent, const int32_t* __restrict__ perm,
                                   const int32_t* __restrict__ inv_perm, int64_t o0, int64_t o1, int bits,
                                   uint32_t* __restrict__ out) {
  GRID_STRIDE(i, o1 - o0) {
    const int64_t o = o0 + i;
    const int32_t p = inv_perm[o];
    const bool reached = (visited[p >> 5] >> (p & 31)) & 1u;
    out[o] = reached ? (uint32_t(level[p]) << bits) | uint32_t(perm[parent[p]]) : 0xffffffffu;
  }
}

__global__ void reached_degree_kernel(const uint32_t* __restrict__ visited,
                                      const int32_t* __restrict__ deg, int64_t n,
                                      unsigned long long* __restrict__ out) {
  unsigned long long s = 0;
  GRID_STRIDE(p, n) {
    if ((visited[p >> 5] >> (p & 31)) & 1u) s += uint32_t(deg[p]);
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// ---- host side ---------------------------------------------------------------

// Shared memory for the frontier image (KB). Not the maximum: the rest of the
// SM's 256 KB goes to L1, which the frontier's exact lookups and the task
// metadata use (A/B at S26: 200 -> 160 KB gives Kronecker +2.5%, ER +26%).
constexpr int kSmemKB = 160;

struct Geometry {
  int64_t NW = 0;  // bitmap words
  int32_t PW = 0, SW = 0, gshift = 0;
  int32_t S = 8;  // log2 vertices per summary bit (Probe<kS>)
  size_t smem = 0;
};

// Summary granularities the kernel is instantiated for.
using Bfs32Fn = void (*)(const Args32, const ResetArgs);
// hashed: the S = 8 engine that also builds / probes the hashed summary (a
// separate instantiation, so graphs without it run the leaner kernel)
Bfs32Fn bfs32_fn(bool sel, int S, bool hashed) {
  if (S == 6) return sel ? bfs32_kernel<true, 6, false> : bfs32_kernel<false, 6, false>;
  if (hashed) return sel ? bfs32_kernel<true, 8, true> : bfs32_kernel<false, 8, true>;
  return sel ? bfs32_kernel<true, 8, false> : bfs32_kernel<false, 8, false>;
}

Geometry geometry32_for(const ssb_graph& g, int S) {
  Geometry G;
  G.NW = (g.n_padded + 31) / 32;
  const int64_t budget_words = int64_t(env_int("SSB_SMEM_KB", kSmemKB)) * 1024 / 4 - 4;
  const int64_t nw4 = (G.NW + 3) & ~int64_t(3);
  G.S = S;
  G.gshift = S - 5;  // summary bit = 2^gshift frontier words
  if (nw4 <= budget_words) {
    G.PW = int32_t(nw4);
    G.SW = 0;
  } else {
    // summary over the whole id range (an upper bound for the tail), rest prefix
    const int64_t groups = (G.NW + (int64_t{1} << G.gshift) - 1) >> G.gshift;
    G.SW = int32_t(((groups + 31) / 32 + 3) / 4 * 4);
    // prefix: a multiple of one summary group (and of 4 words for uint4 staging)
    const int64_t align = std::max<int64_t>(4, int64_t{1} << G.gshift);
    G.PW = int32_t(std::max<int64_t>(0, budget_words - G.SW) / align * align);
  }
  G.smem = size_t(4 + G.PW + G.SW) * 4;  // + 4 zero words for padding cells
  return G;
}

// The prefix's share of the cells' targets: vertex v is the target of deg(v)
// cells and a chunk's rows have degree <= cl, so the cells of the first PW
// chunks estimate it (exactly the cells of those rows' chunks for σ = n).
double prefix_coverage(const ssb_graph& g, int64_t PW) {
  if (g.total_cells <= 0) return 1.0;
  int64_t c = 0;
  for (int64_t i = 0; i < std::min<int64_t>(PW, g.n_chunks); ++i) c += int64_t(g.cl_host[size_t(i)]) * 32;
  return double(c) / double(g.total_cells);
}

Geometry geometry32(const ssb_graph& g) {
  const int forced = env_int("SSB_SUMMARY_SHIFT", 0);
  if (forced == 6 || forced == 8) return geometry32_for(g, forced);
  Geometry G8 = geometry32_for(g, 8);
  // hub-heavy: the prefix catches most probes, keep it large; otherwise most
  // probes fall in the tail, where a finer summary saves exact lookups — if
  // that summary fits the budget (not at S28: 4x the S = 8 summary)
  if (G8.SW == 0 || prefix_coverage(g, G8.PW) >= 0.5) return G8;
  const Geometry G6 = geometry32_for(g, 6);
  const int64_t budget = int64_t(env_int("SSB_SMEM_KB", kSmemKB)) * 1024;
  return int64_t(G6.smem) <= budget ? G6 : G8;
}

// Work units + tasks for the C=32 engine. A unit is a SlimChunk segment of at
// most L columns (the whole chunk when L <= 0, as the reference's task list,
// bfs.cpp:122-138); a task groups up to 32 consecutive units whose cost stays
// under a budget, the grain of the dynamic scheduler.
// segs: the chunk segments this plan covers, [b0, e0, b1, e1, ...]
void build_plan32(ssb_graph& g, int64_t L, const std::vector<int64_t>& segs) {
  ssb_bfs_plan& P = g.plan;
  // Units are SlimChunk segments of at most Lu columns: the reference's L
  // (which alone defines the subchunks_processed counter, computed
  // analytically in the kernel) capped for balance — a unit must stay a
  // small share of one warp's work in a full sweep, or the last long unit of
  // an iteration idles the grid (S22: one 2048-column unit is ~0.2 ms on a
  // warp, longer than the whole iteration). L <= 0 (SlimChunk off) splits at
  // the cap alone.
  // one warp's share of a full sweep (columns); the range sum is host work,
  // cached with the range
  if (P.cap_segs != segs) {
    int64_t cols = 0;
    for (size_t q = 0; q + 1 < segs.size(); q += 2)
      for (int64_t i = segs[q]; i < segs[q + 1]; ++i) cols += g.cl_host[size_t(i)];
    const int64_t per_warp = cols / (int64_t(num_sms()) * (kThreads / 32));
    // unit cap: the largest power of two (64 .. 4096) not above the share
    // (A/B S22: 4096 113.8, 512 136.4, 128 131.6 GTEPS)
    int64_t c = 64;
    while (c * 2 <= per_warp && c < 4096) c *= 2;
    P.cap_auto = c;
    // task budget: the largest power of two (128 .. 8192) not above half the
    // share. Small graphs need fine tasks for the sweeps' tail balance, large
    // ones coarse tasks for cheap skip-only walks in the late iterations
    // (scripts/sweep_budget.sh, GTEPS at 128/256/512/1024/2048/4096/8192:
    // S22 145.8/148.4/136.0/119.5/-/-/-, S24 -/212.1/216.2/211.0/199.9/-/-,
    // S26 215.4/229.8/233.5/236.5/237.4/238.7/239.6, ER 2^26 512 51.6, 2048 53.2)
    int64_t b = 128;
    while (b * 2 <= per_warp / 2 && b < 8192) b *= 2;
    P.budget_auto = b;
    P.cap_segs = segs;
  }
  int64_t cap = env_int("SSB_UNIT_CAP", 0);
  if (cap <= 0) cap = P.cap_auto;
  const int64_t Lu = L > 0 ? std::min(L, cap) : cap;
  if (P.L == L && P.Lu == Lu && P.segs == segs && P.built) return;
  std::vector<ssb_unit> units;
  std::vector<int32_t> split_units;
  P.empty_chunks = 0;
  for (size_t q = 0; q + 1 < segs.size(); q += 2)
  for (int64_t i = segs[q]; i < segs[q + 1]; ++i) {
    const int64_t cl = g.cl_host[i];
    if (cl == 0) {
      // Chunks without cells (all rows isolated; 1.07M of 2.1M at S26) can
      // never reach a row: no unit, counted analytically (bfs_run).
      ++P.empty_chunks;
      continue;
    }
    if (cl <= Lu) {
      units.push_back({int32_t(i), 0, int32_t(cl), -1});
    } else {
      const int32_t sp = int32_t(split_units.size());
      const int64_t nseg = (cl + Lu - 1) / Lu;
      split_units.push_back(int32_t(nseg));
      for (int64_t s = 0; s < nseg; ++s)
        units.push_back({int32_t(i), int32_t(s * Lu), int32_t(std::min(Lu, cl - s * Lu)), sp});
    }
  }
  const int64_t budget = env_int("SSB_TASK_BUDGET", int(P.budget_auto));
  const int64_t overhead = env_int("SSB_UNIT_OVERHEAD", 4);
  // taper: on graphs with fine tasks (budget <= 512, S22) the last 10% of
  // the columns go in tasks of a quarter of the budget, so the sweeps' tails
  // drain faster (A/B over 64 roots: S22 0.433 -> 0.426 ms per BFS; S26, with
  // 4096-column tasks, gains nothing from it)
  const int taper_pct = env_int("SSB_TASK_TAPER", budget <= 512 ? 90 : 100);
  const int taper_div = std::max(1, env_int("SSB_TASK_TAPER_DIV", 4));
  int64_t total_cost = 0;
  for (const auto& un : units) total_cost += un.col_len + overhead;
  const int64_t taper_at = total_cost * taper_pct / 100;
  std::vector<int32_t> tb;
  tb.push_back(0);
  int64_t cost = 0, cnt = 0, cum = 0;
  for (size_t u = 0; u < units.size(); ++u) {
    cost += units[u].col_len + overhead;
    cum += units[u].col_len + overhead;
    ++cnt;
    const int64_t bgt = cum > taper_at ? std::max<int64_t>(32, budget / taper_div) : budget;
    if (cnt == kUnitsPerTask || cost >= bgt) {
      tb.push_back(int32_t(u + 1));
      cost = 0;
      cnt = 0;
    }
  }
  if (cnt) tb.push_back(int32_t(units.size()));
  if (units.size() >= size_t(INT32_MAX)) fail(SSB_EINVAL, "too many work units");
  cudaStream_t s = g.sc.s;
  P.L = L;
  P.Lu = Lu;
  P.segs = segs;
  P.built = true;
  P.n_units = int64_t(units.size());
  P.n_tasks = int64_t(tb.size()) - 1;
  P.n_split = int64_t(split_units.size());
  P.units.alloc(units.size());
  P.task_begin.alloc(tb.size());
  P.split_units.alloc(std::max<size_t>(split_units.size(), 1));
  P.split_hit.alloc(std::max<size_t>(split_units.size(), 1));
  P.split_best.alloc(std::max<size_t>(split_units.size(), 1) * 32);
  P.split_count.alloc(std::max<size_t>(split_units.size(), 1));
  P.tlist.alloc(std::max<size_t>(2 * (tb.size() - 1), 2) * (sizeof(ssb_tentry) / 4));
  P.tskip.alloc(std::max<size_t>(SSB_TLIST64 ? units.size() : tb.size() - 1, 1));
  SSB_CUDA(cudaMemcpyAsync(P.units.p, units.data(), sizeof(ssb_unit) * units.size(),
                           cudaMemcpyHostToDevice, s));
  SSB_CUDA(cudaMemcpyAsync(P.task_begin.p, tb.data(), 4 * tb.size(), cudaMemcpyHostToDevice, s));
  if (!split_units.empty())
    SSB_CUDA(cudaMemcpyAsync(P.split_units.p, split_units.data(), 4 * split_units.size(),
                             cudaMemcpyHostToDevice, s));
  SSB_CUDA(cudaMemsetAsync(P.split_hit.p, 0, P.split_hit.bytes(), s));
  SSB_CUDA(cudaMemsetAsync(P.split_best.p, 0xff, P.split_best.bytes(), s));
  SSB_CUDA(cudaMemsetAsync(P.split_count.p, 0, P.split_count.bytes(), s));
  g.sc.sync();
}

// bits layout: visited | F0 | F1 | S0 | S1 | S2 (each region 16-byte aligned)
struct BitRegions {
  int64_t NW4, SW4;
  uint32_t *visited, *F0, *F1, *S0, *S1, *S2, *H0, *H1, *H2;
};

BitRegions bit_regions(ssb_graph& g, int64_t SW) {
  BitRegions R;
  R.NW4 = ((g.n_padded + 31) / 32 + 3) & ~int64_t(3);
  R.SW4 = std::max<int64_t>((SW + 3) & ~int64_t(3), 4);
  g.bits.ensure(size_t(3 * R.NW4 + 6 * R.SW4));
  R.visited = g.bits.p;
  R.F0 = R.visited + R.NW4;
  R.F1 = R.F0 + R.NW4;
  R.S0 = R.F1 + R.NW4;
  R.S1 = R.S0 + R.SW4;
  R.S2 = R.S1 + R.SW4;
  R.H0 = R.S2 + R.SW4;  // hashed summaries (contiguous with S0..S2: one reset region)
  R.H1 = R.H0 + R.SW4;
  R.H2 = R.H1 + R.SW4;
  return R;
}

void collect_stats(const std::vector<int64_t>& rec, int64_t k0, int64_t count,
                   std::vector<ssb_iter_stats>& out) {
  for (int64_t i = 0; i < count; ++i) {
    const int64_t* r = rec.data() + i * kStatW;
    ssb_iter_stats s;
    s.iteration = k0 + i;
    s.elapsed_ns = r[5];
    s.chunks_processed = r[1];
    s.chunks_skipped = r[2];
    s.subchunks_processed = r[3];
    s.columns_processed = r[4];
    s.frontier_size = r[0];
    out.push_back(s);
  }
}

void configure32(const void* fn, size_t dyn_smem) {
  int dev = 0, optin = 0;
  SSB_CUDA(cudaGetDevice(&dev));
  SSB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa;
  SSB_CUDA(cudaFuncGetAttributes(&fa, fn));
  if (dyn_smem + fa.sharedSizeBytes > size_t(optin))
    fail(SSB_EINVAL, "frontier staging exceeds shared memory (SSB_SMEM_KB too large)");
  SSB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn_smem)));
}

// One C=32 BFS in flight: the kernel arguments and the host-side carry between
// cooperative launches. A full BFS is one launch (or several when it is deeper
// than kItersPerLaunch); a shard of a multi-GPU BFS is stepped one iteration
// per launch with a frontier exchange in between (ssb_bfs_shard_*).
struct Run32 {
  Args32 a;
  Geometry G;
  bool sel = false;
  bool hashed = false;           // the hashed-summary kernel (Args32::hash_on)
  int grid = 0;
  int64_t k = 1;                 // next iteration
  int32_t root_pos = 0;
  bool z_skip = false;           // SlimWork skips the root's cell-less chunk
  uint32_t* task_out = nullptr;
  unsigned long long* gone = nullptr;
  std::vector<int64_t> rec;
  ResetArgs reset{};             // init_state, done by the first bfs32_kernel launch (reset.active)
  cudaEvent_t start = nullptr;   // recorded just before that launch (the BFS's device interval)
  bool stepping = false;         // shard mode: always carry state to the next launch
  bool zeroed = false;           // stats/control words already clear for the next launch
  std::vector<int64_t> segs;     // owned chunk segments
};

// The shared-memory image geometry depends on the layout and the SSB_* knobs
// only: computed once per graph and knob setting.
Geometry cached_geometry(ssb_graph& g) {
  const std::string key = std::to_string(env_int("SSB_SMEM_KB", kSmemKB)) + "/" +
                          std::to_string(env_int("SSB_SUMMARY_SHIFT", 0));
  auto* cached = static_cast<std::pair<std::string, Geometry>*>(g.geom.get());
  if (!cached || cached->first != key) {
    g.geom = std::make_shared<std::pair<std::string, Geometry>>(key, geometry32(g));
    cached = static_cast<std::pair<std::string, Geometry>*>(g.geom.get());
  }
  return cached->second;
}

// ---- the peer-mapped window of a fused multi-GPU BFS ------------------------
// words: F0 [NW4] | F1 [NW4] | S0 | S1 | S2 [SW4 each] | slots int64
// [kSlotRing][kMaxRanks] | arrival counter (u64, padded to 16 bytes)
struct WinGeom {
  int64_t NW4 = 0, SW4 = 0;
  int64_t offF[2] = {0, 0}, offS[3] = {0, 0, 0}, offSlots = 0, offArrive = 0, words = 0;
};

WinGeom win_geom(ssb_graph& g) {
  const Geometry G = cached_geometry(g);
  WinGeom w;
  w.NW4 = ((g.n_padded + 31) / 32 + 3) & ~int64_t(3);
  w.SW4 = std::max<int64_t>((G.SW + 3) & ~int64_t(3), 4);
  w.offF[0] = 0;
  w.offF[1] = w.NW4;
  for (int i = 0; i < 3; ++i) w.offS[i] = 2 * w.NW4 + i * w.SW4;
  w.offSlots = 2 * w.NW4 + 3 * w.SW4;
  w.offArrive = w.offSlots + 2 * kSlotRing * kMaxRanks;
  w.words = w.offArrive + 4;
  return w;
}

struct P2PHost {
  int rank = 0, world = 1;
  std::vector<int64_t> segs;  // owned chunk segments
  uint32_t* win[kMaxRanks] = {};
  std::vector<void*> opened;  // peer windows mapped through CUDA IPC
  unsigned long long gen = 0;  // barrier generations completed
  WinGeom wg;
  ~P2PHost() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
  }
};

// The window is allocated (zeroed) once per graph; its geometry must not
// change while peers have it mapped.
uint32_t* p2p_window_alloc(ssb_graph& g, WinGeom& wg) {
  if (g.C != 32) fail(SSB_EINVAL, "the fused multi-GPU BFS needs the C = 32 layout");
  wg = win_geom(g);
  if (g.p2p_win.n != size_t(wg.words)) {
    g.p2p_win.alloc(size_t(wg.words));
    SSB_CUDA(cudaMemset(g.p2p_win.p, 0, g.p2p_win.bytes()));
    g.p2p.reset();
  }
  return g.p2p_win.p;
}

// init_state (semiring.cpp:56-88) in 1-bit form + kernel arguments for the
// chunk range [cb, ce) (all chunks for a single-GPU BFS). With a window (a
// fused multi-GPU shard) the frontier and summaries live in the window.
// |F_{k-1}| above which an iteration sweeps with early exit.
int64_t dense_threshold(const ssb_graph& g, const Geometry& G, bool hashed) {
  // Early-exit sweeps pay off once rows get decided quickly: on hub-heavy
  // graphs (most probes land in the shared prefix) from |F| > n/4096 on; on
  // low-skew graphs from |F| > n/128 (A/B on config 3 and config 4: the
  // batched exact lookups of the early-exit sweep win once the summary is
  // mostly set, even when few rows exit early).
  const bool hubby = G.S == 8;
  // (hub-heavy: n/8192 since the mask-form early-exit step; A/B at S26 /
  // S22 over 64 roots: 4096 4.455 / 0.434, 8192 4.420 / 0.434, 16384
  // 4.411 / 0.437 ms per BFS)
  // With hashed probes the early exit pays from smaller frontiers on (S26
  // iteration 3 of the |F_2| < 8K roots: their block summary bits were ~99%
  // false positives, the hashed ones are set for ~0.6% of the open cells):
  // n/32768 (A/B at S26, 16 roots: 4.234 -> 4.205-4.215 ms per BFS).
  const int hub_div = env_int("SSB_DENSE_DIV_HUB", hashed ? 32768 : 8192);
  const int div = std::max(1, env_int("SSB_DENSE_DIV", hubby ? hub_div : 128));
  return std::max<int64_t>(1, g.n / div);
}

Run32 prepare32(ssb_graph& g, int32_t root_pos, int32_t root_code, const ssb_bfs_options& o,
                const std::vector<int64_t>& segs, const P2PHost* p2p = nullptr,
                cudaEvent_t start = nullptr, bool reset_in_kernel = false, bool allow_hash = true) {
  cudaStream_t s = g.sc.s;
  Run32 r;
  r.sel = o.variant == SSB_SELMAX;
  r.root_pos = root_pos;
  build_plan32(g, o.slimchunk_len, segs);
  r.segs = segs;
  r.G = cached_geometry(g);
  const Geometry& G = r.G;
  // hashed summaries on hub-heavy graphs (S = 8) with a summary of >= 64K
  // bits (S22's 16K-bit summary is saturated by the frontiers that reach it
  // either way); not where summary words are exchanged between ranks (p2p
  // windows, NCCL shards: allow_hash = false)
  r.hashed = allow_hash && !p2p && G.S == 8 && G.SW > 0 &&
             int64_t(G.SW) * 32 >= env_int("SSB_HASH_MIN_BITS", 65536) && env_int("SSB_HASH_SUMMARY", 1) != 0;
  BitRegions R = bit_regions(g, G.SW);
  if (p2p) {
    uint32_t* w = p2p->win[p2p->rank];
    R.F0 = w + p2p->wg.offF[0];
    R.F1 = w + p2p->wg.offF[1];
    R.S0 = w + p2p->wg.offS[0];
    R.S1 = w + p2p->wg.offS[1];
    R.S2 = w + p2p->wg.offS[2];
  }
  g.level.ensure(size_t(std::max<int64_t>(g.n_padded, 1)));
  g.parent.ensure(size_t(std::max<int64_t>(g.n_padded, 1)));
  g.dstats.ensure(size_t(kItersPerLaunch) * kStatW);
  // control words: task_ctr [K] | task_out [K] | gone_chunks [K] (8-byte)
  g.dctrl.ensure(size_t(kItersPerLaunch) * 4);
  uint32_t* task_ctr = g.dctrl.p;
  r.task_out = task_ctr + kItersPerLaunch;
  r.gone = reinterpret_cast<unsigned long long*>(r.task_out + kItersPerLaunch);

  {
    ResetArgs ra{};
    ra.reg[0] = reinterpret_cast<uint4*>(R.visited);
    ra.n16[0] = R.NW4 / 4;
    ra.reg[1] = reinterpret_cast<uint4*>(R.F0);
    ra.n16[1] = R.NW4 / 4;
    ra.reg[2] = reinterpret_cast<uint4*>(R.S0);       // S0..S2, H0..H2 (contiguous)
    ra.n16[2] = (p2p ? 3 : 6) * R.SW4 / 4;            // (peer windows hold S only; no hashing there)
    ra.reg[3] = reinterpret_cast<uint4*>(g.dstats.p);  // the first launch's records
    ra.n16[3] = int64_t(g.dstats.bytes() / 16);
    ra.reg[4] = reinterpret_cast<uint4*>(g.dctrl.p);   // and control words
    ra.n16[4] = int64_t(g.dctrl.bytes() / 16);
    ra.tskip = g.plan.tskip.p;
    ra.n_tasks = int64_t(g.plan.tskip.bytes());
    ra.visited = R.visited;
    ra.F0 = R.F0;
    ra.S0 = G.SW ? R.S0 : nullptr;
    ra.root_pos = root_pos;
    ra.root_code = root_code;
    ra.PW = G.PW;
    ra.gshift = G.gshift;
    ra.level = g.level.p;
    ra.parent = g.parent.p;
    if (reset_in_kernel) {  // the first bfs32_kernel launch does it (launch32)
      ra.active = 1;
      r.reset = ra;
      r.start = start;
    } else {
      // the BFS's device interval opens with its first device operation (the
      // host-side preparation above is not device work)
      if (start) SSB_CUDA(cudaEventRecord(start, s));
      reset32_kernel<<<num_sms() * 4, 256, 0, s>>>(ra);
      SSB_CUDA(cudaGetLastError());
      g.last_launches += 1;  // reset32_kernel
    }
    r.zeroed = true;       // the first launch's stats/control words are clear
  }

  {
    // The kernel's dynamic shared-memory attribute is set (and the fit
    // checked) only when it differs from what the kernel is configured for on
    // this device: the driver calls are host time on every BFS.
    struct Cfg {
      int dev;
      Bfs32Fn fn;
      size_t smem;
    };
    static std::mutex mu;
    static std::vector<Cfg> current;
    int dev = 0;
    SSB_CUDA(cudaGetDevice(&dev));
    const Bfs32Fn fn = bfs32_fn(r.sel, G.S, r.hashed);
    std::lock_guard<std::mutex> lock(mu);
    Cfg* c = nullptr;
    for (Cfg& x : current)
      if (x.dev == dev && x.fn == fn) c = &x;
    if (!c || c->smem != G.smem) {
      configure32((const void*)fn, G.smem);
      int per_sm = 0;
      SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, kThreads,
                                                             G.smem));
      if (per_sm < 1) fail(SSB_ECUDA, "bfs32 kernel does not fit on an SM");
      if (c) c->smem = G.smem;
      else current.push_back({dev, fn, G.smem});
    }
  }
  r.grid = std::max(1, std::min(num_sms(), env_int("SSB_GRID", num_sms())));  // A/B: fewer CTAs

  Args32& a = r.a;
  a.col = g.col.p;
  a.cs = g.cs.p;
  a.cl = g.cl.p;
  a.units = g.plan.units.p;
  a.task_begin = g.plan.task_begin.p;
  a.split_units = g.plan.split_units.p;
  a.split_hit = g.plan.split_hit.p;
  a.split_best = g.plan.split_best.p;
  a.split_count = g.plan.split_count.p;
  a.visited = R.visited;
  a.F0 = R.F0;
  a.F1 = R.F1;
  a.S0 = R.S0;
  a.S1 = R.S1;
  a.S2 = R.S2;
  a.H0 = R.H0;
  a.H1 = R.H1;
  a.H2 = R.H2;
  a.HB = uint32_t(G.SW) * 32u;
  a.hash_on = r.hashed ? 1 : 0;  // (see r.hashed)
  {
    // hash into the largest power of two of bits the summary words hold
    // (every S26/S28 summary is one; otherwise the top words stay zero)
    int lg = 1;
    while (lg < 31 && (uint32_t{1} << (lg + 1)) <= a.HB) ++lg;
    a.hash_arg = uint32_t(32 - lg);
  }
  a.hash_prev_in = 0;
  {
    // A/B at S26 over 16 roots: HB / 2 4.234, HB 4.205-4.215 ms per BFS
    // (with the n/32768 dense threshold below), no hashing 4.271
    const int64_t ht = env_int("SSB_HASH_THR", -1);
    a.hash_thr = ht >= 0 ? ht : (int64_t{1} << (32 - a.hash_arg));
  }
  a.level = g.level.p;
  a.parent = g.parent.p;
  a.stats = g.dstats.p;
  a.task_ctr = task_ctr;
  a.task_out = r.task_out;
  a.gone_chunks = r.gone;
  a.tlist0 = reinterpret_cast<ssb_tentry*>(g.plan.tlist.p);
  a.tlist1 = a.tlist0 + g.plan.n_tasks;
  a.tskip = g.plan.tskip.p;
  // A task may retire the first time all its units are skipped: its chunks'
  // words in the other frontier buffer then keep the bits of the iteration
  // before (the rows reached last), never cleared. Those bits are harmless to
  // the sweeps — every row with one of those vertices among its cells was
  // reached in the iteration that read them, so later probes that see them
  // belong to visited (decided, masked) rows — but not to anything that
  // counts or gathers frontier WORDS: the NCCL shard exchange (front_count /
  // summary_from_words kernels) keeps the two-iteration rule.
  a.retire_once = env_int("SSB_RETIRE_ONCE", 1) ? 1 : 0;
  a.n_tasks = int32_t(g.plan.n_tasks);
  a.gone_base = 0;
  a.front_in = 1;  // F_0 = {root}
  {
    a.dense_thr = dense_threshold(g, G, a.hash_on != 0);
    // once |F| exceeds the summary's bits most of them are set: probe exactly
    const int64_t dt = env_int("SSB_DIRECT_THR", -1);
    a.direct_thr = dt >= 0 ? dt : (G.SW > 0 ? int64_t(G.SW) * 32 : INT64_MAX);
  }
  a.n_chunks = int32_t(g.n_chunks);
  a.PW = G.PW;
  a.SW = G.SW;
  a.gshift = G.gshift;
  a.L = int32_t(std::max<int64_t>(0, std::min<int64_t>(o.slimchunk_len, INT32_MAX)));
  a.slimwork = o.slimwork ? 1 : 0;
  a.root_code = root_code;
  a.trace = nullptr;
  a.carry = nullptr;
  a.rec_host = nullptr;
  static int* trace_buf = nullptr;
  if (std::getenv("SSB_TRACE")) {
    if (!trace_buf) SSB_CUDA(cudaHostAlloc(&trace_buf, 64, cudaHostAllocMapped));
    std::memset(trace_buf, 0, 64);
    SSB_CUDA(cudaHostGetDevicePointer(&a.trace, trace_buf, 0));
  }
  {
    const int64_t real_last = g.n - (g.n_chunks - 1) * 32;  // 1..32
    a.last_real = real_last >= 32 ? 0xffffffffu : ((1u << real_last) - 1u);
  }
  // chunks without cells are processed (0 columns, 0 segments) unless SlimWork
  // skips the root's own chunk when the root is its only real row
  const int64_t rc = root_pos / 32;
  bool owns_rc = false;
  for (size_t q = 0; q + 1 < segs.size(); q += 2) owns_rc = owns_rc || (rc >= segs[q] && rc < segs[q + 1]);
  r.z_skip = o.slimwork && owns_rc && g.cl_host[rc] == 0 &&
             std::min<int64_t>(32, g.n - rc * 32) == 1;
  r.k = 1;
  return r;
}

// Runs iterations r.k .. kend-1 (stopping early when no row is newly reached
// in this launch's range); appends their stats. Returns the number run.
int64_t launch32(ssb_graph& g, Run32& r, int64_t kend, std::vector<ssb_iter_stats>& stats,
                 bool& conv) {
  cudaStream_t s = g.sc.s;
  Args32& a = r.a;
  a.k_begin = int32_t(r.k);
  a.k_end = int32_t(kend);
  if (!r.zeroed) {
    SSB_CUDA(cudaMemsetAsync(g.dstats.p, 0, g.dstats.bytes(), s));
    SSB_CUDA(cudaMemsetAsync(g.dctrl.p, 0, g.dctrl.bytes(), s));
  }
  r.zeroed = false;
  // the launch's first records land in mapped PINNED host memory, written by
  // the kernel itself as it ends: no copy on the stream after it (a pageable
  // cudaMemcpyAsync cost ~12 us, a pinned one ~6 us, of a 0.41 ms S22 BFS)
  struct RecHost {
    int64_t* p = nullptr;
    ~RecHost() {
      if (p) cudaFreeHost(p);
    }
  };
  if (!g.rec_host) {
    auto h = std::make_shared<RecHost>();
    SSB_CUDA(cudaHostAlloc(&h->p, size_t(kRecFirst) * kStatW * 8, cudaHostAllocMapped | cudaHostAllocPortable));
    g.rec_host = h;
  }
  int64_t* pin = static_cast<RecHost*>(g.rec_host.get())->p;
  SSB_CUDA(cudaHostGetDevicePointer(&a.rec_host, pin, 0));
  void* params[] = {&a, &r.reset};
  if (r.start) SSB_CUDA(cudaEventRecord(r.start, s));
  r.start = nullptr;
  SSB_CUDA(cudaEventRecord(g.sc.e0, s));
  SSB_CUDA(cudaLaunchCooperativeKernel(
      (const void*)bfs32_fn(r.sel, r.G.S, r.hashed), dim3(r.grid),
      dim3(kThreads), params, r.G.smem, s));
  SSB_CUDA(cudaGetLastError());
  SSB_CUDA(cudaEventRecord(g.sc.e1, s));
  r.reset.active = 0;  // later launches of this BFS carry the state on
  if (a.trace) {  // debug: poll progress instead of blocking forever
    cudaEvent_t done;
    SSB_CUDA(cudaEventCreate(&done));
    SSB_CUDA(cudaEventRecord(done, s));
    for (int spin = 0; cudaEventQuery(done) == cudaErrorNotReady; ++spin) {
      if (spin % 1000 == 999)
        fprintf(stderr, "[ssb trace] k=%d phase=%d arrived=%d\n", a.trace[0], a.trace[1], a.trace[2]);
      if (spin > 10000) { fprintf(stderr, "[ssb trace] giving up\n"); std::abort(); }
      usleep(1000);
    }
    cudaEventDestroy(done);
  }
#ifdef SSB_COUNT
  {
    unsigned long long c[8];
    g.sc.sync();
    SSB_CUDA(cudaMemcpyFromSymbol(c, g_cnt, sizeof c));
    fprintf(stderr, "[ssb count] k=%d probes %llu tail %llu exact %llu hits %llu lookup-steps %llu\n",
            a.k_begin, c[0], c[1], c[2], c[3], c[4]);
    const unsigned long long z[8] = {};
    SSB_CUDA(cudaMemcpyToSymbol(g_cnt, z, sizeof z));
  }
#endif
#ifdef SSB_PHASES
  {
    unsigned long long ph[4];
    g.sc.sync();
    SSB_CUDA(cudaMemcpyFromSymbol(ph, g_phase, sizeof ph));
    if (ph[3])
      fprintf(stderr, "[ssb phases] iterations %llu: staging %.2f us, sweep %.2f us, barrier %.2f us\n",
              ph[3], ph[0] / 1e3 / ph[3], ph[1] / 1e3 / ph[3], ph[2] / 1e3 / ph[3]);
    const unsigned long long z[4] = {0, 0, 0, 0};
    SSB_CUDA(cudaMemcpyToSymbol(g_phase, z, sizeof z));
  }
#endif
  // the records of the first kRecFirst iterations come back with the launch;
  // the rest only when the launch got that far
  const int64_t nrec = kend - r.k;
  const int64_t first = std::min<int64_t>(nrec, kRecFirst);
  SSB_CUDA(cudaEventRecord(g.sc.e_end, s));
  // blocking wait (e_end is a blocking-sync event): the host threads widening
  // the previous root's result during a batch keep every core
  SSB_CUDA(cudaEventSynchronize(g.sc.e_end));
  r.rec.assign(pin, pin + first * kStatW);
  if (nrec > first && r.rec[size_t(first - 1) * kStatW] != 0) {
    r.rec.resize(size_t(nrec) * kStatW);
    SSB_CUDA(cudaMemcpy(r.rec.data() + first * kStatW, g.dstats.p + first * kStatW,
                        size_t(nrec - first) * kStatW * 8, cudaMemcpyDeviceToHost));
  }
  {
    float kms = 0;
    SSB_CUDA(cudaEventElapsedTime(&kms, g.sc.e0, g.sc.e1));
    g.last_kernel_ms += kms;
    g.last_launches += 1;  // bfs32_kernel
  }
  // the launch ran iterations k .. until a record with frontier 0 or kend
  int64_t ran = 0;
  conv = false;
  for (int64_t i = 0; i < kend - r.k; ++i) {
    ++ran;
    if (r.rec[size_t(i) * kStatW] == 0) {
      conv = true;
      break;
    }
  }
  collect_stats(r.rec, r.k, ran, stats);
  for (int64_t i = 0; i < ran; ++i) g.last_swept += r.rec[size_t(i) * kStatW + 6];
  for (size_t i = stats.size() - size_t(ran); i < stats.size(); ++i) {
    stats[i].chunks_processed += g.plan.empty_chunks - (r.z_skip ? 1 : 0);
    stats[i].chunks_skipped += r.z_skip ? 1 : 0;
  }
  if (conv && !r.stepping) {
    r.k += ran;
    return ran;
  }
  // carry the active task list and the retired-chunk count into the next launch
  std::vector<uint32_t> outs(static_cast<size_t>(ran));
  std::vector<unsigned long long> gones(static_cast<size_t>(ran));
  SSB_CUDA(cudaMemcpyAsync(outs.data(), r.task_out, 4 * ran, cudaMemcpyDeviceToHost, s));
  SSB_CUDA(cudaMemcpyAsync(gones.data(), r.gone, 8 * ran, cudaMemcpyDeviceToHost, s));
  g.sc.sync();
  a.n_tasks = int32_t(outs.back());
  for (auto x : gones) a.gone_base += x;
  // the launch's last iteration built the hashed summary iff it swept sparse
  // (its input frontier |F_{k-1}| at most the dense threshold)
  const int64_t f_in_last = ran >= 2 ? r.rec[size_t(ran - 2) * kStatW] : a.front_in;
  a.hash_prev_in = (r.hashed && f_in_last <= a.dense_thr) ? 1 : 0;
  a.front_in = r.rec[size_t(ran - 1) * kStatW];
  r.k += ran;
  return ran;
}

// Returns true when converged; appends per-iteration stats.
bool run32(ssb_graph& g, int32_t root_pos, int32_t root_code, const ssb_bfs_options& o,
           int64_t cap, std::vector<ssb_iter_stats>& stats, cudaEvent_t start = nullptr) {
  const auto h0 = std::chrono::steady_clock::now();
  Run32 r = prepare32(g, root_pos, root_code, o, {0, g.n_chunks}, nullptr, start, true);
  if (std::getenv("SSB_GAPS"))
    fprintf(stderr, "[ssb gaps] host prepare32 %.1f us\n",
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count());
  // SSB_ITERS_PER_LAUNCH=1 (profiling): one cooperative launch per iteration
  const int64_t per = std::max(1, std::min(kItersPerLaunch, env_int("SSB_ITERS_PER_LAUNCH", kItersPerLaunch)));
  while (r.k <= cap) {
    bool conv = false;
    launch32(g, r, std::min<int64_t>(cap + 1, r.k + per), stats, conv);
    if (conv) return true;
  }
  return false;
}

bool run_generic(ssb_graph& g, int32_t root_pos, int32_t root_code, const ssb_bfs_options& o,
                 int64_t cap, std::vector<ssb_iter_stats>& stats) {
  cudaStream_t s = g.sc.s;
  const int64_t np = g.n_padded;
  g.level.ensure(size_t(std::max<int64_t>(np, 1)));
  g.parent.ensure(size_t(std::max<int64_t>(np, 1)));
  g.gbytes.ensure(size_t(3 * np + g.n_chunks + 16));
  g.dstats.ensure(size_t(kItersPerLaunch) * kStatW);
  // the unit plan (host, from cl) and the per-row hit slots, cached per graph
  struct GenPlan {
    DevBuf<GenUnit> units;
    int64_t n_units = 0;
    DevBuf<int32_t> hitbest;
  };
  if (!g.gen_plan) {
    auto gp = std::make_shared<GenPlan>();
    std::vector<GenUnit> us;
    for (int64_t i = 0; i < g.n_chunks; ++i)
      for (int32_t c = 0; c < g.cl_host[size_t(i)]; c += kGenUnitCols)
        us.push_back({int32_t(i), c, std::min(kGenUnitCols, g.cl_host[size_t(i)] - c)});
    // longest first: hub pieces start early instead of trailing the sweep
    std::stable_sort(us.begin(), us.end(), [](const GenUnit& x, const GenUnit& y) { return x.col_len > y.col_len; });
    gp->n_units = int64_t(us.size());
    gp->units.alloc(std::max<size_t>(us.size(), 1));
    if (!us.empty())
      SSB_CUDA(cudaMemcpy(gp->units.p, us.data(), us.size() * sizeof(GenUnit), cudaMemcpyHostToDevice));
    gp->hitbest.alloc(size_t(std::max<int64_t>(np, 1)));
    SSB_CUDA(cudaMemset(gp->hitbest.p, 0xff, gp->hitbest.bytes()));  // -1
    g.gen_plan = gp;
  }
  GenPlan& GP = *static_cast<GenPlan*>(g.gen_plan.get());
  uint8_t* vis = g.gbytes.p;
  uint8_t* f0 = vis + np;
  uint8_t* f1 = f0 + np;
  uint8_t* skip = f1 + np;
  SSB_CUDA(cudaMemsetAsync(vis, 0, size_t(2 * np), s));  // visited + F_0
  const uint8_t one = 1;
  SSB_CUDA(cudaMemcpyAsync(vis + root_pos, &one, 1, cudaMemcpyHostToDevice, s));
  SSB_CUDA(cudaMemcpyAsync(f0 + root_pos, &one, 1, cudaMemcpyHostToDevice, s));
  const int32_t zero = 0;
  SSB_CUDA(cudaMemcpyAsync(g.level.p + root_pos, &zero, 4, cudaMemcpyHostToDevice, s));
  SSB_CUDA(cudaMemcpyAsync(g.parent.p + root_pos, &root_code, 4, cudaMemcpyHostToDevice, s));
  ArgsG a;
  a.col = g.col.p;
  a.cs = g.cs.p;
  a.cl = g.cl.p;
  a.C = g.C;
  a.n = g.n;
  a.n_chunks = g.n_chunks;
  a.vis = vis;
  a.f0 = f0;
  a.f1 = f1;
  a.skip = skip;
  a.level = g.level.p;
  a.parent = g.parent.p;
  a.units = GP.units.p;
  a.n_units = GP.n_units;
  a.hitbest = GP.hitbest.p;
  a.stats = reinterpret_cast<unsigned long long*>(g.dstats.p);
  a.L = int32_t(std::max<int64_t>(0, std::min<int64_t>(o.slimchunk_len, INT32_MAX)));
  a.slimwork = o.slimwork ? 1 : 0;
  a.root_code = root_code;
  a.selmax = o.variant == SSB_SELMAX;
  static int grid = 0;  // co-resident CTAs of 1024 threads, once per process
  if (!grid) {
    int per_sm = 0;
    SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)genc_kernel, 1024, 0));
    if (per_sm < 1) fail(SSB_ECUDA, "genc kernel does not fit on an SM");
    grid = num_sms() * std::min(per_sm, 2);
  }
  bool conv = false;
  std::vector<int64_t> rec(size_t(kItersPerLaunch) * kStatW);
  for (int64_t kb = 1; kb <= cap && !conv;) {
    const int64_t ke = std::min<int64_t>(cap + 1, kb + kItersPerLaunch);
    a.k_begin = int32_t(kb);
    a.k_end = int32_t(ke);
    SSB_CUDA(cudaMemsetAsync(g.dstats.p, 0, size_t(ke - kb) * kStatW * 8, s));
    void* params[] = {&a};
    SSB_CUDA(cudaEventRecord(g.sc.e0, s));
    SSB_CUDA(cudaLaunchCooperativeKernel((const void*)genc_kernel, dim3(grid), dim3(1024), params, 0, s));
    SSB_CUDA(cudaGetLastError());
    SSB_CUDA(cudaEventRecord(g.sc.e1, s));
    SSB_CUDA(cudaMemcpyAsync(rec.data(), g.dstats.p, size_t(ke - kb) * kStatW * 8, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaEventRecord(g.sc.e_end, s));  // bfs_run's device-time end
    g.sc.sync();
    float ms = 0;
    SSB_CUDA(cudaEventElapsedTime(&ms, g.sc.e0, g.sc.e1));
    g.last_kernel_ms += ms;
    g.last_launches += 1;
    int64_t ran = 0;
    for (int64_t i = 0; i < ke - kb && !conv; ++i) {
      ++ran;
      g.last_swept += rec[size_t(i) * kStatW + 4];  // the generic engine streams every processed column
      conv = rec[size_t(i) * kStatW] == 0;
    }
    collect_stats(rec, kb, ran, stats);
    kb += ran;
  }
  // the shared epilogue reads the visited bitmap
  BitRegions R = bit_regions(g, 0);
  bytes_to_bits_kernel<<<grid_for((np + 31) / 32), 256, 0, s>>>(vis, np, R.visited);
  SSB_CUDA(cudaGetLastError());
  g.last_launches += 1;
  g.sc.sync();
  return conv;
}

}  // namespace

int num_sms() {
  static int sms = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    return v;
  }();
  return sms;
}

int bfs_run(ssb_graph& g, int64_t root, const ssb_bfs_options& o, ssb_iter_stats* stats,
            int64_t stats_cap, int64_t* iterations, double* device_ms) {
  g.need_full("a single-GPU BFS");
  if (o.variant < 0 || o.variant > 3) fail(SSB_EINVAL, "bad variant");
  // semiring.cpp:57-60
  if (root < 0 || root >= g.n)
    fail(SSB_ERANGE, "root " + std::to_string(root) + " outside [0, " + std::to_string(g.n) + ")");
  g.last_valid = false;
  const int32_t root_pos = [&] {
    int32_t p = 0;
    SSB_CUDA(cudaMemcpy(&p, g.inv_perm.p + root, 4, cudaMemcpyDeviceToHost));
    return p;
  }();
  // sel-max: the reference seeds x[root] = root+1 in ORIGINAL numbering and
  // decodes it as a position; compat keeps that encoding.
  const int32_t root_code = (o.variant == SSB_SELMAX && o.selmax_compat) ? int32_t(root) : root_pos;
  const int64_t cap = o.max_iterations > 0 ? o.max_iterations : g.n + 1;
  std::vector<ssb_iter_stats> st;
  g.last_kernel_ms = 0;
  g.last_launches = 0;
  g.last_swept = 0;
  cudaEvent_t t0, t1;
  SSB_CUDA(cudaEventCreate(&t0));
  SSB_CUDA(cudaEventCreate(&t1));
  if (g.C != 32) SSB_CUDA(cudaEventRecord(t0, g.sc.s));  // (C = 32: before its first launch)
  bool conv;
  try {
    conv = g.C == 32 ? run32(g, root_pos, root_code, o, cap, st, t0)
                     : run_generic(g, root_pos, root_code, o, cap, st);
  } catch (...) {
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    throw;
  }
  SSB_CUDA(cudaEventRecord(t1, g.sc.s));
  SSB_CUDA(cudaEventSynchronize(t1));
  // device time: from the first enqueued operation to the end of the last
  // launch (its records land in mapped host memory as it ends) — the host's
  // wake-up after that is not device work (t1 bounds it when the engine
  // enqueued nothing that records e_end)
  float ms = 0;
  SSB_CUDA(cudaEventElapsedTime(&ms, t0, g.sc.e_end));
  {
    float ms1 = 0;
    SSB_CUDA(cudaEventElapsedTime(&ms1, t0, t1));
    if (ms <= 0.f || ms > ms1) ms = ms1;
  }
  if (std::getenv("SSB_GAPS") && g.C == 32) {  // debug: where the time outside the kernel goes
    float pre = 0, post = 0;
    SSB_CUDA(cudaEventElapsedTime(&pre, t0, g.sc.e0));
    SSB_CUDA(cudaEventElapsedTime(&post, g.sc.e1, g.sc.e_end));
    fprintf(stderr, "[ssb gaps] before last launch %.1f us, after it %.1f us, device %.3f ms\n",
            pre * 1e3, post * 1e3, ms);
  }
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  if (device_ms) *device_ms = ms;
  if (iterations) *iterations = int64_t(st.size());
  if (stats)
    for (int64_t i = 0; i < std::min<int64_t>(stats_cap, int64_t(st.size())); ++i) stats[i] = st[i];
  g.last_root = root;
  g.last_variant = o.variant;
  g.last_compat = o.selmax_compat;
  g.last_iterations = int64_t(st.size());
  g.last_valid = true;
  return conv ? SSB_OK : SSB_ECAP;
}

void fetch_rows(ssb_graph& g, int want_parents, int64_t* dist, int64_t* parent,
                int64_t* parent_len, const uint8_t* owned);

void bfs_fetch(ssb_graph& g, int want_parents, int64_t* dist, int64_t* parent,
               int64_t* parent_len) {
  fetch_rows(g, want_parents, dist, parent, parent_len, nullptr);
}

// Pinned host copy of the wire buffer and the per-chunk completion events.
// One slot of the result fetch: the device wire buffer, its pinned host copy,
// a copy stream and the per-chunk events (pack done / copy done). Two slots
// let a batch pack root i+1 while the host still widens root i.
struct WireSlot {
  DevBuf<uint8_t> dev;
  uint8_t* host = nullptr;
  size_t bytes = 0;
  cudaStream_t copy = nullptr;
  std::vector<cudaEvent_t> packed, ready;
  DevBuf<int> flag;        // dp_transform consistency flag of this slot's root
  int* hflag = nullptr;    // ... its pinned host copy
  std::vector<int64_t> bounds;
  int packed_bits = 0;     // > 0: the packed 4-byte wire (pack_wire32_kernel) of this slot's root
  ~WireSlot() {
    if (host) cudaFreeHost(host);
    if (hflag) cudaFreeHost(hflag);
    for (auto e : packed) cudaEventDestroy(e);
    for (auto e : ready) cudaEventDestroy(e);
    if (copy) cudaStreamDestroy(copy);
  }
};
struct WireSlots {
  WireSlot slot[2];
};

WireSlot& wire_slot(ssb_graph& g, int k, size_t bytes, int K) {
  auto* W = static_cast<WireSlots*>(g.wire_host.get());
  if (!W) {
    auto w = std::make_shared<WireSlots>();
    g.wire_host = w;
    W = w.get();
  }
  WireSlot& S = W->slot[k];
  if (S.bytes < bytes) {
    S.dev.alloc(bytes);
    if (S.host) cudaFreeHost(S.host);
    S.host = nullptr;
    SSB_CUDA(cudaHostAlloc(&S.host, bytes, cudaHostAllocDefault));
    S.bytes = bytes;
  }
  if (!S.copy) SSB_CUDA(cudaStreamCreateWithFlags(&S.copy, cudaStreamNonBlocking));
  if (!S.hflag) SSB_CUDA(cudaHostAlloc(&S.hflag, sizeof(int), cudaHostAllocDefault));
  S.flag.ensure(1);
  while (int(S.ready.size()) < K) {
    cudaEvent_t a, b;
    SSB_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    SSB_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming | cudaEventBlockingSync));
    S.packed.push_back(a);
    S.ready.push_back(b);
  }
  return S;
}

size_t wire_poff(int64_t n) { return (size_t(n) + 255) & ~size_t(255); }

// Device half of a whole-result fetch through the narrow wire format: the
// pack kernels run on the BFS stream (so the next BFS may reuse level /
// parent once they are done), each chunk's D2H copy on the slot's copy stream
// as soon as that chunk is packed. Returns at once.
void wire_launch(ssb_graph& g, WireSlot& S, int K, bool want_dist, bool want_parents) {
  cudaStream_t s = g.sc.s;
  const int64_t n = g.n;
  const bool sel = g.last_variant == SSB_SELMAX;
  const size_t poff = wire_poff(n);
  uint8_t* lev8 = S.dev.p;
  int32_t* par32 = reinterpret_cast<int32_t*>(S.dev.p + poff);
  uint8_t* hlev = S.host;
  int32_t* hpar = reinterpret_cast<int32_t*>(S.host + poff);
  BitRegions R = bit_regions(g, 0);
  const bool dp = want_parents && !sel;
  // the packed 4-byte wire when ids and levels fit one word together
  int idb = 1;
  while (idb < 32 && (int64_t{1} << idb) < n) ++idb;
  const bool packed = want_dist && want_parents && sel && idb <= 31 &&
                      g.last_iterations < int64_t(0xffffffffu >> idb) && env_int("SSB_WIRE_PACKED", 1) != 0;
  S.packed_bits = packed ? idb : 0;
  *S.hflag = 0;
  if (dp) SSB_CUDA(cudaMemsetAsync(S.flag.p, 0, 4, s));
  S.bounds.assign(size_t(K) + 1, 0);
  for (int c = 0; c <= K; ++c) S.bounds[size_t(c)] = std::min(n, (n * c / K + 63) / 64 * 64);
  for (int c = 0; c < K; ++c) {
    const int64_t b = S.bounds[size_t(c)], len = S.bounds[size_t(c) + 1] - b;
    if (len > 0 && packed) {
      pack_wire32_kernel<<<grid_for(len), 256, 0, s>>>(R.visited, g.level.p, g.parent.p, g.perm.p, g.inv_perm.p,
                                                       b, b + len, idb, reinterpret_cast<uint32_t*>(par32));
      SSB_CUDA(cudaGetLastError());
    } else if (len > 0) {
      pack_wire_kernel<<<grid_for(len), 256, 0, s>>>(R.visited, g.level.p, g.parent.p, g.perm.p,
                                                     g.inv_perm.p, b, b + len, want_dist ? lev8 : nullptr,
                                                     want_parents && sel ? par32 : nullptr);
      if (dp)
        dp_parent_kernel<int32_t><<<grid_for(len), 256, 0, s>>>(g.col.p, g.cs.p, g.cl.p, g.C, R.visited,
                                                                g.level.p, g.perm.p, g.inv_perm.p, b + len,
                                                                par32, S.flag.p, nullptr, b);
      SSB_CUDA(cudaGetLastError());
    }
    SSB_CUDA(cudaEventRecord(S.packed[size_t(c)], s));
    SSB_CUDA(cudaStreamWaitEvent(S.copy, S.packed[size_t(c)], 0));
    if (len > 0 && want_dist && !packed)
      SSB_CUDA(cudaMemcpyAsync(hlev + b, lev8 + b, size_t(len), cudaMemcpyDeviceToHost, S.copy));
    if (len > 0 && want_parents)
      SSB_CUDA(cudaMemcpyAsync(hpar + b, par32 + b, 4 * size_t(len), cudaMemcpyDeviceToHost, S.copy));
    SSB_CUDA(cudaEventRecord(S.ready[size_t(c)], S.copy));
  }
  if (dp) SSB_CUDA(cudaMemcpyAsync(S.hflag, S.flag.p, 4, cudaMemcpyDeviceToHost, S.copy));
}

// Host half: the pool widens chunk c into the caller's int64 arrays once it
// has landed (dist INT64_MAX where unreached, parent -1).
void wire_finish(WireSlot& S, int64_t n, int64_t* dist, int64_t* parent) {
  const int K = int(S.bounds.size()) - 1;
  std::vector<cudaEvent_t> ready(S.ready.begin(), S.ready.begin() + K);
  widen_chunks(S.bounds, ready, S.host, reinterpret_cast<int32_t*>(S.host + wire_poff(n)), dist, parent,
               dist && parent ? S.packed_bits : 0);
  SSB_CUDA(cudaStreamSynchronize(S.copy));
  if (*S.hflag) fail(SSB_EINVAL, "inconsistent distances: a reached vertex has no neighbor one level closer");
}

// 64 chunks (5 MB of wire each at S26): a chunk the DMA just wrote is widened
// while it is still in the host LLC (A/B: 16 -> 64 chunks, batch e2e +11%)
int wire_chunks() { return std::max(1, std::min(256, env_int("SSB_WIRE_CHUNKS", 64))); }

// Whole-result fetch through the narrow wire format: pack (device) -> chunked
// D2H into pinned staging -> host threads widen chunk c while c+1 is in
// flight. 5 bytes per vertex cross PCIe instead of 16.
void fetch_wire(ssb_graph& g, int want_parents, int64_t* dist, int64_t* parent, int64_t* parent_len) {
  const int64_t n = g.n;
  const int K = wire_chunks();
  WireSlot& S = wire_slot(g, 0, wire_poff(n) + 4 * size_t(n), K);
  const bool want_p = want_parents && parent != nullptr;
  wire_launch(g, S, K, dist != nullptr, want_p);
  wire_finish(S, n, dist, want_p ? parent : nullptr);
  g.sc.sync();
  if (parent_len) *parent_len = want_parents ? n : 0;
}

// A batch of BFS from `roots`, results delivered like ssb_bfs_spmv's into
// dist[i] / parent[i] (entries may repeat: root i's result then replaces
// root i-1's): root i's result is packed on the device, crosses PCIe and is
// widened by the host threads WHILE root i+1's BFS runs — the device and the
// PCIe / host-memory bound fetch overlap (two wire slots). Returns the index
// of the first root that hit the iteration cap (its dist delivered, no
// parents, later roots not run), or -1.
int64_t bfs_batch(ssb_graph& g, const int64_t* roots, int64_t nroots, const ssb_bfs_options& o,
                  int64_t* const* dist, int64_t* const* parent, int64_t* iterations) {
  g.need_full("a single-GPU BFS");
  const int64_t n = g.n;
  const int K = wire_chunks();
  std::future<void> pending;
  auto join = [&] {
    if (pending.valid()) pending.get();
  };
  try {
    for (int64_t i = 0; i < nroots; ++i) {
      int64_t it = 0;
      const int rc = bfs_run(g, roots[i], o, nullptr, 0, &it, nullptr);
      if (iterations) iterations[i] = it;
      const bool want_p = rc == SSB_OK && o.want_parents && parent && parent[i];
      if (rc != SSB_OK || it > 254 || n < env_int("SSB_WIRE_MIN", 1 << 16) || env_int("SSB_WIRE", 1) == 0) {
        join();  // the direct path (deep or capped BFS, small graphs)
        fetch_rows(g, want_p, dist ? dist[i] : nullptr, want_p ? parent[i] : nullptr, nullptr, nullptr);
        if (rc == SSB_ECAP) return i;
        continue;
      }
      join();  // root i-1 widened: its slot is free for root i+1
      WireSlot& S = wire_slot(g, int(i & 1), wire_poff(n) + 4 * size_t(n), K);
      int64_t* d = dist ? dist[i] : nullptr;
      int64_t* p = want_p ? parent[i] : nullptr;
      wire_launch(g, S, K, d != nullptr, want_p);
      pending = std::async(std::launch::async, [&S, n, d, p] { wire_finish(S, n, d, p); });
    }
    join();
  } catch (...) {
    if (pending.valid()) pending.wait();
    throw;
  }
  g.sc.sync();
  return -1;
}

// Results in original ids; owned (device, per chunk, may be null = all): only
// the rows of a shard's chunks, the caller's other entries kept.
void fetch_rows(ssb_graph& g, int want_parents, int64_t* dist, int64_t* parent,
                int64_t* parent_len, const uint8_t* owned) {
  if (!g.last_valid) fail(SSB_EINVAL, "no BFS result on this graph");
  cudaStream_t s = g.sc.s;
  const int64_t n = g.n;
  if (n == 0) {
    if (parent_len) *parent_len = 0;
    return;
  }
  // whole results of shallow BFS (levels fit a byte) of graphs worth it take
  // the narrow wire format (SSB_WIRE=0: the direct int64 path below)
  const bool whole = owned == nullptr;
  if (whole && g.last_iterations <= 254 && n >= env_int("SSB_WIRE_MIN", 1 << 16) &&
      env_int("SSB_WIRE", 1) != 0) {
    fetch_wire(g, want_parents, dist, parent, parent_len);
    return;
  }
  BitRegions R = bit_regions(g, 0);  // visited is the first region for both engines
  const bool sel = g.last_variant == SSB_SELMAX;
  // Pinned (page-locked) host buffers are written by the kernels directly over
  // PCIe; pageable ones go through a persistent device staging buffer.
  auto direct = [](int64_t* h) -> int64_t* {
    if (!h) return nullptr;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return at.type == cudaMemoryTypeHost ? static_cast<int64_t*>(at.devicePointer) : nullptr;
  };
  int64_t* dd = direct(dist);
  int64_t* dp = want_parents ? direct(parent) : nullptr;
  if ((dist && !dd) || (want_parents && parent && !dp)) g.stage.ensure(size_t(2 * n));
  int64_t* d_out = dd ? dd : (dist ? g.stage.p : nullptr);
  int64_t* p_out = dp ? dp : (want_parents && parent ? g.stage.p + n : nullptr);
  const bool partial = !whole;  // a shard: keep the caller's other rows
  if (partial && dist && !dd)
    SSB_CUDA(cudaMemcpyAsync(d_out, dist, 8 * n, cudaMemcpyHostToDevice, s));
  if (partial && p_out && !dp)
    SSB_CUDA(cudaMemcpyAsync(p_out, parent, 8 * n, cudaMemcpyHostToDevice, s));
  unpermute_kernel<<<grid_for(n), 256, 0, s>>>(R.visited, g.level.p, g.parent.p, g.perm.p,
                                               g.inv_perm.p, n, sel && p_out != nullptr, d_out,
                                               p_out, owned);
  SSB_CUDA(cudaGetLastError());
  int64_t plen = 0;
  if (want_parents && !sel) {
    g.flag.ensure(1);
    SSB_CUDA(cudaMemsetAsync(g.flag.p, 0, 4, s));
    if (p_out)
      dp_parent_kernel<int64_t><<<grid_for(n), 256, 0, s>>>(g.col.p, g.cs.p, g.cl.p, g.C, R.visited,
                                                   g.level.p, g.perm.p, g.inv_perm.p, n, p_out,
                                                   g.flag.p, owned);
    SSB_CUDA(cudaGetLastError());
    int hbad = 0;
    SSB_CUDA(cudaMemcpyAsync(&hbad, g.flag.p, 4, cudaMemcpyDeviceToHost, s));
    g.sc.sync();
    if (hbad) fail(SSB_EINVAL, "inconsistent distances: a reached vertex has no neighbor one level closer");
  }
  if (want_parents) plen = n;
  if (dist && !dd) SSB_CUDA(cudaMemcpyAsync(dist, d_out, 8 * n, cudaMemcpyDeviceToHost, s));
  if (parent && plen && !dp)
    SSB_CUDA(cudaMemcpyAsync(parent, p_out, 8 * n, cudaMemcpyDeviceToHost, s));
  g.sc.sync();
  if (parent_len) *parent_len = plen;
}

// ---- chunk-range shards of a multi-GPU BFS ---------------
// Each rank owns chunks [cb, ce) and the replicated 1-bit frontier. One
// iteration = shard_step (this rank's sweep, its owned frontier words copied
// out) -> the caller all-gathers every rank's words -> shard_exchange (the
// full frontier installed, the summary rebuilt, |F| made global).
constexpr int kFrontRing = 64;  // iterations whose |F| the host can still query
struct ShardState {
  Run32 r;
  ssb_bfs_options o;
  std::vector<ssb_iter_stats> stats;
  DevBuf<uint8_t> owned;  // per chunk: owned by this rank (result fetch)
  // asynchronous stepping (no host round trip per iteration)
  DevBuf<int64_t> carry;                    // {|F|, active tasks, retired chunks, spare}
  std::vector<std::unique_ptr<DevBuf<int64_t>>> recs;  // per-iteration records, 1024 per block
  int64_t* hfront = nullptr;                // pinned ring: global |F_k|
  cudaEvent_t ev[kFrontRing] = {};
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  bool async = false;
  ~ShardState() {
    if (hfront) cudaFreeHost(hfront);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
  }
  int64_t* rec_slot(int64_t k) {  // device record of iteration k (1-based)
    const size_t blk = size_t((k - 1) / 1024);
    while (recs.size() <= blk) recs.emplace_back(new DevBuf<int64_t>(size_t(1024) * kStatW));
    return recs[blk]->p + ((k - 1) % 1024) * kStatW;
  }
};

// device mask of the owned chunks of a segment list
void owned_mask(const ssb_graph& g, const std::vector<int64_t>& segs, DevBuf<uint8_t>& out) {
  std::vector<uint8_t> h(size_t(std::max<int64_t>(g.n_chunks, 1)), 0);
  for (size_t q = 0; q + 1 < segs.size(); q += 2)
    for (int64_t c = segs[q]; c < segs[q + 1]; ++c) h[size_t(c)] = 1;
  out.alloc(h.size());
  SSB_CUDA(cudaMemcpy(out.p, h.data(), h.size(), cudaMemcpyHostToDevice));
}

void shard_begin(ssb_graph& g, int64_t root, const ssb_bfs_options& o, int64_t cb, int64_t ce) {
  if (g.C != 32) fail(SSB_EINVAL, "sharded BFS needs the C = 32 layout");
  if (o.variant < 0 || o.variant > 3) fail(SSB_EINVAL, "bad variant");
  if (cb < 0 || ce > g.n_chunks || cb > ce) fail(SSB_EINVAL, "chunk range out of bounds");
  if (!g.holds(cb, ce)) fail(SSB_EINVAL, "owned chunks outside the segments this handle holds");
  if (root < 0 || root >= g.n)
    fail(SSB_ERANGE, "root " + std::to_string(root) + " outside [0, " + std::to_string(g.n) + ")");
  int32_t root_pos = 0;
  SSB_CUDA(cudaMemcpy(&root_pos, g.inv_perm.p + root, 4, cudaMemcpyDeviceToHost));
  const int32_t root_code =
      (o.variant == SSB_SELMAX && o.selmax_compat) ? int32_t(root) : root_pos;
  auto st = std::make_shared<ShardState>();
  g.last_kernel_ms = 0;
  g.last_launches = 0;
  g.last_swept = 0;
  // (no hashed summary: the exchange builds the block summary from the
  // gathered words)
  st->r = prepare32(g, root_pos, root_code, o, {cb, ce}, nullptr, nullptr, false, false);
  st->r.a.retire_once = 0;  // the exchange counts and summarises frontier words
  st->r.stepping = true;
  owned_mask(g, st->r.segs, st->owned);
  st->o = o;
  g.shard = st;
  g.last_root = root;
  g.last_variant = o.variant;
  g.last_compat = o.selmax_compat;
  g.last_valid = false;
}

void shard_step(ssb_graph& g, ssb_iter_stats* local, uint32_t* owned_words) {
  auto st = std::static_pointer_cast<ShardState>(g.shard);
  if (!st) fail(SSB_EINVAL, "no sharded BFS in progress (ssb_bfs_shard_begin)");
  Run32& r = st->r;
  const int64_t k = r.k;
  std::vector<ssb_iter_stats> one;
  bool conv = false;
  launch32(g, r, k + 1, one, conv);
  if (local) *local = one.front();
  st->stats.push_back(one.front());
  const uint32_t* Fn = (k & 1) ? r.a.F1 : r.a.F0;
  const int64_t cb = r.segs[0], ce = r.segs[1];
  if (owned_words && ce > cb)
    SSB_CUDA(cudaMemcpyAsync(owned_words, Fn + cb, 4 * (ce - cb), cudaMemcpyDeviceToDevice,
                             g.sc.s));
  g.sc.sync();
}

void shard_exchange(ssb_graph& g, const uint32_t* frontier_words, int64_t newly_total) {
  auto st = std::static_pointer_cast<ShardState>(g.shard);
  if (!st) fail(SSB_EINVAL, "no sharded BFS in progress (ssb_bfs_shard_begin)");
  Run32& r = st->r;
  const int64_t k = r.k - 1;  // the iteration just stepped
  cudaStream_t s = g.sc.s;
  uint32_t* Fn = (k & 1) ? r.a.F1 : r.a.F0;
  if (!frontier_words) fail(SSB_EINVAL, "frontier_words is NULL");
  SSB_CUDA(cudaMemcpyAsync(Fn, frontier_words, 4 * g.n_chunks, cudaMemcpyDeviceToDevice, s));
  if (r.G.SW > 0) {
    uint32_t* Sn = (k % 3) == 0 ? r.a.S0 : ((k % 3) == 1 ? r.a.S1 : r.a.S2);
    summary_from_words_kernel<<<grid_for(r.G.SW), 256, 0, s>>>(Fn, r.G.PW, g.n_chunks, Sn, r.G.SW,
                                                               r.G.gshift);
    SSB_CUDA(cudaGetLastError());
    g.last_launches += 1;
  }
  r.a.front_in = newly_total;
  g.sc.sync();
  g.last_iterations = int64_t(st->stats.size());
  g.last_valid = true;  // results of the owned rows can be fetched at any point
}

// ---- asynchronous form: no host synchronisation inside the BFS -------------
// step_async (sweep k; record k and the owned words copied on the stream) ->
// the caller's all-gather on the SAME stream (ssb_graph_stream) ->
// exchange_async (install, summary, global |F_k| counted on the device into
// the carry the next sweep reads, and copied to a pinned slot). The host only
// polls |F_{k-1}| (ssb_bfs_shard_front) while iteration k is already queued,
// and takes the counters once at the end (ssb_bfs_shard_finish).
void shard_begin_async(ssb_graph& g, int64_t root, const ssb_bfs_options& o, int64_t cb, int64_t ce) {
  shard_begin(g, root, o, cb, ce);
  auto st = std::static_pointer_cast<ShardState>(g.shard);
  st->async = true;
  st->carry.alloc(4);
  if (!st->hfront) SSB_CUDA(cudaHostAlloc(&st->hfront, sizeof(int64_t) * kFrontRing, cudaHostAllocDefault));
  for (auto& e : st->ev) SSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  SSB_CUDA(cudaEventCreate(&st->t0));
  SSB_CUDA(cudaEventCreate(&st->t1));
  const int64_t init[4] = {1, st->r.a.n_tasks, 0, 0};  // F_0 = {root}
  SSB_CUDA(cudaMemcpyAsync(st->carry.p, init, sizeof init, cudaMemcpyHostToDevice, g.sc.s));
  st->r.a.carry = st->carry.p;
  SSB_CUDA(cudaStreamSynchronize(g.sc.s));  // init lives on this stack frame
  SSB_CUDA(cudaEventRecord(st->t0, g.sc.s));
}

void shard_step_async(ssb_graph& g, uint32_t* owned_words) {
  auto st = std::static_pointer_cast<ShardState>(g.shard);
  if (!st || !st->async) fail(SSB_EINVAL, "no asynchronous sharded BFS in progress (ssb_bfs_shard_begin_async)");
  Run32& r = st->r;
  cudaStream_t s = g.sc.s;
  Args32& a = r.a;
  const int64_t k = r.k;
  a.k_begin = int32_t(k);
  a.k_end = int32_t(k + 1);
  if (!r.zeroed) {
    SSB_CUDA(cudaMemsetAsync(g.dstats.p, 0, size_t(kStatW) * 8, s));
    SSB_CUDA(cudaMemsetAsync(g.dctrl.p, 0, g.dctrl.bytes(), s));
  }
  r.zeroed = false;
  void* params[] = {&a, &r.reset};  // (reset.active = 0: begin_async ran the reset kernel)
  SSB_CUDA(cudaLaunchCooperativeKernel((const void*)bfs32_fn(r.sel, r.G.S, r.hashed), dim3(r.grid), dim3(kThreads),
                                       params, r.G.smem, s));
  SSB_CUDA(cudaGetLastError());
  g.last_launches += 1;
  SSB_CUDA(cudaMemcpyAsync(st->rec_slot(k), g.dstats.p, size_t(kStatW) * 8, cudaMemcpyDeviceToDevice, s));
  const uint32_t* Fn = (k & 1) ? a.F1 : a.F0;
  const int64_t cb = r.segs[0], ce = r.segs[1];
  if (owned_words && ce > cb)
    SSB_CUDA(cudaMemcpyAsync(owned_words, Fn + cb, 4 * (ce - cb), cudaMemcpyDeviceToDevice, s));
  r.k = k + 1;
}

void shard_exchange_async(ssb_graph& g, const uint32_t* frontier_words) {
  auto st = std::static_pointer_cast<ShardState>(g.shard);
  if (!st || !st->async) fail(SSB_EINVAL, "no asynchronous sharded BFS in progress (ssb_bfs_shard_begin_async)");
  if (!frontier_words) fail(SSB_EINVAL, "frontier_words is NULL");
  Run32& r = st->r;
  const int64_t k = r.k - 1;  // the iteration just stepped
  cudaStream_t s = g.sc.s;
  uint32_t* Fn = (k & 1) ? r.a.F1 : r.a.F0;
  SSB_CUDA(cudaMemcpyAsync(Fn, frontier_words, 4 * g.n_chunks, cudaMemcpyDeviceToDevice, s));
  if (r.G.SW > 0) {
    uint32_t* Sn = (k % 3) == 0 ? r.a.S0 : ((k % 3) == 1 ? r.a.S1 : r.a.S2);
    summary_from_words_kernel<<<grid_for(r.G.SW), 256, 0, s>>>(Fn, r.G.PW, g.n_chunks, Sn, r.G.SW,
                                                               r.G.gshift);
    SSB_CUDA(cudaGetLastError());
    g.last_launches += 1;
  }
  SSB_CUDA(cudaMemsetAsync(st->carry.p, 0, 8, s));
  front_count_kernel<<<grid_for(g.n_chunks), 256, 0, s>>>(Fn, g.cl.p, g.n_chunks, st->carry.p);
  SSB_CUDA(cudaGetLastError());
  g.last_launches += 1;
  const int slot = int(k % kFrontRing);
  SSB_CUDA(cudaMemcpyAsync(st->hfront + slot, st->carry.p, 8, cudaMemcpyDeviceToHost, s));
  SSB_CUDA(cudaEventRecord(st->ev[slot], s));
}

int64_t shard_front(ssb_graph& g, int64_t k) {
  auto st = std::static_pointer_cast<ShardState>(g.shard);
  if (!st || !st->async) fail(SSB_EINVAL, "no asynchronous sharded BFS in progress (ssb_bfs_shard_begin_async)");
  if (k < 1 || k >= st->r.k || k < st->r.k - kFrontRing)
    fail(SSB_EINVAL, "iteration " + std::to_string(k) + " not exchanged or no longer held");
  const int slot = int(k % kFrontRing);
  SSB_CUDA(cudaEventSynchronize(st->ev[slot]));
  return st->hfront[slot];
}

// The BFS took `iterations` iterations (the caller saw |F_iterations| = 0 or
// hit its cap): this rank's per-iteration counters (local to its chunks —
// sum them over ranks) and the device time since begin.
void shard_finish(ssb_graph& g, int64_t iterations, ssb_iter_stats* out, int64_t cap, double* device_ms) {
  auto st = std::static_pointer_cast<ShardState>(g.shard);
  if (!st || !st->async) fail(SSB_EINVAL, "no asynchronous sharded BFS in progress (ssb_bfs_shard_begin_async)");
  Run32& r = st->r;
  if (iterations < 0 || iterations >= r.k) fail(SSB_EINVAL, "more iterations than were stepped");
  cudaStream_t s = g.sc.s;
  SSB_CUDA(cudaEventRecord(st->t1, s));
  SSB_CUDA(cudaStreamSynchronize(s));
  std::vector<int64_t> rec(size_t(iterations) * kStatW);
  for (int64_t k = 1; k <= iterations; ++k)
    SSB_CUDA(cudaMemcpy(rec.data() + (k - 1) * kStatW, st->rec_slot(k), size_t(kStatW) * 8,
                        cudaMemcpyDeviceToHost));
  std::vector<ssb_iter_stats> stats;
  collect_stats(rec, 1, iterations, stats);
  g.last_swept = 0;
  for (int64_t i = 0; i < iterations; ++i) {
    stats[size_t(i)].chunks_processed += g.plan.empty_chunks - (r.z_skip ? 1 : 0);
    stats[size_t(i)].chunks_skipped += r.z_skip ? 1 : 0;
    g.last_swept += rec[size_t(i) * kStatW + 6];
  }
  for (int64_t i = 0; i < std::min<int64_t>(cap, iterations); ++i) out[i] = stats[size_t(i)];
  st->stats = stats;
  float ms = 0;
  SSB_CUDA(cudaEventElapsedTime(&ms, st->t0, st->t1));
  if (device_ms) *device_ms = ms;
  g.last_kernel_ms = ms;
  g.last_iterations = iterations;
  g.last_valid = true;
}

void shard_fetch(ssb_graph& g, int want_parents, int64_t* dist, int64_t* parent) {
  auto st = std::static_pointer_cast<ShardState>(g.shard);
  if (!st) fail(SSB_EINVAL, "no sharded BFS (ssb_bfs_shard_begin)");
  g.last_valid = true;
  fetch_rows(g, want_parents, dist, parent, nullptr, st->owned.p);
}

// ---- fused multi-GPU chunk-range BFS (frontier exchange inside the kernel) ----

void p2p_window(ssb_graph& g, void* ipc_handle, int64_t* bytes) {
  WinGeom wg;
  uint32_t* w = p2p_window_alloc(g, wg);
  if (bytes) *bytes = int64_t(g.p2p_win.bytes());
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    SSB_CUDA(cudaIpcGetMemHandle(&h, w));
    std::memcpy(ipc_handle, &h, sizeof h);
  }
}

std::vector<int64_t> check_segments(ssb_graph& g, const int64_t* bounds, int64_t nseg) {
  std::vector<int64_t> segs = normalize_segments(bounds, nseg, g.n_chunks);
  if (int64_t(segs.size() / 2) > kMaxSeg) fail(SSB_EINVAL, "at most 8 owned segments per rank");
  if (!g.holds_segments(segs)) fail(SSB_EINVAL, "owned chunks outside the segments this handle holds");
  return segs;
}

// Maps every peer's window (CUDA IPC; peer access over NVLink). Collective in
// spirit: every rank attaches before any rank runs a BFS, and the windows'
// arrival counters start at zero together.
void p2p_attach(ssb_graph& g, int rank, int world, const void* handles, const int64_t* bounds,
                int64_t nseg) {
  if (world < 1 || world > kMaxRanks) fail(SSB_EINVAL, "world must be in [1, 8]");
  if (rank < 0 || rank >= world) fail(SSB_EINVAL, "rank outside [0, world)");
  const std::vector<int64_t> segs = check_segments(g, bounds, nseg);
  auto h = std::make_shared<P2PHost>();
  uint32_t* mine = p2p_window_alloc(g, h->wg);
  SSB_CUDA(cudaMemset(mine, 0, g.p2p_win.bytes()));
  h->rank = rank;
  h->world = world;
  h->segs = segs;
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      h->win[r] = mine;
      continue;
    }
    if (!handles) fail(SSB_EINVAL, "ipc_handles is NULL");
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, static_cast<const char*>(handles) + size_t(r) * sizeof ih, sizeof ih);
    void* p = nullptr;
    SSB_CUDA(cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess));
    h->opened.push_back(p);
    h->win[r] = static_cast<uint32_t*>(p);
  }
  g.p2p = h;
}

// Kernel-side view of one rank's peer table.
P2PArgs p2p_args(const ssb_graph& g, const P2PHost& h, const Geometry& G, unsigned long long arrivals) {
  P2PArgs x{};
  for (int r = 0; r < h.world; ++r) x.win[r] = h.win[r];
  for (int i = 0; i < 2; ++i) x.offF[i] = h.wg.offF[i];
  for (int i = 0; i < 3; ++i) x.offS[i] = h.wg.offS[i];
  x.offSlots = h.wg.offSlots;
  x.offArrive = h.wg.offArrive;
  x.gen_base = h.gen;
  x.timeout_ns = (unsigned long long)std::max(0, env_int("SSB_P2P_TIMEOUT_S", 60)) * 1000000000ull;
  x.arrivals = arrivals;
  x.rank = h.rank;
  x.world = h.world;
  x.nseg = int32_t(h.segs.size() / 2);
  for (int q = 0; q < x.nseg; ++q) {
    const int64_t cb = h.segs[size_t(2 * q)], ce = h.segs[size_t(2 * q + 1)];
    x.wseg[2 * q] = int32_t(cb);
    x.wseg[2 * q + 1] = int32_t(ce);
    // summary words holding bits of the segment's chunks
    x.sseg[2 * q] = x.sseg[2 * q + 1] = 0;
    const int64_t lo = std::max<int64_t>(cb, G.PW);
    if (G.SW > 0 && ce > lo) {
      x.sseg[2 * q] = int32_t(((lo - G.PW) >> G.gshift) >> 5);
      x.sseg[2 * q + 1] = int32_t((((ce - 1 - G.PW) >> G.gshift) >> 5) + 1);
    }
  }
  (void)g;
  return x;
}

const void* bfs32p_fn(bool sel, int S, bool group) {
  if (group) {
    if (S == 6) return sel ? (const void*)bfs32p_kernel<true, 6> : (const void*)bfs32p_kernel<false, 6>;
    return sel ? (const void*)bfs32p_kernel<true, 8> : (const void*)bfs32p_kernel<false, 8>;
  }
  if (S == 6) return sel ? (const void*)bfs32x_kernel<true, 6> : (const void*)bfs32x_kernel<false, 6>;
  return sel ? (const void*)bfs32x_kernel<true, 8> : (const void*)bfs32x_kernel<false, 8>;
}

// One BFS over chunk-range shards with the exchange fused into the kernel.
// n_local = 1: this process's rank of a multi-GPU job (peers attached with
// p2p_attach); n_local > 1: all ranks emulated on this device in ONE
// cooperative launch (ranges[2i], ranges[2i+1] = rank i's chunk range).
// stats: per iteration, counters summed over the local shards.
int bfs_p2p(ssb_graph* const* gs, int n_local, const int64_t* bounds, const int64_t* seg_counts,
            int64_t root, const ssb_bfs_options& o, ssb_iter_stats* stats, int64_t stats_cap,
            int64_t* iterations, double* device_ms) {
  if (n_local < 1 || n_local > kMaxVRanks) fail(SSB_EINVAL, "local shards must be in [1, 8]");
  if (o.variant < 0 || o.variant > 3) fail(SSB_EINVAL, "bad variant");
  ssb_graph& g0 = *gs[0];
  for (int i = 0; i < n_local; ++i) {
    ssb_graph& g = *gs[i];
    if (g.C != 32) fail(SSB_EINVAL, "the fused multi-GPU BFS needs the C = 32 layout");
    if (g.n != g0.n || g.n_chunks != g0.n_chunks || g.total_cells != g0.total_cells)
      fail(SSB_EINVAL, "shards hold different layouts");
  }
  if (root < 0 || root >= g0.n)
    fail(SSB_ERANGE, "root " + std::to_string(root) + " outside [0, " + std::to_string(g0.n) + ")");
  if (n_local > 1) {
    // emulated group: the windows are plain device memory of this device
    std::vector<uint32_t*> wins(static_cast<size_t>(n_local));
    std::vector<std::shared_ptr<P2PHost>> hs(static_cast<size_t>(n_local));
    std::vector<std::vector<int64_t>> segs(static_cast<size_t>(n_local));
    int64_t at = 0;  // bounds offset of rank i's segments
    for (int i = 0; i < n_local; ++i) {
      const int64_t ns = seg_counts ? seg_counts[i] : 1;
      segs[size_t(i)] = check_segments(*gs[i], bounds + 2 * at, ns);
      at += ns;
      auto* prev = static_cast<P2PHost*>(gs[i]->p2p.get());
      hs[size_t(i)] = std::make_shared<P2PHost>();
      wins[size_t(i)] = p2p_window_alloc(*gs[i], hs[size_t(i)]->wg);
      hs[size_t(i)]->gen = prev && prev->world == n_local && prev->rank == i ? prev->gen : ~0ull;
    }
    // keep the barrier generation count only for the same group of windows
    for (int i = 0; i < n_local; ++i) {
      auto* prev = static_cast<P2PHost*>(gs[i]->p2p.get());
      for (int r = 0; prev && r < n_local; ++r)
        if (prev->win[r] != wins[size_t(r)]) hs[size_t(i)]->gen = ~0ull;
    }
    unsigned long long gen = hs[0]->gen;
    for (int i = 0; i < n_local; ++i)
      if (hs[size_t(i)]->gen != gen) gen = ~0ull;
    for (int i = 0; i < n_local; ++i) {
      P2PHost& h = *hs[size_t(i)];
      h.rank = i;
      h.world = n_local;
      h.segs = segs[size_t(i)];
      for (int r = 0; r < n_local; ++r) h.win[r] = wins[size_t(r)];
      if (gen == ~0ull) {  // a new group: restart the barrier counters together
        SSB_CUDA(cudaMemset(wins[size_t(i)], 0, gs[i]->p2p_win.bytes()));
        h.gen = 0;
      }
      gs[i]->p2p = hs[size_t(i)];
    }
  }
  std::vector<P2PHost*> H(static_cast<size_t>(n_local));
  for (int i = 0; i < n_local; ++i) {
    H[size_t(i)] = static_cast<P2PHost*>(gs[i]->p2p.get());
    if (!H[size_t(i)]) fail(SSB_EINVAL, "no peer windows attached (ssb_p2p_attach)");
  }
  const int world = H[0]->world;
  int dev = 0;
  SSB_CUDA(cudaGetDevice(&dev));

  int32_t root_pos = 0;
  SSB_CUDA(cudaMemcpy(&root_pos, g0.inv_perm.p + root, 4, cudaMemcpyDeviceToHost));
  const int32_t root_code = (o.variant == SSB_SELMAX && o.selmax_compat) ? int32_t(root) : root_pos;
  const int64_t cap = o.max_iterations > 0 ? o.max_iterations : g0.n + 1;

  std::vector<Run32> rs;
  rs.reserve(size_t(n_local));
  for (int i = 0; i < n_local; ++i) {
    ssb_graph& g = *gs[i];
    g.last_kernel_ms = 0;
    g.last_launches = 0;
    g.last_swept = 0;
    g.last_valid = false;
    rs.push_back(prepare32(g, root_pos, root_code, o, H[size_t(i)]->segs, H[size_t(i)]));
  }
  const Geometry G = rs[0].G;
  const bool sel = rs[0].sel;
  const void* fn = bfs32p_fn(sel, G.S, n_local > 1);
  {
    configure32(fn, G.smem);
    int per_sm = 0;
    SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, G.smem));
    if (per_sm < 1) fail(SSB_ECUDA, "bfs32p kernel does not fit on an SM");
  }
  // every rank runs the same CTA count (same GPU model): arrivals = world x nvb
  const int nvb = num_sms() / n_local;
  const int grid = nvb * n_local;
  for (int i = 0; i < n_local; ++i) gs[i]->sc.sync();  // resets done before anyone stores

  cudaStream_t s = g0.sc.s;
  cudaEvent_t t0, t1;
  SSB_CUDA(cudaEventCreate(&t0));
  SSB_CUDA(cudaEventCreate(&t1));
  SSB_CUDA(cudaEventRecord(t0, s));
  std::vector<std::vector<ssb_iter_stats>> st(static_cast<size_t>(n_local));
  std::vector<std::vector<int64_t>> rec(size_t(n_local), std::vector<int64_t>(size_t(kItersPerLaunch) * kStatW));
  int64_t k = 1;
  bool conv = false;
  double kms_total = 0;
  while (!conv && k <= cap) {
    const int64_t kend = std::min<int64_t>(cap + 1, k + kItersPerLaunch);
    GroupArgs ga{};
    ga.nvb = nvb;
    for (int i = 0; i < n_local; ++i) {
      Run32& r = rs[size_t(i)];
      if (!r.zeroed) {
        SSB_CUDA(cudaMemsetAsync(gs[i]->dstats.p, 0, gs[i]->dstats.bytes(), s));
        SSB_CUDA(cudaMemsetAsync(gs[i]->dctrl.p, 0, gs[i]->dctrl.bytes(), s));
      }
      r.zeroed = false;
      r.a.k_begin = int32_t(k);
      r.a.k_end = int32_t(kend);
      ga.a[i] = r.a;
      ga.x[i] = p2p_args(*gs[i], *H[size_t(i)], G, (unsigned long long)world * (unsigned long long)nvb);
    }
    static int* trace_buf = nullptr;  // debug (SSB_TRACE): per-rank progress words in mapped host memory
    if (std::getenv("SSB_TRACE")) {
      if (!trace_buf) SSB_CUDA(cudaHostAlloc(&trace_buf, 4096, cudaHostAllocMapped));
      std::memset(trace_buf, 0, 4096);
      for (int i = 0; i < n_local; ++i) {
        int* d = nullptr;
        SSB_CUDA(cudaHostGetDevicePointer(&d, trace_buf + 16 * i, 0));
        ga.a[i].trace = d;
      }
    }
    void* params_group[] = {&ga};
    void* params_rank[] = {&ga.a[0], &ga.x[0]};
    SSB_CUDA(cudaEventRecord(g0.sc.e0, s));
    SSB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads),
                                         n_local > 1 ? params_group : params_rank, G.smem, s));
    SSB_CUDA(cudaGetLastError());
    SSB_CUDA(cudaEventRecord(g0.sc.e1, s));
    if (ga.a[0].trace) {  // debug: poll progress instead of blocking forever
      for (int spin = 0; cudaEventQuery(g0.sc.e1) == cudaErrorNotReady; ++spin) {
        if (spin % 1000 == 999) {
          for (int i = 0; i < n_local; ++i)
            fprintf(stderr, "[ssb p2p trace] rank %d k=%d phase=%d arrived=%d front=%d\n", i,
                    trace_buf[16 * i], trace_buf[16 * i + 1], trace_buf[16 * i + 2], trace_buf[16 * i + 3]);
        }
        if (spin > 10000) {
          fprintf(stderr, "[ssb p2p trace] giving up\n");
          std::abort();
        }
        usleep(1000);
      }
    }
    for (int i = 0; i < n_local; ++i)
      SSB_CUDA(cudaMemcpyAsync(rec[size_t(i)].data(), gs[i]->dstats.p, size_t(kend - k) * kStatW * 8,
                               cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaEventRecord(g0.sc.e_end, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    float kms = 0;
    SSB_CUDA(cudaEventElapsedTime(&kms, g0.sc.e0, g0.sc.e1));
    kms_total += kms;
    // iterations run: up to the first with global |newly| = 0 (slot 7)
    int64_t ran = 0;
    for (int64_t j = 0; j < kend - k; ++j) {
      ++ran;
      if (rec[0][size_t(j) * kStatW + 7] == 0) {
        conv = true;
        break;
      }
    }
    for (int i = 0; i < n_local; ++i) {
      ssb_graph& g = *gs[i];
      Run32& r = rs[size_t(i)];
      const size_t before = st[size_t(i)].size();
      collect_stats(rec[size_t(i)], k, ran, st[size_t(i)]);
      for (int64_t j = 0; j < ran; ++j) g.last_swept += rec[size_t(i)][size_t(j) * kStatW + 6];
      for (size_t j = before; j < st[size_t(i)].size(); ++j) {
        st[size_t(i)][j].chunks_processed += g.plan.empty_chunks - (r.z_skip ? 1 : 0);
        st[size_t(i)][j].chunks_skipped += r.z_skip ? 1 : 0;
      }
      H[size_t(i)]->gen += static_cast<unsigned long long>(1 + ran);
      if (!conv) {
        std::vector<uint32_t> outs(static_cast<size_t>(ran));
        std::vector<unsigned long long> gones(static_cast<size_t>(ran));
        SSB_CUDA(cudaMemcpy(outs.data(), r.task_out, 4 * ran, cudaMemcpyDeviceToHost));
        SSB_CUDA(cudaMemcpy(gones.data(), r.gone, 8 * ran, cudaMemcpyDeviceToHost));
        r.a.n_tasks = int32_t(outs.back());
        for (auto v : gones) r.a.gone_base += v;
        r.a.front_in = rec[size_t(i)][size_t(ran - 1) * kStatW + 7];
      }
    }
    k += ran;
  }
  SSB_CUDA(cudaEventRecord(t1, s));
  SSB_CUDA(cudaEventSynchronize(t1));
  float ms = 0;
  SSB_CUDA(cudaEventElapsedTime(&ms, t0, g0.sc.e_end));
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  const int64_t iters = int64_t(st[0].size());
  for (int i = 0; i < n_local; ++i) {
    ssb_graph& g = *gs[i];
    g.last_kernel_ms = kms_total;
    g.last_launches = 1 + (iters + kItersPerLaunch - 1) / kItersPerLaunch;  // reset + BFS launches
    g.last_root = root;
    g.last_variant = o.variant;
    g.last_compat = o.selmax_compat;
    g.last_iterations = iters;
    g.last_valid = true;
    auto ss = std::make_shared<ShardState>();
    ss->r = rs[size_t(i)];
    owned_mask(g, ss->r.segs, ss->owned);
    ss->o = o;
    ss->stats = st[size_t(i)];
    g.shard = ss;  // results of the owned rows: ssb_bfs_shard_fetch
  }
  if (device_ms) *device_ms = ms;
  if (iterations) *iterations = iters;
  if (stats) {
    for (int64_t j = 0; j < std::min<int64_t>(stats_cap, iters); ++j) {
      ssb_iter_stats a = st[0][size_t(j)];
      for (int i = 1; i < n_local; ++i) {
        const ssb_iter_stats& b = st[size_t(i)][size_t(j)];
        a.chunks_processed += b.chunks_processed;
        a.chunks_skipped += b.chunks_skipped;
        a.subchunks_processed += b.subchunks_processed;
        a.columns_processed += b.columns_processed;
        a.frontier_size += b.frontier_size;
      }
      stats[j] = a;
    }
  }
  return conv ? SSB_OK : SSB_ECAP;
}

int64_t bfs_edges_traversed(ssb_graph& g) {
  if (!g.last_valid) fail(SSB_EINVAL, "no BFS result on this graph");
  cudaStream_t s = g.sc.s;
  BitRegions R = bit_regions(g, 0);
  DevBuf<unsigned long long> acc(1);
  SSB_CUDA(cudaMemsetAsync(acc.p, 0, 8, s));
  reached_degree_kernel<<<grid_for(g.n), 256, 0, s>>>(R.visited, g.deg.p, g.n, acc.p);
  SSB_CUDA(cudaGetLastError());
  unsigned long long v = 0;
  SSB_CUDA(cudaMemcpyAsync(&v, acc.p, 8, cudaMemcpyDeviceToHost, s));
  g.sc.sync();
  return int64_t(v / 2);
}


// ---- single-process multi-device context (SURVEY.md §8(b) ssb_ctx_create) ----
// One host thread drives every rank of a sharded layout:
//  * distinct devices: peer access enabled between every pair; each rank's
//    frontier window is a plain device pointer the peers store into over
//    NVLink (no IPC), and every BFS runs one cooperative launch per rank —
//    the same per-rank path as a multi-process job (bfs_p2p, n_local = 1),
//    each launched from its own host thread because the ranks meet at an
//    in-kernel barrier;
//  * one device listed several times: the ranks run as ONE cooperative
//    launch on it (the emulated group, bfs_p2p n_local > 1).

// partition_chunks + the snake deal of partition_segments (sharding.py):
// k·W contiguous pieces of near-equal C·cl + 1 weight, dealt 0..W-1, W-1..0, ...
std::vector<std::vector<int64_t>> partition_segments_host(const std::vector<int32_t>& cl, int64_t C, int world,
                                                          int k) {
  const int64_t nc = int64_t(cl.size());
  const int pieces = world * k;
  std::vector<int64_t> cum(size_t(nc) + 1, 0);
  for (int64_t i = 0; i < nc; ++i) cum[size_t(i + 1)] = cum[size_t(i)] + C * int64_t(cl[size_t(i)]) + 1;
  std::vector<int64_t> bounds{0};
  for (int r = 1; r < pieces; ++r) {
    const int64_t target = cum.back() * r / pieces;
    int64_t b = int64_t(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
    b = std::min(std::max(b, bounds.back()), nc);
    bounds.push_back(b);
  }
  bounds.push_back(nc);
  std::vector<std::vector<int64_t>> out(static_cast<size_t>(world));
  for (int j = 0; j < pieces; ++j) {
    const int rnd = j / world, pos = j % world;
    const int r = rnd % 2 == 0 ? pos : world - 1 - pos;
    out[size_t(r)].push_back(bounds[size_t(j)]);
    out[size_t(r)].push_back(bounds[size_t(j + 1)]);
  }
  return out;
}

namespace {
struct DeviceGuard {  // restores the caller's current device
  int prev = 0;
  DeviceGuard() { SSB_CUDA(cudaGetDevice(&prev)); }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// the normalised edge set on `dev` (a device-to-device copy of e's keys)
std::unique_ptr<ssb_edges> edges_on(const ssb_edges& e, int src_dev, int dev) {
  SSB_CUDA(cudaSetDevice(dev));
  auto c = std::make_unique<ssb_edges>();
  c->n = e.n;
  c->m = e.m;
  c->bits = e.bits;
  c->keys.alloc(e.keys.n);
  SSB_CUDA(cudaStreamSynchronize(e.sc.s));
  if (e.keys.n) SSB_CUDA(cudaMemcpyPeer(c->keys.p, dev, e.keys.p, src_dev, e.keys.bytes()));
  return c;
}
}  // namespace

ssb_ctx* ctx_create(int n_ranks, const int* device_ids) {
  if (n_ranks < 1 || n_ranks > kMaxRanks) fail(SSB_EINVAL, "ranks must be in [1, 8]");
  int n_dev = 0;
  SSB_CUDA(cudaGetDeviceCount(&n_dev));
  auto c = std::make_unique<ssb_ctx>();
  for (int i = 0; i < n_ranks; ++i) {
    const int d = device_ids ? device_ids[i] : i;
    if (d < 0 || d >= n_dev) fail(SSB_EINVAL, "device id " + std::to_string(d) + " not present");
    c->devs.push_back(d);
  }
  bool all_same = true, all_distinct = true;
  for (int i = 0; i < n_ranks; ++i)
    for (int j = 0; j < n_ranks; ++j)
      if (i != j) {
        all_same = all_same && c->devs[size_t(i)] == c->devs[size_t(j)];
        all_distinct = all_distinct && c->devs[size_t(i)] != c->devs[size_t(j)];
      }
  if (!all_same && !all_distinct)
    fail(SSB_EINVAL, "ranks must be on distinct devices, or all on one device (emulated group)");
  c->group = n_ranks > 1 && all_same;
  if (n_ranks > 1 && all_distinct) {
    DeviceGuard guard;
    for (int i = 0; i < n_ranks; ++i)
      for (int j = 0; j < n_ranks; ++j) {
        if (i == j) continue;
        int ok = 0;
        SSB_CUDA(cudaDeviceCanAccessPeer(&ok, c->devs[size_t(i)], c->devs[size_t(j)]));
        if (!ok)
          fail(SSB_ECUDA, "device " + std::to_string(c->devs[size_t(i)]) + " cannot access device " +
                              std::to_string(c->devs[size_t(j)]) + " (no peer path for the fused exchange)");
        SSB_CUDA(cudaSetDevice(c->devs[size_t(i)]));
        const cudaError_t rc = cudaDeviceEnablePeerAccess(c->devs[size_t(j)], 0);
        if (rc == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else SSB_CUDA(rc);
      }
  }
  return c.release();
}

ssb_sharded* ctx_build(ssb_ctx& c, const ssb_edges& e, int64_t C, int64_t sigma, int k) {
  if (C != 32) fail(SSB_EINVAL, "the sharded BFS needs the C = 32 layout");
  if (k < 1 || k > kMaxSeg) fail(SSB_EINVAL, "segments per rank must be in [1, 8]");
  DeviceGuard guard;
  const int world = int(c.devs.size());
  const int src = guard.prev;  // e lives on the current device
  auto sh = std::make_unique<ssb_sharded>();
  sh->ctx = &c;
  {
    std::unique_ptr<ssb_graph> meta(build_range_from_edges(e, C, sigma, {0, 0}));  // cl for the partition
    sh->segs = partition_segments_host(meta->cl_host, C, world, k);
    sh->n = meta->n;
  }
  for (int i = 0; i < world; ++i) {
    const int d = c.devs[size_t(i)];
    const ssb_edges* ei = &e;
    std::unique_ptr<ssb_edges> copy;
    if (d != src) {
      copy = edges_on(e, src, d);
      ei = copy.get();
    }
    SSB_CUDA(cudaSetDevice(d));
    sh->g.emplace_back(build_range_from_edges(*ei, C, sigma, sh->segs[size_t(i)]));
  }
  if (!c.group && world > 1) {
    // windows: every rank's frontier window as a raw peer pointer
    std::vector<uint32_t*> wins(static_cast<size_t>(world));
    std::vector<WinGeom> wgs(static_cast<size_t>(world));
    for (int i = 0; i < world; ++i) {
      SSB_CUDA(cudaSetDevice(c.devs[size_t(i)]));
      wins[size_t(i)] = p2p_window_alloc(*sh->g[size_t(i)], wgs[size_t(i)]);
      SSB_CUDA(cudaMemset(wins[size_t(i)], 0, sh->g[size_t(i)]->p2p_win.bytes()));
    }
    for (int i = 0; i < world; ++i) {
      auto h = std::make_shared<P2PHost>();
      h->rank = i;
      h->world = world;
      h->wg = wgs[size_t(i)];
      h->segs = check_segments(*sh->g[size_t(i)], sh->segs[size_t(i)].data(),
                               int64_t(sh->segs[size_t(i)].size() / 2));
      for (int r = 0; r < world; ++r) h->win[r] = wins[size_t(r)];
      sh->g[size_t(i)]->p2p = h;
    }
  }
  for (int i = 0; i < world; ++i) {
    SSB_CUDA(cudaSetDevice(c.devs[size_t(i)]));
    sh->g[size_t(i)]->sc.sync();
  }
  return sh.release();
}

int sharded_bfs(ssb_sharded& sh, int64_t root, const ssb_bfs_options& o, int64_t* dist, int64_t* parent,
                int64_t* parent_len, ssb_iter_stats* stats, int64_t stats_cap, int64_t* iterations,
                double* device_ms) {
  if (o.variant < 0 || o.variant > 3) fail(SSB_EINVAL, "bad variant");
  if (root < 0 || root >= sh.n)
    fail(SSB_ERANGE, "root " + std::to_string(root) + " outside [0, " + std::to_string(sh.n) + ")");
  DeviceGuard guard;
  ssb_ctx& c = *sh.ctx;
  const int world = int(c.devs.size());
  std::vector<ssb_graph*> gs;
  for (auto& g : sh.g) gs.push_back(g.get());
  std::vector<std::vector<ssb_iter_stats>> st(static_cast<size_t>(world));
  std::vector<int64_t> its(static_cast<size_t>(world), 0);
  std::vector<double> ms(static_cast<size_t>(world), 0);
  std::vector<int> rcs(static_cast<size_t>(world), SSB_OK);
  std::vector<std::string> errs(static_cast<size_t>(world));
  const int64_t cap = std::max<int64_t>(stats_cap, 0) + 64;
  if (world == 1 || c.group) {
    SSB_CUDA(cudaSetDevice(c.devs[0]));
    std::vector<int64_t> bounds, counts;
    for (auto& s : sh.segs) {
      counts.push_back(int64_t(s.size() / 2));
      bounds.insert(bounds.end(), s.begin(), s.end());
    }
    if (world == 1 && !gs[0]->p2p) {  // a single rank: attach its own window
      WinGeom wg;
      uint32_t* w = p2p_window_alloc(*gs[0], wg);
      SSB_CUDA(cudaMemset(w, 0, gs[0]->p2p_win.bytes()));
      auto h = std::make_shared<P2PHost>();
      h->wg = wg;
      h->segs = check_segments(*gs[0], sh.segs[0].data(), int64_t(sh.segs[0].size() / 2));
      h->win[0] = w;
      gs[0]->p2p = h;
    }
    st[0].resize(size_t(cap));
    rcs[0] = bfs_p2p(gs.data(), world == 1 ? 1 : world, bounds.data(), counts.data(), root, o, st[0].data(),
                     cap, &its[0], &ms[0]);
  } else {
    std::vector<std::thread> th;
    for (int i = 0; i < world; ++i) {
      st[size_t(i)].resize(size_t(cap));
      th.emplace_back([&, i] {
        try {
          SSB_CUDA(cudaSetDevice(c.devs[size_t(i)]));
          rcs[size_t(i)] = bfs_p2p(&gs[size_t(i)], 1, nullptr, nullptr, root, o, st[size_t(i)].data(), cap,
                                   &its[size_t(i)], &ms[size_t(i)]);
        } catch (const Error& ex) {
          rcs[size_t(i)] = ex.code;
          errs[size_t(i)] = ex.what();
        } catch (const std::exception& ex) {
          rcs[size_t(i)] = SSB_ECUDA;
          errs[size_t(i)] = ex.what();
        }
      });
    }
    for (auto& t : th) t.join();
    for (int i = 0; i < world; ++i)
      if (rcs[size_t(i)] != SSB_OK && rcs[size_t(i)] != SSB_ECAP) fail(rcs[size_t(i)], errs[size_t(i)]);
  }
  const int64_t iters = its[0];
  // counters: summed over the ranks (each returns its own chunks' counts)
  if (stats) {
    for (int64_t j = 0; j < std::min<int64_t>(stats_cap, iters); ++j) {
      ssb_iter_stats a = st[0][size_t(j)];
      for (int i = 1; i < (c.group ? 1 : world); ++i) {
        const ssb_iter_stats& b = st[size_t(i)][size_t(j)];
        a.chunks_processed += b.chunks_processed;
        a.chunks_skipped += b.chunks_skipped;
        a.subchunks_processed += b.subchunks_processed;
        a.columns_processed += b.columns_processed;
        a.frontier_size += b.frontier_size;
        a.elapsed_ns = std::max(a.elapsed_ns, b.elapsed_ns);
      }
      stats[j] = a;
    }
  }
  if (iterations) *iterations = iters;
  if (device_ms) *device_ms = *std::max_element(ms.begin(), ms.end());
  // results: each rank writes its owned rows (original ids)
  const bool want = o.want_parents && o.variant == SSB_SELMAX && rcs[0] == SSB_OK;
  for (int64_t v = 0; dist && v < sh.n; ++v) dist[v] = INT64_MAX;
  if (want && parent)
    for (int64_t v = 0; v < sh.n; ++v) parent[v] = -1;
  for (int i = 0; i < world; ++i) {
    SSB_CUDA(cudaSetDevice(c.devs[size_t(i)]));
    if (dist) shard_fetch(*gs[size_t(i)], want && parent, dist, want && parent ? parent : nullptr);
  }
  if (parent_len) *parent_len = want && parent ? sh.n : 0;
  return rcs[0];
}

}  // namespace ssb
