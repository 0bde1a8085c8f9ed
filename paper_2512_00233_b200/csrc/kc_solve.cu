// kc_solve.cu — the FastK coreness fixed point as ONE persistent cooperative
// kernel on sm_100a.
//
// Reference path (paths under /root/reference/proj):
//   fastk_run            src/fastk.cpp:57-187  — rounds of process | apply | notify
//   recompute_node       src/fastk.cpp:15-20   — gather est[nb] over the row
//   compute_index_over   include/kcore/kernel.hpp:27-42 — capped h-index
//   should_notify        include/kcore/fastk.hpp:25-27  — extended activation rule
//
// State.  E (est[0]) is the round's snapshot, N (est[1]) the settled values;
// N == E at every round start.  The frontier is a byte flag per vertex:
// flag[r&1] is round r's active set, flag[(r+1)&1] collects the next one with
// plain stores.  Vertices are relabelled by descending degree at upload, so
// the degree classes (kc_internal.h) are id ranges that workers scan in
// chunks, and est[0, cache_n) — the most-gathered estimates — is cached in
// every CTA's shared memory.
//
// One round = two grid barriers:
//   EVALUATE  every active u computes t = capped h-index of E over its row
//             (the reference's process phase on a frozen snapshot,
//             fastk.cpp:128-149) and writes N[u] = t; under the counting rule
//             also cnt[u] = #{w : E[w] >= t}.
//   --- grid.sync (a round without a drop ends here, fastk.cpp:109-110) ---
//   NOTIFY    every dropper u (N[u] < E[u]) re-streams its row against the
//             SETTLED values N (fastk.cpp:156-163), activates neighbours for
//             round r+1, and applies E[u] = N[u] (fastk.cpp:153).
//             Reference rule: activate w iff should_notify(t, cap, N[w]).
//             Counting rule: if should_notify, atomicSub(cnt[w]); the one
//             decrement that takes cnt[w] below N[w] activates w.  cnt[v]
//             stays exactly #{neighbours at or above v's level}, so a vertex
//             is evaluated iff it will drop: same Jacobi trajectory as the
//             reference (shadow_run, tests/test_fastk.cpp:41-92), no wasted
//             evaluations.
//   --- grid.sync ---
// No host synchronisation happens between rounds.
#include <cooperative_groups.h>
#include <cstdint>

// 4-entry streams like the counting solver (kc_count.cu): R-MAT 22 15.45 -> 14.91 ms, R-MAT 26
// 137.2 -> 132.9 ms, Chung-Lu 25.3 -> 25.0 ms with the reference's defaults.
#ifndef KC_STREAM_K
#define KC_STREAM_K 4
#endif
#include "kc_dev.cuh"
#include "kc_internal.h"

namespace cg = cooperative_groups;

#ifndef KC_SOLVE_DCUT
#define KC_SOLVE_DCUT 1  // degree cut table in the reference-rule scans
#endif
#ifndef KC_SOLVE_FINE
#define KC_SOLVE_FINE 1  // hub windows: the 256 levels below cap first (sorted rows)
#endif
constexpr uint32_t HUB_FINE = 256;
#ifndef KC_SOLVE_R0
#define KC_SOLVE_R0 1    // round 0 on sorted rows by the prefix rule (r0_sorted_warp)
#ifndef KC_SOLVE_R0_LANE
#define KC_SOLVE_R0_LANE 0  // ... BIG / WARP rows by a lane each (r0_sorted_lane): slower here (8-16
                            // items per grab leave most lanes idle: R-MAT 26 137 -> 143 ms)
#endif
#endif

namespace kcb {
namespace {
using namespace dev;

// Active vertices grabbed per atomic, per class.
constexpr uint32_t G_BIG = 2, G_WARP = 8, G_SUB = 32, G_THREAD = 32;
constexpr uint32_t COMPACT_IDS = SOLVE_THREADS * 16;  // ids per CTA compaction block
#ifndef KC_SOLVE_CACHE_MIN
#define KC_SOLVE_CACHE_MIN 4096
#endif
constexpr uint32_t CACHE_MIN_ACTIVE = KC_SOLVE_CACHE_MIN;  // smaller rounds skip the shared-memory cache

template <typename OffT, typename EstT>
struct P {
  const OffT* off;
  const uint32_t* adj;
  uint32_t n_nz;
  uint32_t cb[NCLS + 1];
  EstT* E;  // snapshot
  EstT* N;  // settled
  uint32_t* cnt;
  uint8_t* flag[2];
  uint32_t* queue;
  Ctl* ctl;
  uint32_t* anydrop;
  RoundStat* stats;
  uint32_t* status;
  unsigned long long* prof;
  uint32_t r_begin, r_end;
  int rule;
  uint32_t cache_n;
  uint32_t clamp_drop;  // max degree > H: the reference's round 0 lowers deg -> <= H
  uint32_t tail_batch;  // hybrid_tail: switch threshold (0 = off)
  const uint32_t* dcut;  // degree cut table (kc_count.cu DegCut), dcut_n entries
  uint32_t dcut_n;
  bool sorted;           // rows sorted ascending: scans stop at the first id >= their cut
};

// Ids >= id_cut(x) have degree, hence estimate, < x: skipped without a gather.
template <typename OffT, typename EstT>
__device__ __forceinline__ uint32_t id_cut(const P<OffT, EstT>& p, uint32_t x) {
  return !p.dcut ? 0xffffffffu : x < p.dcut_n ? p.dcut[x] : 0u;
}

__device__ __forceinline__ uint32_t window_floor(uint32_t top, uint32_t bins, uint32_t lo) {
  uint32_t f = top > bins ? top - bins : 0u;
  if (lo > f) f = lo;
  return f ? f : 1u;
}

// Per-round view: what this round reads and writes.
template <typename EstT>
struct RoundView {
  const EstT* snap;  // gathered estimates of the current phase (E, then N)
  uint8_t* fnxt;     // activations for round r+1
  const uint32_t* qcnt;  // active vertices per class (round r's compacted queue)
  uint32_t* grab;    // work cursors of the current phase
  bool count;        // counting rule
  bool ext;          // extended_notify (reference rule)
  bool skip_a;       // counting rule, r > 0: every active vertex drops
  bool r0;           // round 0 (E = min(deg, H))
  uint32_t cache_n;  // ids cached in shared memory this round (0: none)
};

struct Acc {  // per-thread counters, flushed per round
  unsigned long long evals, escan, drops, fires, nscan;
  bool any_drop;
};

// One evaluation result (the evaluate phase): lower N[u], keep cnt[u] exact.
template <typename OffT, typename EstT>
__device__ __forceinline__ void finish_eval(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                                            uint32_t u, uint32_t t, uint32_t cap, uint32_t c,
                                            uint64_t deg, Acc& acc) {
  acc.evals += 1;
  acc.escan += deg;
  if (rv.count) p.cnt[u] = c;
  if (t < cap) {
    p.N[u] = (EstT)t;
    acc.drops += 1;
    acc.any_drop = true;
  }
}

// What a dropper u (cap -> t) does to K neighbours ids[k] with settled
// levels x[k] (valid where bit k of ok) in the notify phase.  All counter
// atomics are issued before any result is consumed (a byte store to the
// flags could alias cnt, so interleaving would serialise them).
template <int K, typename OffT, typename EstT>
__device__ __forceinline__ void notify_batch(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                                             uint32_t ok, const uint32_t (&ids)[K],
                                             const uint32_t (&x)[K], uint32_t t, uint32_t cap,
                                             Acc& acc) {
  uint32_t fire = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool f = (ok >> k & 1) && (rv.count || rv.ext ? (t < x[k] && x[k] <= cap) : (x[k] > t));
    fire |= (uint32_t)f << k;
  }
  acc.fires += __popc(fire);
  if (rv.count) {  // should_notify on the settled value -> decrement cnt[w]
    uint32_t old[K];
#pragma unroll
    for (int k = 0; k < K; ++k) old[k] = (fire >> k & 1) ? atomicSub(&p.cnt[ids[k]], 1u) : 0u;
#pragma unroll
    for (int k = 0; k < K; ++k)  // the decrement that took cnt[w] below N[w]
      if ((fire >> k & 1) && old[k] == x[k]) rv.fnxt[ids[k]] = 1;
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (fire >> k & 1) rv.fnxt[ids[k]] = 1;
  }
}

// ------------------------------------------------------------------------
// Frontier compaction (round start, all CTAs): round r's flags become a
// dense per-class queue.  CTAs take interleaved blocks of COMPACT_IDS ids,
// each thread reads 16 flags with one 128-bit load and clears them; one
// atomicAdd per CTA block reserves the block's slots in the class segment.
// ------------------------------------------------------------------------
template <typename OffT, typename EstT>
__device__ void compact_frontier(const P<OffT, EstT>& p, uint8_t* flags, uint32_t* qcnt,
                                 uint32_t* s_red, uint32_t* s_item) {
  const uint32_t tid = threadIdx.x;
  for (int c = 0; c < NCLS; ++c) {
    const uint32_t b0 = p.cb[c], b1 = p.cb[c + 1];
    const uint32_t a0 = b0 & ~15u;
    const uint32_t nblk = (b1 - a0 + COMPACT_IDS - 1) / COMPACT_IDS;
    for (uint32_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
      const uint32_t a = a0 + blk * COMPACT_IDS + 16 * tid;
      uint4 w = make_uint4(0, 0, 0, 0);
      if (a < b1) w = *reinterpret_cast<const uint4*>(flags + a);
      uint32_t m = 0;  // bit j: id a+j active and inside the class
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t word = j < 4 ? w.x : j < 8 ? w.y : j < 12 ? w.z : w.w;
        const uint32_t id = a + j;
        if ((word >> (8 * (j & 3)) & 0xffu) && id >= b0 && id < b1) m |= 1u << j;
      }
      const uint32_t mine = __popc(m);
      const uint32_t off = block_excl_scan(mine, s_red);
      if (tid == SOLVE_THREADS - 1) {
        const uint32_t tot = off + mine;
        *s_item = tot ? atomicAdd(&qcnt[c], tot) : 0u;
      }
      __syncthreads();
      uint32_t pos = b0 + *s_item + off;
      __syncthreads();
      if (m) {
        // clear exactly this class's bytes of the 16 (a neighbouring class
        // may share the 16-byte granule)
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (m >> j & 1) {
            KC_BOUNDS(pos < b1);
            p.queue[pos++] = a + j;
            flags[a + j] = 0;
          }
      }
    }
  }
}

// Warp-level dense-queue grab: up to G (<= 32) items per atomic; `proc` gets
// the warp's slice (lane i may read q[i] for i < n).
template <uint32_t G, typename F>
__device__ __forceinline__ void for_queue(const uint32_t* q, uint32_t cnt, uint32_t* cursor,
                                          F&& proc) {
  static_assert(G <= 32, "one item per lane at most");
  if (cnt == 0) return;
  for (;;) {
    uint32_t base = 0;
    if (lane_id() == 0)  // plain read first: no atomic once the queue is drained
      base = *reinterpret_cast<volatile uint32_t*>(cursor) >= cnt ? cnt : atomicAdd(cursor, G);
    base = __shfl_sync(FULL, base, 0);
    if (base >= cnt) break;
    proc(q + base, cnt - base < G ? cnt - base : G);
  }
}

// CTA-level grab of the next queued HUGE vertex (0xffffffff when none).
template <typename OffT, typename EstT>
__device__ __forceinline__ uint32_t grab_huge(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                                              uint32_t* s_item) {
  if (threadIdx.x == 0) {
    const uint32_t cnt = rv.qcnt[C_HUGE];
    const uint32_t k = (cnt == 0 || *reinterpret_cast<volatile uint32_t*>(&rv.grab[C_HUGE]) >= cnt)
                           ? cnt
                           : atomicAdd(&rv.grab[C_HUGE], 1u);
    *s_item = k < cnt ? p.queue[p.cb[C_HUGE] + k] : 0xffffffffu;
  }
  __syncthreads();
  const uint32_t u = *s_item;
  __syncthreads();
  return u;
}

// ------------------------------------------------------------------------
// HUGE class (deg > DEG_BIG_MAX): CTA per vertex.  Pass A counts values >=
// cap in registers ("no change" costs one read + one block reduction); a drop
// runs windowed histogram passes (values >= top in registers, the window
// [top - HIST_BINS, top) binned in shared memory).  Re-reads hit L2.
// ------------------------------------------------------------------------
template <typename OffT, typename EstT>
__device__ __noinline__ void huge_window(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                                         const EstT* s_cache, uint32_t* s_hist, uint32_t* s_red,
                                         uint64_t ob, uint64_t oe, uint32_t cap, uint32_t lo,
                                         uint32_t* out) {
  const uint32_t tid = threadIdx.x;
  uint32_t top = cap;
  // sorted rows: the FINE levels below cap first — most drops are small, and
  // that window's cut reads a short prefix of a hub's row
  bool fine = KC_SOLVE_FINE && p.sorted && cap > HUB_FINE;
  for (;;) {
    const uint32_t fl = fine && top - HUB_FINE > lo ? top - HUB_FINE : lo;  // tally floor
    const int minx = fine ? (int)(top - HUB_FINE) : 1;  // levels this pass decides
    for (int i = tid; i < HIST_BINS; i += SOLVE_THREADS) s_hist[i] = 0;
    __syncthreads();
    uint32_t above = 0;
    stream_row<SOLVE_THREADS, true>(p.adj, rv.snap, tid, ob, oe, s_cache, rv.cache_n,
                              [&](uint32_t ok, const uint32_t(&)[8], const uint32_t(&x)[8]) {
#pragma unroll
                                for (int k = 0; k < 8; ++k)
                                  if (ok >> k & 1) tally<HIST_BINS>(x[k], top, fl, above, s_hist);
                              }, id_cut(p, window_floor(top, fine ? HUB_FINE : HIST_BINS, lo)),
                              p.sorted);
    const uint32_t C = block_sum(above, s_red);
    constexpr int PER = (HIST_BINS + SOLVE_THREADS - 1) / SOLVE_THREADS;  // bins per thread
    uint32_t h[PER];
    uint32_t sm = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      h[j] = tid * PER + j < HIST_BINS ? s_hist[tid * PER + j] : 0u;
      sm += h[j];
    }
    uint32_t run = C + block_excl_scan(sm, s_red);
    uint32_t found = 0xffffffffu, frun = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      run += h[j];
      const int i = tid * PER + j;
      const int x = i < HIST_BINS ? (int)top - 1 - i : 0;  // x = 0 never qualifies
      if (found == 0xffffffffu && x >= minx && run >= (uint32_t)x) {
        found = (uint32_t)i;
        frun = run;
      }
    }
    const uint32_t g = block_min(found, s_red);
    if (g != 0xffffffffu) {
      if (found == g) {
        out[0] = top - 1 - g;
        out[1] = frun;
      }
      __syncthreads();
      return;
    }
    if (fine) {  // no level in [top - HUB_FINE, top) qualifies: the regular windows below
      fine = false;
      top -= HUB_FINE;
      __syncthreads();
      continue;
    }
    if ((int)top - HIST_BINS <= 0) {
      if (tid == 0) {
        out[0] = 0;
        out[1] = (uint32_t)(oe - ob);
      }
      __syncthreads();
      return;
    }
    top -= HIST_BINS;
  }
}

template <typename OffT, typename EstT>
__device__ void eval_huge(const P<OffT, EstT>& p, const RoundView<EstT>& rv, const EstT* s_cache,
                          uint32_t* s_hist, uint32_t* s_red, uint32_t* s_item, Acc& acc) {
  const uint32_t tid = threadIdx.x;
  __shared__ uint32_t s_out[2];
  for (;;) {
    const uint32_t u = grab_huge(p, rv, s_item);
    if (u == 0xffffffffu) break;
    const uint64_t ob = p.off[u], oe = p.off[u + 1];
    const uint32_t cap = est_at(s_cache, rv.cache_n, rv.snap, u);
    if (KC_SOLVE_R0 && rv.r0 && p.sorted) {  // a prefix of the row: one warp's
      if (warp_id() == 0) {
        uint32_t sc = 0;
        const uint2 tc = r0_sorted_warp(p.adj, p.dcut, ob, (uint32_t)(oe - ob), cap, sc);
        if (tid == 0) finish_eval(p, rv, u, tc.x, cap, tc.y, oe - ob, acc);
      }
      __syncthreads();
      continue;
    }
    bool keep = false;
    uint32_t cA = 0;
    if (!rv.skip_a) {
      uint32_t c = 0;
      stream_row<SOLVE_THREADS, true>(p.adj, rv.snap, tid, ob, oe, s_cache, rv.cache_n,
                                [&](uint32_t ok, const uint32_t(&)[8], const uint32_t(&x)[8]) {
#pragma unroll
                                  for (int k = 0; k < 8; ++k) c += (ok >> k & 1) && x[k] >= cap;
                                }, id_cut(p, cap), p.sorted);
      cA = block_sum(c, s_red);
      keep = cA >= cap;
    }
    uint32_t t = cap, cn = cA;
    if (!keep) {
      // counting rule: the new level is >= cnt[u] = count(>= cap)
      const uint32_t lo = rv.skip_a ? p.cnt[u] : 0u;
      huge_window(p, rv, s_cache, s_hist, s_red, ob, oe, cap, lo, s_out);
      t = s_out[0];
      cn = s_out[1];
    }
    if (tid == 0) finish_eval(p, rv, u, t, cap, cn, oe - ob, acc);
    __syncthreads();
  }
}

// ------------------------------------------------------------------------
// Warp-per-vertex classes.  Metadata (offsets, cap) of a batch of up to 32
// active vertices is loaded in parallel, one lane per vertex, then the warp
// walks the batch.
// ------------------------------------------------------------------------
struct Meta {
  uint32_t u, cap;
  uint64_t ob, oe;
};

template <typename OffT, typename EstT>
__device__ __forceinline__ Meta load_meta(const P<OffT, EstT>& p, const EstT* capsrc,
                                          const EstT* s_cache, uint32_t cache_n,
                                          const uint32_t* q, uint32_t n) {
  Meta m{0, 0, 0, 0};
  const uint32_t lane = lane_id();
  if (lane < n) {
    m.u = q[lane];
    m.ob = p.off[m.u];
    m.oe = p.off[m.u + 1];
    m.cap = est_at(s_cache, cache_n, capsrc, m.u);
  }
  return m;
}

__device__ __forceinline__ Meta shfl_meta(const Meta& m, int src) {
  Meta it;
  it.u = __shfl_sync(FULL, m.u, src);
  it.cap = __shfl_sync(FULL, m.cap, src);
  it.ob = __shfl_sync(FULL, m.ob, src);
  it.oe = __shfl_sync(FULL, m.oe, src);
  return it;
}

// Windowed histogram passes of one warp over a row: capped h-index + count.
template <typename OffT, typename EstT>
__device__ __noinline__ uint2 warp_window(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                                          const EstT* s_cache, uint32_t* bins, uint64_t ob,
                                          uint64_t oe, uint32_t cap, uint32_t lo) {
  const uint32_t lane = lane_id();
  uint32_t top = cap;
  for (;;) {
    warp_zero_bins(bins);
    uint32_t above = 0;
    stream_row<32, true>(p.adj, rv.snap, lane, ob, oe, s_cache, rv.cache_n,
                   [&](uint32_t ok, const uint32_t(&)[8], const uint32_t(&x)[8]) {
#pragma unroll
                     for (int k = 0; k < 8; ++k)
                       if (ok >> k & 1) tally<WARP_BINS>(x[k], top, lo, above, bins);
                   }, id_cut(p, window_floor(top, WARP_BINS, lo)), p.sorted);
    __syncwarp();
    const uint32_t C = __reduce_add_sync(FULL, above);
    uint32_t level = 0, c = 0;
    const bool hit = warp_resolve(bins, C, top, level, c);
    __syncwarp();
    if (hit) return make_uint2(level, c);
    if ((int)top - WARP_BINS <= 0) return make_uint2(0u, (uint32_t)(oe - ob));
    top -= WARP_BINS;
  }
}

// WARP and BIG classes (DEG_SUB_MAX < deg <= DEG_BIG_MAX): warp per vertex,
// 256 entries per warp step (two 128-bit id loads + 8 gathers per lane).
template <uint32_t G, typename OffT, typename EstT>
__device__ void eval_wstream(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                             const EstT* s_cache, int cls, uint32_t* bins, Acc& acc) {
  const uint32_t lane = lane_id();
  for_queue<G>(p.queue + p.cb[cls], rv.qcnt[cls], &rv.grab[cls],
               [&](const uint32_t* lst, uint32_t n) {
    const Meta mine = load_meta(p, rv.snap, s_cache, rv.cache_n, lst, n);
    if (KC_SOLVE_R0 && KC_SOLVE_R0_LANE && rv.r0 && p.sorted) {
      // round 0 on sorted rows: a lane per vertex, two binary searches (r0_sorted_lane, kc_dev.cuh)
      if (lane < n) {
        uint32_t sc = 0;
        const uint2 tc = r0_sorted_lane(p.adj, p.dcut, mine.ob, (uint32_t)(mine.oe - mine.ob), mine.cap, sc);
        finish_eval(p, rv, mine.u, tc.x, mine.cap, tc.y, mine.oe - mine.ob, acc);
      }
      return;
    }
    for (uint32_t i = 0; i < n; ++i) {
      const Meta it = shfl_meta(mine, i);
      const uint32_t cap = it.cap;
      if (KC_SOLVE_R0 && rv.r0 && p.sorted) {
        uint32_t sc = 0;
        const uint2 tc = r0_sorted_warp(p.adj, p.dcut, it.ob, (uint32_t)(it.oe - it.ob), cap, sc);
        if (lane == 0) finish_eval(p, rv, it.u, tc.x, cap, tc.y, it.oe - it.ob, acc);
        continue;
      }
      bool keep = false;
      uint32_t cA = 0;
      if (!rv.skip_a) {
        uint32_t c = 0;
        stream_row<32, true>(p.adj, rv.snap, lane, it.ob, it.oe, s_cache, rv.cache_n,
                       [&](uint32_t ok, const uint32_t(&)[8], const uint32_t(&x)[8]) {
#pragma unroll
                         for (int k = 0; k < 8; ++k) c += (ok >> k & 1) && x[k] >= cap;
                       }, id_cut(p, cap), p.sorted);
        cA = __reduce_add_sync(FULL, c);
        keep = cA >= cap;
      }
      uint2 tc = make_uint2(cap, cA);
      if (!keep)
        tc = warp_window(p, rv, s_cache, bins, it.ob, it.oe, cap, rv.skip_a ? p.cnt[it.u] : 0u);
      if (lane == 0) finish_eval(p, rv, it.u, tc.x, cap, tc.y, it.oe - it.ob, acc);
    }
  });
}

// ------------------------------------------------------------------------
// SUB class (DEG_THREAD_MAX < deg <= DEG_SUB_MAX): 8-lane tile per vertex
// (4 vertices per warp), 8 values per lane in registers, bisection.
// ------------------------------------------------------------------------
template <typename OffT, typename EstT>
__device__ void eval_sub(const P<OffT, EstT>& p, const RoundView<EstT>& rv, const EstT* s_cache,
                         Acc& acc) {
  constexpr int R = DEG_SUB_MAX / 8;
  const uint32_t g = lane_id() >> 3, k = lane_id() & 7;
  for_queue<G_SUB>(p.queue + p.cb[C_SUB], rv.qcnt[C_SUB], &rv.grab[C_SUB],
                   [&](const uint32_t* lst, uint32_t n) {
    const Meta mine = load_meta(p, rv.snap, s_cache, rv.cache_n, lst, n);
    for (uint32_t i0 = 0; i0 < n; i0 += 4) {
      // every lane runs the shuffles; tiles beyond n idle
      const Meta it = shfl_meta(mine, (int)(i0 + g) & 31);
      const bool has = i0 + g < n;
      const uint32_t deg = has ? (uint32_t)(it.oe - it.ob) : 0u;
      const uint32_t cap = has ? it.cap : 0u;
      Vals<EstT, R> vals;
      vals.clear();
      {
        uint32_t ids[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const uint32_t q = k + 8 * j;
          ids[j] = q < deg ? p.adj[it.ob + q] : 0xffffffffu;
        }
        if (KC_SOLVE_R0 && rv.r0 && p.sorted) {  // prefix rule on the ids (r0_sorted_warp)
          const uint32_t m = deg < cap ? deg : cap;
          uint32_t hc = 0;
#pragma unroll
          for (int j = 0; j < R; ++j) hc += k + 8 * j < m && ids[j] < __ldg(p.dcut + k + 8 * j + 1);
          const uint32_t t = tile8_sum(hc);
          const uint32_t ct = __ldg(p.dcut + t);
          uint32_t cc = 0;
#pragma unroll
          for (int j = 0; j < R; ++j) cc += ids[j] < ct;
          const uint32_t c = tile8_sum(cc);
          if (has && k == 0) finish_eval(p, rv, it.u, t, cap, t ? c : deg, deg, acc);
          continue;
        }
#pragma unroll
        for (int j = 0; j < R; ++j)
          if (ids[j] != 0xffffffffu) vals.set(j, est_at(s_cache, rv.cache_n, rv.snap, ids[j]));
      }
      // capped h-index by bisection, all four tiles in lockstep
      const uint32_t cA = tile8_sum(vals.count_ge(cap));
      uint32_t lo = 0, hi = cap;
#pragma unroll 1
      for (int s = 0; s < 7; ++s) {  // cap <= 64
        const uint32_t mid = (lo + hi) >> 1;
        const bool okm = tile8_sum(vals.count_ge(mid)) >= mid;
        if (hi - lo > 1) {
          if (okm) lo = mid; else hi = mid;
        }
      }
      const uint32_t t = cA >= cap ? cap : lo;
      const uint32_t c = tile8_sum(vals.count_ge(t));
      if (has && k == 0) finish_eval(p, rv, it.u, t, cap, c, deg, acc);
    }
  });
}

// ------------------------------------------------------------------------
// THREAD class (deg <= DEG_THREAD_MAX): thread per vertex.  h-index =
// max_i min(x_i, #{j : x_j >= x_i}) — the classic identity — capped at cap.
// ------------------------------------------------------------------------
template <typename OffT, typename EstT>
__device__ void eval_thread(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                            const EstT* s_cache, Acc& acc) {
  constexpr int R = DEG_THREAD_MAX;
  const uint32_t lane = lane_id();
  for_queue<G_THREAD>(p.queue + p.cb[C_THREAD], rv.qcnt[C_THREAD], &rv.grab[C_THREAD],
                      [&](const uint32_t* lst, uint32_t n) {
    if (lane >= n) return;
    const uint32_t u = lst[lane];
    const uint64_t ob = p.off[u];
    const uint32_t deg = (uint32_t)(p.off[u + 1] - ob);
    const uint32_t cap = est_at(s_cache, rv.cache_n, rv.snap, u);
    uint32_t x[R];
#pragma unroll
    for (int j = 0; j < R; ++j) x[j] = (uint32_t)j < deg ? p.adj[ob + j] : 0xffffffffu;
    if (KC_SOLVE_R0 && rv.r0 && p.sorted) {  // prefix rule on the ids (r0_sorted_warp)
      const uint32_t m = deg < cap ? deg : cap;
      uint32_t t = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) t += (uint32_t)j < m && x[j] < __ldg(p.dcut + j + 1);
      const uint32_t ct = __ldg(p.dcut + t);
      uint32_t c = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) c += x[j] < ct;
      finish_eval(p, rv, u, t, cap, t ? c : deg, deg, acc);
      return;
    }
#pragma unroll
    for (int j = 0; j < R; ++j)
      x[j] = x[j] != 0xffffffffu ? est_at(s_cache, rv.cache_n, rv.snap, x[j]) : 0u;
    uint32_t h = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      uint32_t c = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) c += x[j] >= x[i];
      const uint32_t m = x[i] < c ? x[i] : c;
      h = m > h ? m : h;
    }
    const uint32_t t = h < cap ? h : cap;
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) c += x[j] >= t;
    finish_eval(p, rv, u, t, cap, t ? c : deg, deg, acc);
  });
}

// ------------------------------------------------------------------------
// NOTIFY phase: every dropper u of round r (flag set, N[u] < E[u]) streams
// its row against the settled values N, activates neighbours for round r+1
// (notify_one) and applies E[u] = N[u].  All of round r's flags are cleared.
// Gathers go through the shared-memory cache of N.
// ------------------------------------------------------------------------
template <typename OffT, typename EstT>
__device__ void notify_huge(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                            const EstT* s_cache, uint32_t* s_item, Acc& acc) {
  const uint32_t tid = threadIdx.x;
  for (;;) {
    const uint32_t u = grab_huge(p, rv, s_item);
    if (u == 0xffffffffu) break;
    const uint32_t t = p.N[u], cap = p.E[u];
    if (t < cap) {
      const uint64_t ob = p.off[u], oe = p.off[u + 1];
      if (tid == 0) acc.nscan += oe - ob;
      // only N[w] > t notifies (both guards): ids >= cut(t + 1) cannot
      stream_row<SOLVE_THREADS, true>(p.adj, p.N, tid, ob, oe, s_cache, rv.cache_n,
                                [&](uint32_t ok, const uint32_t(&ids)[8], const uint32_t(&x)[8]) {
                                  notify_batch<8>(p, rv, ok, ids, x, t, cap, acc);
                                }, id_cut(p, t + 1), p.sorted);
    }
    // Apply only after every thread of the CTA has read cap = E[u]: stream_row
    // has no CTA barrier, so a warp that leaves its share of the row early
    // (degree cut, `stop`) could otherwise store E[u] = t before a lagging
    // warp's load, which then sees t >= cap and skips its share of the
    // notifications (the rare `fires` / messages_sent deficit).
    __syncthreads();
    if (tid == 0 && t < cap) p.E[u] = (EstT)t;  // apply (fastk.cpp:153)
  }
}

template <uint32_t G, typename OffT, typename EstT>
__device__ void notify_wstream(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                               const EstT* s_cache, int cls, Acc& acc) {
  const uint32_t lane = lane_id();
  for_queue<G>(p.queue + p.cb[cls], rv.qcnt[cls], &rv.grab[cls],
               [&](const uint32_t* lst, uint32_t n) {
    Meta mine = load_meta(p, (const EstT*)p.E, (const EstT*)nullptr, 0u, lst, n);  // cap = old E
    const uint32_t tn = lane < n ? (uint32_t)p.N[mine.u] : 0u;
    for (uint32_t i = 0; i < n; ++i) {
      const Meta it = shfl_meta(mine, i);
      const uint32_t t = __shfl_sync(FULL, tn, i);
      if (t >= it.cap) continue;  // evaluated but did not drop (warp-uniform)
      if (lane == 0) acc.nscan += it.oe - it.ob;
      stream_row<32, true>(p.adj, (const EstT*)p.N, lane, it.ob, it.oe, s_cache, rv.cache_n,
                     [&](uint32_t ok, const uint32_t(&ids)[8], const uint32_t(&x)[8]) {
                       notify_batch<8>(p, rv, ok, ids, x, t, it.cap, acc);
                     }, id_cut(p, t + 1), p.sorted);
      if (lane == 0) p.E[it.u] = (EstT)t;
    }
  });
}

// SUB and THREAD droppers: 8-lane tile per dropper, up to 8 neighbours per lane.
template <uint32_t G, typename OffT, typename EstT>
__device__ void notify_small(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                             const EstT* s_cache, int cls, Acc& acc) {
  const uint32_t g = lane_id() >> 3, k = lane_id() & 7;
  for_queue<G>(p.queue + p.cb[cls], rv.qcnt[cls], &rv.grab[cls],
               [&](const uint32_t* lst, uint32_t n) {
    for (uint32_t i0 = 0; i0 < n; i0 += 4) {
      if (i0 + g >= n) continue;
      const uint32_t u = lst[i0 + g];
      const uint32_t t = p.N[u], cap = p.E[u];
      if (t >= cap) continue;
      const uint64_t ob = p.off[u];
      const uint32_t deg = (uint32_t)(p.off[u + 1] - ob);
      if (k == 0) acc.nscan += deg;
      uint32_t ids[8], x[8], ok = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bool v = k + 8u * j < deg;
        ids[j] = v ? p.adj[ob + k + 8u * j] : 0u;
        ok |= (uint32_t)v << j;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        x[j] = (ok >> j & 1) ? est_at(s_cache, rv.cache_n, (const EstT*)p.N, ids[j]) : 0u;
      notify_batch<8>(p, rv, ok, ids, x, t, cap, acc);
      if (k == 0) p.E[u] = (EstT)t;
    }
  });
}

template <typename OffT, typename EstT>
__device__ __forceinline__ void flush_acc(const P<OffT, EstT>& p, uint32_t sr, const Acc& acc,
                                          unsigned long long* s_acc) {
  const unsigned long long v[5] = {acc.evals, acc.escan, acc.drops, acc.fires, acc.nscan};
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    unsigned long long x = v[q];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(FULL, x, d);
    if (lane_id() == 0 && x) atomicAdd(&s_acc[q], x);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 5; ++q)
      if (s_acc[q]) atomicAdd(&p.stats[sr].evals + q, s_acc[q]);
  }
}

#ifndef KC_CTAS_PER_SM
#define KC_CTAS_PER_SM 1
#endif
template <typename OffT, typename EstT>
__global__ void __launch_bounds__(SOLVE_THREADS, KC_CTAS_PER_SM) rounds_kernel(P<OffT, EstT> p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem[];
  EstT* s_cache = opaque_ptr(reinterpret_cast<EstT*>(smem));  // see opaque_ptr
  const size_t cache_bytes = ((size_t)p.cache_n * sizeof(EstT) + 15) & ~(size_t)15;
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(smem + cache_bytes);
  // per-warp regions (alias s_hist once the HUGE phase is over):
  // windowed-histogram bins + the flat-stream batch state
  uint32_t* w_bins = s_hist + WARP_BINS * warp_id();
  __shared__ uint32_t s_red[33];
  __shared__ uint32_t s_item;
  __shared__ uint32_t s_drop;
  __shared__ unsigned long long s_acc[5];
  const uint32_t tid = threadIdx.x;
  const bool count = p.rule == R_COUNT;

  for (uint32_t r = p.r_begin; r < p.r_end; ++r) {
    const uint32_t cur = r & 1, nxt = cur ^ 1;
    const uint32_t sr = r < STAT_SLOTS - 1 ? r : STAT_SLOTS - 1;
    RoundView<EstT> rv;
    rv.snap = p.E;
    rv.fnxt = p.flag[nxt];
    rv.qcnt = p.ctl[cur].qcnt;
    rv.grab = p.ctl[cur].grab;
    rv.count = count;
    rv.ext = p.rule != R_REF_PLAIN;
    rv.skip_a = count && r > 0;
    rv.r0 = r == 0;
    unsigned long long* pf = (p.prof && r < PROF_ROUNDS && tid == 0)
                                 ? p.prof + ((size_t)r * gridDim.x + blockIdx.x) * PROF_PHASES
                                 : nullptr;
    if (pf) pf[0] = gtimer();
    // cursors, queue counts and drop flag of the NEXT round (idle now)
    if (blockIdx.x == 0 && tid < NCLS) {
      p.ctl[nxt].grab[tid] = 0;
      p.ctl[nxt].grab2[tid] = 0;
      p.ctl[nxt].qcnt[tid] = 0;
    }
    if (blockIdx.x == 0 && tid == 32) p.anydrop[(r + 1) % 3] = 0;
    // ---------------- COMPACT round r's flags ----------------
    compact_frontier(p, p.flag[cur], p.ctl[cur].qcnt, s_red, &s_item);
    if (tid < 5) s_acc[tid] = 0;
    if (tid == 0) s_drop = 0;
    grid.sync();
    // the shared-memory cache pays off only when the round has real work
    uint32_t active = 0;
#pragma unroll
    for (int c = 0; c < NCLS; ++c) active += rv.qcnt[c];
    if (r >= 1 && active < p.tail_batch) {
      // hybrid switch (fastk.cpp:113-115, switch_condition fastk.hpp:29-31):
      // round r-1 changed something and fewer than `batch` vertices are
      // active — stop here, leave round r's active set in flag[cur] for the
      // sequential tail (kc_tail.cu).  Grid-uniform: every CTA read the
      // same class sizes after the grid sync.
      for (int c = 0; c < NCLS; ++c)
        for (uint32_t i = blockIdx.x * SOLVE_THREADS + tid; i < rv.qcnt[c];
             i += gridDim.x * SOLVE_THREADS)
          p.flag[cur][p.queue[p.cb[c] + i]] = 1;
      if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = r;  // rounds executed (rep.iterations at the switch)
        p.status[1] = 1;
        p.status[2] = 1;
        p.status[3] = 0;
      }
      if (pf) pf[1] = pf[2] = pf[3] = pf[4] = pf[5] = pf[6] = pf[7] = gtimer();
      return;
    }
    const uint32_t cache_n = active >= CACHE_MIN_ACTIVE ? p.cache_n : 0u;
    if (blockIdx.x == 0 && tid == 0) {
      p.stats[sr].q01 = rv.qcnt[0] | (unsigned long long)rv.qcnt[1] << 32;
      p.stats[sr].q23 = rv.qcnt[2] | (unsigned long long)rv.qcnt[3] << 32;
      p.stats[sr].q4 = rv.qcnt[4];
    }
    rv.cache_n = cache_n;
    if (cache_n) fill_cache(s_cache, (const EstT*)p.E, cache_n);
    __syncthreads();
    Acc acc{0, 0, 0, 0, 0, false};
    if (pf) pf[1] = gtimer();
    // ---------------- EVALUATE ----------------
    eval_huge(p, rv, s_cache, s_hist, s_red, &s_item, acc);
    if (pf) pf[2] = gtimer();
    {
      eval_wstream<G_BIG>(p, rv, s_cache, C_BIG, w_bins, acc);
      eval_wstream<G_WARP>(p, rv, s_cache, C_WARP, w_bins, acc);
      if (pf) pf[3] = gtimer();
      eval_sub(p, rv, s_cache, acc);
      eval_thread(p, rv, s_cache, acc);
    }
    if (pf) pf[4] = gtimer();
    if (__any_sync(FULL, acc.any_drop) && lane_id() == 0) s_drop = 1;
    __syncthreads();
    if (tid == 0 && s_drop) p.anydrop[r % 3] = 1;
    grid.sync();
    // The reference starts at est = deg (fastk.cpp:67-68); the solver starts
    // at min(deg, H), so round 0 "changed" also when some degree exceeds H
    // (that drop is already applied).  Keeps iterations equal to the reference.
    const bool any = *reinterpret_cast<volatile uint32_t*>(&p.anydrop[r % 3]) != 0 ||
                     (r == 0 && p.clamp_drop);
    if (!any) {  // quiescent round: converged (fastk.cpp:109-110)
      flush_acc(p, sr, acc, s_acc);
      if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = r + 1;
        p.status[1] = 1;
        p.status[3] = 0;
      }
      if (pf) pf[5] = pf[6] = pf[7] = gtimer();
      return;
    }
    if (pf) pf[5] = gtimer();
    // ---------------- NOTIFY + APPLY ----------------
    rv.snap = p.N;
    rv.grab = p.ctl[cur].grab2;
    if (cache_n) fill_cache(s_cache, (const EstT*)p.N, cache_n);
    __syncthreads();
    if (pf) pf[6] = gtimer();
    notify_huge(p, rv, s_cache, &s_item, acc);
    {
      notify_wstream<G_BIG>(p, rv, s_cache, C_BIG, acc);
      notify_wstream<G_WARP>(p, rv, s_cache, C_WARP, acc);
      notify_small<G_SUB>(p, rv, s_cache, C_SUB, acc);
      notify_small<G_THREAD>(p, rv, s_cache, C_THREAD, acc);
    }
    flush_acc(p, sr, acc, s_acc);
    grid.sync();
    if (pf) pf[7] = gtimer();
    if (blockIdx.x == 0 && tid == 0) {
      p.status[0] = r + 1;
      p.status[3] = 0;
    }
  }
}

// Round-0 state: E = N = min(deg, H) (identical trajectory
// from round 1; the reference starts at deg, fastk.cpp:67-68), every
// non-isolated vertex active, everything else cleared.
template <typename OffT, typename EstT>
__global__ void init_kernel(P<OffT, EstT> p, uint32_t h_graph, uint32_t n_pad) {
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t gsize = gridDim.x * blockDim.x;
  for (uint32_t u = gtid; u < n_pad; u += gsize) {
    EstT e = 0;
    if (u < p.n_nz) {
      const uint32_t d = (uint32_t)(p.off[u + 1] - p.off[u]);
      e = (EstT)(d < h_graph ? d : h_graph);
    }
    p.E[u] = e;
    p.N[u] = e;
    p.cnt[u] = 0;
    p.flag[0][u] = u < p.n_nz ? 1 : 0;
    p.flag[1][u] = 0;
  }
  for (uint32_t k = gtid; k < STAT_SLOTS * (uint32_t)(sizeof(RoundStat) / 8); k += gsize)
    reinterpret_cast<unsigned long long*>(p.stats)[k] = 0;
  if (gtid < NCLS) {
    p.ctl[0].grab[gtid] = p.ctl[0].grab2[gtid] = p.ctl[0].qcnt[gtid] = 0;
    p.ctl[1].grab[gtid] = p.ctl[1].grab2[gtid] = p.ctl[1].qcnt[gtid] = 0;
  }
  if (gtid < 3) p.anydrop[gtid] = 0;
  if (gtid < 4) p.status[gtid] = 0;
}

template <typename OffT, typename EstT>
P<OffT, EstT> make_params(const SolveBuffers& b) {
  P<OffT, EstT> p{};
  p.off = static_cast<const OffT*>(b.off);
  p.adj = b.adj;
  p.dcut = KC_SOLVE_DCUT ? b.dcut : nullptr;
  p.dcut_n = b.dcut_n;
  p.sorted = p.dcut && b.rows_sorted;
  p.n_nz = b.n_nz;
  for (int c = 0; c <= NCLS; ++c) p.cb[c] = b.cls_begin[c];
  p.E = static_cast<EstT*>(b.est[0]);
  p.N = static_cast<EstT*>(b.est[1]);
  p.cnt = b.cnt;
  p.flag[0] = b.flag[0];
  p.flag[1] = b.flag[1];
  p.queue = b.queue;
  p.ctl = b.ctl;
  p.anydrop = b.anydrop;
  p.stats = b.stats;
  p.status = b.status;
  p.prof = b.prof;
  return p;
}

template <typename OffT, typename EstT>
cudaError_t launch_rounds_t(const SolveBuffers& b, const SolveConfig& c, uint32_t r_begin,
                            uint32_t r_end, cudaStream_t stream) {
  P<OffT, EstT> p = make_params<OffT, EstT>(b);
  p.r_begin = r_begin;
  p.r_end = r_end;
  p.rule = c.rule;
  p.cache_n = c.cache_n;
  p.clamp_drop = c.clamp_drop;
  p.tail_batch = c.tail_threshold;
  const size_t warp_region = (size_t)NWARPS * WARP_BINS;
  const size_t hist = (size_t)HIST_BINS > warp_region ? (size_t)HIST_BINS : warp_region;
  const size_t smem = (((size_t)c.cache_n * sizeof(EstT) + 15) & ~(size_t)15) +
                      hist * sizeof(uint32_t);
  auto kern = rounds_kernel<OffT, EstT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SOLVE_THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int ctas = per_sm < KC_CTAS_PER_SM ? per_sm : KC_CTAS_PER_SM;
  dim3 grid(c.num_sms * ctas), block(SOLVE_THREADS);
  void* args[] = {&p};
  return cudaLaunchCooperativeKernel((const void*)kern, grid, block, args, smem, stream);
}

template <typename OffT, typename EstT>
cudaError_t launch_init_t(const SolveBuffers& b, uint32_t h_graph, cudaStream_t stream) {
  P<OffT, EstT> p = make_params<OffT, EstT>(b);
  const uint32_t n_pad = (b.n_nz + 15) & ~15u;
  init_kernel<OffT, EstT><<<148 * 4, 256, 0, stream>>>(p, h_graph, n_pad);
  return cudaGetLastError();
}

}  // namespace

size_t solver_cache_bytes_max() {
  // 48 KB of hub estimates per CTA; the rest of the 228 KB unified L1 /
  // shared memory stays L1 for the other gathers (32-128 KB measured within
  // 4% of each other on R-MAT 22/26 and Chung-Lu; 48 KB best).
#ifdef KC_CACHE_KB
  return KC_CACHE_KB * 1024;
#else
  return 48 * 1024;
#endif
}

cudaError_t launch_rounds(const SolveBuffers& b, const SolveConfig& c, bool est16, bool off64,
                          uint32_t r_begin, uint32_t r_end, cudaStream_t stream) {
  if (est16)
    return off64 ? launch_rounds_t<uint64_t, uint16_t>(b, c, r_begin, r_end, stream)
                 : launch_rounds_t<uint32_t, uint16_t>(b, c, r_begin, r_end, stream);
  return off64 ? launch_rounds_t<uint64_t, uint32_t>(b, c, r_begin, r_end, stream)
               : launch_rounds_t<uint32_t, uint32_t>(b, c, r_begin, r_end, stream);
}

cudaError_t launch_init(const SolveBuffers& b, bool est16, bool off64, uint32_t h_graph,
                        uint32_t max_rounds, cudaStream_t stream) {
  (void)max_rounds;
  if (est16)
    return off64 ? launch_init_t<uint64_t, uint16_t>(b, h_graph, stream)
                 : launch_init_t<uint32_t, uint16_t>(b, h_graph, stream);
  return off64 ? launch_init_t<uint64_t, uint32_t>(b, h_graph, stream)
               : launch_init_t<uint32_t, uint32_t>(b, h_graph, stream);
}

}  // namespace kcb
