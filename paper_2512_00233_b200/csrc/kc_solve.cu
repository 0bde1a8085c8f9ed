// kc_solve.cu — the FastK coreness fixed point as ONE persistent cooperative
// kernel on sm_100a.
//
// Reference path (paths under /root/reference/proj):
//   fastk_run            src/fastk.cpp:57-187  — rounds of process | apply | notify
//   recompute_node       src/fastk.cpp:15-20   — gather est[nb] over the row
//   compute_index_over   include/kcore/kernel.hpp:27-42 — capped h-index
//   should_notify        include/kcore/fastk.hpp:25-27  — extended activation rule
//
// State: the frontier is a byte flag per vertex (flag[r&1] is read and
// cleared in round r, flag[(r+1)&1] collects activations with plain stores —
// no atomics, no queue appends); vertices are relabelled by descending degree
// so the degree classes (kc_internal.h) are id ranges that workers scan in
// chunks.
//
// Snapshot rule (default), one grid barrier per round:
//   est[r&1] is the round's snapshot (Jacobi, like the reference's process
//   phase reading est while updates are buffered, fastk.cpp:128-153); every
//   evaluated vertex writes its new value to est[(r+1)&1].  Every dropper
//   re-activates itself, so a vertex not evaluated in round r did not change
//   in round r-1 and its est[(r+1)&1] entry (written two rounds ago) is
//   already current: no drop list, no apply pass.  Neighbours are activated
//   with the extended rule judged on the snapshot (SURVEY §7.3 rule C).
// Reference rule (exact RunReport counters), three barriers per round:
//   evaluate (droppers record new/old value), apply (fastk.cpp:153), notify
//   on settled values (fastk.cpp:156-163).
// Per round every CTA first caches est[0, cache_n) — the highest-degree ids —
// in shared memory.  No host synchronisation happens between rounds.
#include <cooperative_groups.h>
#include <cstdint>

#include "kc_internal.h"

namespace cg = cooperative_groups;

namespace kcb {
namespace {

constexpr unsigned FULL = 0xffffffffu;
// Chunk sizes (ids) grabbed per atomic, per class.
constexpr uint32_t CH_BIG = 1, CH_WARP = 8, CH_SUB = 32, CH_THREAD = 256, CH_NOTIFY = 32;

template <typename OffT, typename EstT>
struct P {
  const OffT* off;
  const uint32_t* adj;
  uint32_t n_nz;
  uint32_t cb[NCLS + 1];
  EstT* est[2];
  EstT* old;
  uint8_t* flag[2];
  uint8_t* dropped;
  Ctl* ctl;
  uint32_t* anydrop;
  RoundStat* stats;
  uint32_t* status;
  unsigned long long* prof;
  uint32_t r_begin, r_end;
  int rule;
  uint32_t cache_n;
};

// What one round reads and writes (resolved once per round).
template <typename EstT>
struct RoundView {
  const EstT* snap;  // estimates read this round
  EstT* next;        // snapshot rule: new values of evaluated vertices
  uint8_t* fcur;     // frontier flags read + cleared this round
  uint8_t* fnxt;     // activations for the next round
  uint32_t* grab;    // chunk cursors of this round
  bool snapshot;     // snapshot rule (else reference rule)
  bool ext;          // extended_notify
};

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint32_t lanemask_lt() { return (1u << lane_id()) - 1u; }
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Estimate of v in this round's snapshot: shared-memory cache for the
// highest-degree ids, global (L1/L2) otherwise.
// One generic load per gather (the pointer selects shared or global memory),
// which keeps the many inlined gather sites small for the instruction cache.
template <typename EstT>
__device__ __forceinline__ uint32_t est_at(const EstT* __restrict__ s_cache, uint32_t cache_n,
                                           const EstT* snap, uint32_t v) {
#ifdef KC_NO_SMEM_CACHE
  (void)s_cache; (void)cache_n;
  return (uint32_t)snap[v];
#else
  const EstT* base = v < cache_n ? s_cache : snap;
  return (uint32_t)base[v];
#endif
}

// Activation predicate for neighbour estimate x after a drop cap -> t
// (t < cap): should_notify(t, cap, x) (fastk.hpp:25-27) or, with
// extended_notify off, the plain guard x > t (fastk.cpp:22-24).
__device__ __forceinline__ bool fires(bool ext, uint32_t t, uint32_t cap, uint32_t x) {
  return ext ? (t < x && x <= cap) : (x > t);
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, v, d);
    if (lane >= (uint32_t)d) v += y;
  }
  return v;
}

// ------------------------------------------------------------------------
// Values held in registers: R per lane.  16-bit estimates are < 2^15
// (EST16_LIMIT), so two share a register and "x >= t" for both halves is
// one OR + one subtract: the top bit of ((x | 0x8000) - t) is set iff x >= t.
// ------------------------------------------------------------------------
template <typename EstT, int R>
struct Vals;

template <int R>
struct Vals<uint16_t, R> {
  static_assert(R % 2 == 0, "pairs");
  uint32_t w[R / 2];
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int j = 0; j < R / 2; ++j) w[j] = 0;
  }
  __device__ __forceinline__ void set(int j, uint32_t x) {
    if (j & 1) w[j >> 1] |= x << 16; else w[j >> 1] |= x;
  }
  __device__ __forceinline__ uint32_t get(int j) const {
    return (j & 1) ? (w[j >> 1] >> 16) : (w[j >> 1] & 0xffffu);
  }
  __device__ __forceinline__ uint32_t count_ge(uint32_t t) const {
    const uint32_t tt = t | (t << 16);
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < R / 2; ++j) c += __popc(((w[j] | 0x80008000u) - tt) & 0x80008000u);
    return c;
  }
};

template <int R>
struct Vals<uint32_t, R> {
  uint32_t w[R];
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int j = 0; j < R; ++j) w[j] = 0;
  }
  __device__ __forceinline__ void set(int j, uint32_t x) { w[j] = x; }
  __device__ __forceinline__ uint32_t get(int j) const { return w[j]; }
  __device__ __forceinline__ uint32_t count_ge(uint32_t t) const {
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) c += w[j] >= t;
    return c;
  }
};

// 128-bit load of the 4 neighbour ids at aligned position a (multiple of 4).
// The adjacency is immutable for the kernel's lifetime: non-coherent path,
// no L1 allocation (L1 is left to the estimate gathers).
__device__ __forceinline__ uint4 ld_ids4(const uint32_t* adj, uint64_t a) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(adj + a));
  return r;
}
__device__ __forceinline__ uint32_t u4_get(const uint4& q, int e) {
  return e == 0 ? q.x : e == 1 ? q.y : e == 2 ? q.z : q.w;
}

// ------------------------------------------------------------------------
// Block-wide helpers (blockDim == SOLVE_THREADS)
// ------------------------------------------------------------------------
constexpr uint32_t NWARPS = SOLVE_THREADS / 32;

__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t* s_red) {
  v = __reduce_add_sync(FULL, v);
  if (lane_id() == 0) s_red[warp_id()] = v;
  __syncthreads();
  if (warp_id() == 0) {
    uint32_t w = __reduce_add_sync(FULL, lane_id() < NWARPS ? s_red[lane_id()] : 0u);
    if (lane_id() == 0) s_red[32] = w;
  }
  __syncthreads();
  return s_red[32];
}

__device__ __forceinline__ uint32_t block_min(uint32_t v, uint32_t* s_red) {
  v = __reduce_min_sync(FULL, v);
  if (lane_id() == 0) s_red[warp_id()] = v;
  __syncthreads();
  if (warp_id() == 0) {
    uint32_t w = __reduce_min_sync(FULL, lane_id() < NWARPS ? s_red[lane_id()] : 0xffffffffu);
    if (lane_id() == 0) s_red[32] = w;
  }
  __syncthreads();
  return s_red[32];
}

// Exclusive prefix sum over the block (thread order).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_red) {
  const uint32_t incl = warp_incl_scan(v);
  if (lane_id() == 31) s_red[warp_id()] = incl;
  __syncthreads();
  if (warp_id() == 0) {
    const uint32_t w = lane_id() < NWARPS ? s_red[lane_id()] : 0u;
    const uint32_t e = warp_incl_scan(w) - w;
    if (lane_id() < NWARPS) s_red[lane_id()] = e;
  }
  __syncthreads();
  const uint32_t r = s_red[warp_id()] + incl - v;
  __syncthreads();
  return r;
}

struct Acc {  // per-thread counters, flushed per round
  unsigned long long evals, escan, drops, fires;
  bool any_drop;
};

// Windowed histogram step of compute_index_over (kernel.hpp:31-41).  The
// window holds levels [top - NB, top): bin i counts values x == top-1-i;
// C counts values >= top.  Returns the smallest bin i whose level
// x = top-1-i >= 1 satisfies C + sum(bins[0..i]) >= x, or 0xffffffff.
// Warp version: lane l owns bins [8l, 8l+8).
__device__ __forceinline__ uint32_t warp_resolve(const uint32_t* bins, uint32_t C, uint32_t top) {
  static_assert(WARP_BINS == 256, "8 bins per lane");
  const uint32_t lane = lane_id();
  const uint4 b0 = reinterpret_cast<const uint4*>(bins)[2 * lane];
  const uint4 b1 = reinterpret_cast<const uint4*>(bins)[2 * lane + 1];
  const uint32_t b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += b[j];
  uint32_t run = C + warp_incl_scan(s) - s;
  uint32_t found = 0xffffffffu;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    run += b[j];
    const int i = (int)lane * 8 + j;
    const int x = (int)top - 1 - i;
    if (found == 0xffffffffu && x >= 1 && run >= (uint32_t)x) found = (uint32_t)i;
  }
  return __reduce_min_sync(FULL, found);
}

__device__ __forceinline__ void warp_zero_bins(uint32_t* bins) {
  const uint32_t lane = lane_id();
  reinterpret_cast<uint4*>(bins)[2 * lane] = make_uint4(0, 0, 0, 0);
  reinterpret_cast<uint4*>(bins)[2 * lane + 1] = make_uint4(0, 0, 0, 0);
  __syncwarp();
}

// Tally one gathered value into the window [top - NB, top).
template <int NB>
__device__ __forceinline__ void tally(uint32_t x, uint32_t top, uint32_t& above, uint32_t* bins) {
  if (x >= top) ++above;
  else if ((int)x >= (int)top - NB) atomicAdd(&bins[top - 1 - x], 1u);
}

// ------------------------------------------------------------------------
// Streaming over a row with 128-bit id loads: each of NT cooperating threads
// takes 8 entries per step (two 16-byte loads, software-pipelined one step
// ahead), gathers their 8 estimates, then hands (valid mask, ids, estimates)
// to the callback.  Rows need not be 16-byte aligned: positions outside
// [ob, oe) are masked (the adjacency has ADJ_PAD spare entries).
// ------------------------------------------------------------------------
template <int NT, typename OffT, typename EstT, typename F>
__device__ __forceinline__ void stream_row(const P<OffT, EstT>& p, const EstT* snap, uint32_t me,
                                           uint64_t ob, uint64_t oe, const EstT* s_cache,
                                           uint32_t cache_n, F&& f) {
  constexpr uint64_t STEP = (uint64_t)NT * 8;
  uint64_t a = ob & ~(uint64_t)3;
  uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0;
  if (a + 4 * me < oe) q0 = ld_ids4(p.adj, a + 4 * me);
  if (a + 4 * me + 4 * NT < oe) q1 = ld_ids4(p.adj, a + 4 * me + 4 * NT);
  for (; a < oe; a += STEP) {
    uint4 n0 = make_uint4(0, 0, 0, 0), n1 = n0;
    const uint64_t nb = a + STEP;
    if (nb + 4 * me < oe) n0 = ld_ids4(p.adj, nb + 4 * me);
    if (nb + 4 * me + 4 * NT < oe) n1 = ld_ids4(p.adj, nb + 4 * me + 4 * NT);
    uint32_t ids[8], x[8];
    uint32_t ok = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint64_t pos = a + 4 * me + (k >> 2) * 4 * NT + (k & 3);
      ids[k] = u4_get(k < 4 ? q0 : q1, k & 3);
      const bool v = pos >= ob && pos < oe;
      ok |= (uint32_t)v << k;
      x[k] = v ? est_at(s_cache, cache_n, snap, ids[k]) : 0u;
    }
    f(ok, ids, x);
    q0 = n0;
    q1 = n1;
  }
}

// Record one evaluation result.  Snapshot rule: write the new value of every
// evaluated vertex (keeps the double buffer current) and self-activate on a
// drop.  Reference rule: droppers record new/old values and a dropped mark
// for the apply and notify phases.
template <typename OffT, typename EstT>
__device__ __forceinline__ void finish_eval(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                                            uint32_t u, uint32_t t, uint32_t cap, Acc& acc) {
  if (rv.snapshot) {
    rv.next[u] = (EstT)t;
    if (t < cap) rv.fnxt[u] = 1;
  } else if (t < cap) {
    p.est[1][u] = (EstT)t;
    p.old[u] = (EstT)cap;
    p.dropped[u] = 1;
  }
  if (t < cap) {
    acc.drops += 1;
    acc.any_drop = true;
  }
}

// ------------------------------------------------------------------------
// Frontier scan: a warp grabs CH ids of class `cls` at a time, reads their
// flags four per lane (one 32-bit load), clears the set ones, and hands
// batches of up to 32 active ids (compacted in the warp's shared list) to
// `proc(list, n)`.
// ------------------------------------------------------------------------
template <uint32_t CH, bool ACCUM, typename F>
__device__ __forceinline__ void scan_class(uint8_t* flags, uint32_t* grab, uint32_t b0,
                                           uint32_t b1, uint32_t* list, F&& proc) {
  const uint32_t lane = lane_id();
  uint32_t cnt = 0;  // warp-uniform
  for (;;) {
    uint32_t start = 0;
    if (lane == 0) start = atomicAdd(grab, CH);
    start = __shfl_sync(FULL, start, 0);
    const uint32_t lo = b0 + start;
    if (start >= b1 - b0) break;
    const uint32_t hi = lo + CH < b1 ? lo + CH : b1;
    for (uint32_t s = lo & ~3u; s < hi; s += 128) {
      const uint32_t a = s + 4 * lane;
      uint32_t w = a < hi ? *reinterpret_cast<const uint32_t*>(flags + a) : 0u;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t id = a + b;
        const bool act = (w >> (8 * b) & 0xffu) && id >= lo && id < hi;
        if (act) flags[id] = 0;
        const uint32_t m = __ballot_sync(FULL, act);
        if (act) list[cnt + __popc(m & lanemask_lt())] = id;
        cnt += __popc(m);
        if (cnt >= 32) {
          __syncwarp();
          proc(list, 32u);
          __syncwarp();
          if (lane < cnt - 32) list[lane] = list[32 + lane];
          __syncwarp();
          cnt -= 32;
        }
      }
    }
    if (!ACCUM && cnt) {  // warp-per-vertex classes: no batching across chunks
      __syncwarp();
      proc(list, cnt);
      __syncwarp();
      cnt = 0;
    }
  }
  if (cnt) {
    __syncwarp();
    proc(list, cnt);
    __syncwarp();
  }
}

// ------------------------------------------------------------------------
// HUGE class: CTA per vertex (deg > DEG_BIG_MAX).  Pass A only counts
// values >= cap in registers ("no change" — the common case after the first
// rounds — costs one read of the row and one block reduction).  A drop runs
// windowed histogram passes: values >= top in registers, the window
// [top - HIST_BINS, top) binned in shared memory; then, under the snapshot
// rule, one more pass activates neighbours.  Re-reads hit L2.
// ------------------------------------------------------------------------
template <typename OffT, typename EstT>
__device__ __noinline__ uint32_t huge_window(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                                             const EstT* s_cache, uint32_t* s_hist,
                                             uint32_t* s_red, uint64_t ob, uint64_t oe,
                                             uint32_t cap) {
  const uint32_t tid = threadIdx.x;
  uint32_t top = cap;
  for (;;) {
    for (int i = tid; i < HIST_BINS; i += SOLVE_THREADS) s_hist[i] = 0;
    __syncthreads();
    uint32_t above = 0;
    stream_row<SOLVE_THREADS>(p, rv.snap, tid, ob, oe, s_cache, p.cache_n,
                              [&](uint32_t ok, const uint32_t(&)[8], const uint32_t(&x)[8]) {
#pragma unroll
                                for (int k = 0; k < 8; ++k)
                                  if (ok >> k & 1) tally<HIST_BINS>(x[k], top, above, s_hist);
                              });
    const uint32_t C = block_sum(above, s_red);
    uint32_t h[HIST_BINS / SOLVE_THREADS];
    uint32_t sm = 0;
#pragma unroll
    for (int j = 0; j < HIST_BINS / SOLVE_THREADS; ++j) {
      h[j] = s_hist[tid * (HIST_BINS / SOLVE_THREADS) + j];
      sm += h[j];
    }
    uint32_t run = C + block_excl_scan(sm, s_red);
    uint32_t found = 0xffffffffu;
#pragma unroll
    for (int j = 0; j < HIST_BINS / SOLVE_THREADS; ++j) {
      run += h[j];
      const int i = tid * (HIST_BINS / SOLVE_THREADS) + j;
      const int x = (int)top - 1 - i;
      if (found == 0xffffffffu && x >= 1 && run >= (uint32_t)x) found = (uint32_t)i;
    }
    found = block_min(found, s_red);
    if (found != 0xffffffffu) return top - 1 - found;
    if ((int)top - HIST_BINS <= 0) return 0;
    top -= HIST_BINS;
  }
}

template <typename OffT, typename EstT>
__device__ void eval_huge(const P<OffT, EstT>& p, const RoundView<EstT>& rv, const EstT* s_cache,
                          uint32_t* s_hist, uint32_t* s_red, uint32_t* s_item, Acc& acc) {
  const uint32_t tid = threadIdx.x;
  const uint32_t b0 = p.cb[C_HUGE], b1 = p.cb[C_HUGE + 1];
  for (;;) {
    if (tid == 0) {
      uint32_t u = 0xffffffffu;
      for (;;) {  // next active HUGE vertex
        const uint32_t k = atomicAdd(&rv.grab[C_HUGE], 1u);
        if (k >= b1 - b0) break;
        if (rv.fcur[b0 + k]) {
          rv.fcur[b0 + k] = 0;
          u = b0 + k;
          break;
        }
      }
      *s_item = u;
    }
    __syncthreads();
    const uint32_t u = *s_item;
    __syncthreads();
    if (u == 0xffffffffu) break;
    const uint64_t ob = p.off[u], oe = p.off[u + 1];
    const uint32_t cap = est_at(s_cache, p.cache_n, rv.snap, u);
    uint32_t c = 0;
    stream_row<SOLVE_THREADS>(p, rv.snap, tid, ob, oe, s_cache, p.cache_n,
                              [&](uint32_t ok, const uint32_t(&)[8], const uint32_t(&x)[8]) {
#pragma unroll
                                for (int k = 0; k < 8; ++k) c += (ok >> k & 1) && x[k] >= cap;
                              });
    uint32_t t = cap;
    if (block_sum(c, s_red) < cap) t = huge_window(p, rv, s_cache, s_hist, s_red, ob, oe, cap);
    if (tid == 0) {
      acc.evals += 1;
      acc.escan += oe - ob;
      finish_eval(p, rv, u, t, cap, acc);
    }
    if (t < cap && rv.snapshot) {  // re-stream the row (L2-resident) and activate
      stream_row<SOLVE_THREADS>(p, rv.snap, tid, ob, oe, s_cache, p.cache_n,
                                [&](uint32_t ok, const uint32_t(&ids)[8], const uint32_t(&x)[8]) {
#pragma unroll
                                  for (int k = 0; k < 8; ++k)
                                    if ((ok >> k & 1) && fires(rv.ext, t, cap, x[k])) {
                                      rv.fnxt[ids[k]] = 1;
                                      acc.fires += 1;
                                    }
                                });
    }
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
__device__ __forceinline__ Meta load_meta(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                                          const EstT* s_cache, const uint32_t* list, uint32_t n) {
  Meta m{0, 0, 0, 0};
  const uint32_t lane = lane_id();
  if (lane < n) {
    m.u = list[lane];
    m.ob = p.off[m.u];
    m.oe = p.off[m.u + 1];
    m.cap = est_at(s_cache, p.cache_n, rv.snap, m.u);
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

// Windowed histogram passes of one warp over a row (after pass A found a
// drop): returns the capped h-index.
template <typename OffT, typename EstT>
__device__ __noinline__ uint32_t warp_window(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                                             const EstT* s_cache, uint32_t* bins, uint64_t ob,
                                             uint64_t oe, uint32_t cap) {
  const uint32_t lane = lane_id();
  uint32_t top = cap;
  for (;;) {
    warp_zero_bins(bins);
    uint32_t above = 0;
    stream_row<32>(p, rv.snap, lane, ob, oe, s_cache, p.cache_n,
                   [&](uint32_t ok, const uint32_t(&)[8], const uint32_t(&x)[8]) {
#pragma unroll
                     for (int k = 0; k < 8; ++k)
                       if (ok >> k & 1) tally<WARP_BINS>(x[k], top, above, bins);
                   });
    __syncwarp();
    const uint32_t C = __reduce_add_sync(FULL, above);
    const uint32_t found = warp_resolve(bins, C, top);
    __syncwarp();
    if (found != 0xffffffffu) return top - 1 - found;
    if ((int)top - WARP_BINS <= 0) return 0;
    top -= WARP_BINS;
  }
}

// WARP and BIG classes: warp per vertex (DEG_SUB_MAX < deg <= DEG_BIG_MAX),
// 256 entries per warp step (two 128-bit id loads + 8 gathers per lane).
template <uint32_t CH, typename OffT, typename EstT>
__device__ void eval_wstream(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                             const EstT* s_cache, int cls, uint32_t* bins, uint32_t* list,
                             Acc& acc) {
  const uint32_t lane = lane_id();
  scan_class<CH, false>(rv.fcur, &rv.grab[cls], p.cb[cls], p.cb[cls + 1], list,
                        [&](const uint32_t* lst, uint32_t n) {
    const Meta mine = load_meta(p, rv, s_cache, lst, n);
    for (uint32_t i = 0; i < n; ++i) {
      const Meta it = shfl_meta(mine, i);
      const uint32_t cap = it.cap;
      uint32_t c = 0;
      stream_row<32>(p, rv.snap, lane, it.ob, it.oe, s_cache, p.cache_n,
                     [&](uint32_t ok, const uint32_t(&)[8], const uint32_t(&x)[8]) {
#pragma unroll
                       for (int k = 0; k < 8; ++k) c += (ok >> k & 1) && x[k] >= cap;
                     });
      uint32_t t = cap;
      if (__reduce_add_sync(FULL, c) < cap) t = warp_window(p, rv, s_cache, bins, it.ob, it.oe, cap);
      if (lane == 0) {
        acc.evals += 1;
        acc.escan += it.oe - it.ob;
        finish_eval(p, rv, it.u, t, cap, acc);
      }
      if (t < cap && rv.snapshot) {
        stream_row<32>(p, rv.snap, lane, it.ob, it.oe, s_cache, p.cache_n,
                       [&](uint32_t ok, const uint32_t(&ids)[8], const uint32_t(&x)[8]) {
#pragma unroll
                         for (int k = 0; k < 8; ++k)
                           if ((ok >> k & 1) && fires(rv.ext, t, cap, x[k])) {
                             rv.fnxt[ids[k]] = 1;
                             acc.fires += 1;
                           }
                       });
      }
    }
  });
}

// ------------------------------------------------------------------------
// SUB class: 8-lane tile per vertex (4 vertices per warp), 8 values per lane.
// ------------------------------------------------------------------------
__device__ __forceinline__ uint32_t tile8_sum(uint32_t v) {
  v += __shfl_xor_sync(FULL, v, 4, 8);
  v += __shfl_xor_sync(FULL, v, 2, 8);
  v += __shfl_xor_sync(FULL, v, 1, 8);
  return v;
}

template <typename OffT, typename EstT>
__device__ void eval_sub(const P<OffT, EstT>& p, const RoundView<EstT>& rv, const EstT* s_cache,
                         uint32_t* list, Acc& acc) {
  constexpr int R = DEG_SUB_MAX / 8;
  const uint32_t lane = lane_id(), g = lane >> 3, k = lane & 7;
  scan_class<CH_SUB, true>(rv.fcur, &rv.grab[C_SUB], p.cb[C_SUB], p.cb[C_SUB + 1], list,
                     [&](const uint32_t* lst, uint32_t n) {
    const Meta mine = load_meta(p, rv, s_cache, lst, n);
    for (uint32_t i0 = 0; i0 < n; i0 += 4) {
      // every lane runs the shuffles; tiles beyond n idle
      const Meta it = shfl_meta(mine, (int)(i0 + g) & 31);
      const bool has = i0 + g < n;
      const uint32_t u = it.u;
      const uint32_t deg = has ? (uint32_t)(it.oe - it.ob) : 0u;
      const uint32_t cap = has ? it.cap : 0u;
      uint32_t ids[R];
      Vals<EstT, R> vals;
      vals.clear();
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const uint32_t q = k + 8 * j;
        ids[j] = q < deg ? p.adj[it.ob + q] : 0xffffffffu;
      }
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (ids[j] != 0xffffffffu) vals.set(j, est_at(s_cache, p.cache_n, rv.snap, ids[j]));
      // capped h-index by bisection, all four tiles in lockstep
      const bool keep = tile8_sum(vals.count_ge(cap)) >= cap;
      uint32_t lo = 0, hi = cap;
#pragma unroll 1
      for (int s = 0; s < 7; ++s) {  // cap <= 64
        const uint32_t mid = (lo + hi) >> 1;
        const bool okm = tile8_sum(vals.count_ge(mid)) >= mid;
        if (hi - lo > 1) {
          if (okm) lo = mid; else hi = mid;
        }
      }
      const uint32_t t = keep ? cap : lo;
      if (has && k == 0) {
        acc.evals += 1;
        acc.escan += deg;
        finish_eval(p, rv, u, t, cap, acc);
      }
      if (has && t < cap && rv.snapshot) {
#pragma unroll
        for (int j = 0; j < R; ++j)
          if (ids[j] != 0xffffffffu && fires(rv.ext, t, cap, vals.get(j))) {
            rv.fnxt[ids[j]] = 1;
            acc.fires += 1;
          }
      }
    }
  });
}

// ------------------------------------------------------------------------
// THREAD class: one thread per vertex (deg <= 8), h-index = max_i min(x_i,
// #{j : x_j >= x_i}) — the classic h-index identity, capped at est[u].
// ------------------------------------------------------------------------
template <typename OffT, typename EstT>
__device__ void eval_thread(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                            const EstT* s_cache, uint32_t* list, Acc& acc) {
  constexpr int R = DEG_THREAD_MAX;
  const uint32_t lane = lane_id();
  scan_class<CH_THREAD, true>(rv.fcur, &rv.grab[C_THREAD], p.cb[C_THREAD], p.cb[C_THREAD + 1], list,
                        [&](const uint32_t* lst, uint32_t n) {
    if (lane >= n) return;
    const uint32_t u = lst[lane];
    const uint64_t ob = p.off[u];
    const uint32_t deg = (uint32_t)(p.off[u + 1] - ob);
    const uint32_t cap = est_at(s_cache, p.cache_n, rv.snap, u);
    uint32_t ids[R], x[R];
#pragma unroll
    for (int j = 0; j < R; ++j) ids[j] = (uint32_t)j < deg ? p.adj[ob + j] : 0xffffffffu;
#pragma unroll
    for (int j = 0; j < R; ++j)
      x[j] = ids[j] != 0xffffffffu ? est_at(s_cache, p.cache_n, rv.snap, ids[j]) : 0u;
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
    acc.evals += 1;
    acc.escan += deg;
    finish_eval(p, rv, u, t, cap, acc);
    if (t < cap && rv.snapshot) {
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (ids[j] != 0xffffffffu && fires(rv.ext, t, cap, x[j])) {
          rv.fnxt[ids[j]] = 1;
          acc.fires += 1;
        }
    }
  });
}

// ------------------------------------------------------------------------
// Reference rule, after the apply barrier: re-stream every dropper's row
// and activate on SETTLED estimates (fastk.cpp:156-163); warp per dropper.
// ------------------------------------------------------------------------
template <typename OffT, typename EstT>
__device__ void notify_settled(const P<OffT, EstT>& p, const RoundView<EstT>& rv,
                               uint32_t* list, Acc& acc) {
  const uint32_t lane = lane_id();
  scan_class<CH_NOTIFY, false>(p.dropped, &rv.grab[NCLS], 0u, p.n_nz, list,
                        [&](const uint32_t* lst, uint32_t n) {
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t u = lst[i];
      const uint32_t t = p.est[0][u], oc = p.old[u];
      const uint64_t ob = p.off[u], oe = p.off[u + 1];
      stream_row<32>(p, p.est[0], lane, ob, oe, (const EstT*)nullptr, 0u,
                     [&](uint32_t ok, const uint32_t(&ids)[8], const uint32_t(&x)[8]) {
#pragma unroll
                       for (int j = 0; j < 8; ++j)
                         if ((ok >> j & 1) && fires(rv.ext, t, oc, x[j])) {
                           rv.fnxt[ids[j]] = 1;
                           acc.fires += 1;
                         }
                     });
    }
  });
}

template <typename OffT, typename EstT>
__device__ __forceinline__ void flush_acc(const P<OffT, EstT>& p, uint32_t sr, const Acc& acc,
                                          unsigned long long* s_acc) {
  unsigned long long v[4] = {acc.evals, acc.escan, acc.drops, acc.fires};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    unsigned long long x = v[q];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(FULL, x, d);
    if (lane_id() == 0 && x) atomicAdd(&s_acc[q], x);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (s_acc[q]) atomicAdd(&p.stats[sr].evals + q, s_acc[q]);
  }
}

template <typename OffT, typename EstT>
__global__ void __launch_bounds__(SOLVE_THREADS, 1) rounds_kernel(P<OffT, EstT> p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem[];
  EstT* s_cache = reinterpret_cast<EstT*>(smem);
  const size_t cache_bytes = ((size_t)p.cache_n * sizeof(EstT) + 15) & ~(size_t)15;
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(smem + cache_bytes);
  // per-warp regions (alias s_hist once the HUGE phase is over):
  // 256 histogram bins + a 64-entry active list
  uint32_t* w_bins = s_hist + (WARP_BINS + 64) * warp_id();
  uint32_t* w_list = w_bins + WARP_BINS;
  __shared__ uint32_t s_red[33];
  __shared__ uint32_t s_item;
  __shared__ uint32_t s_drop;
  __shared__ unsigned long long s_acc[4];
  const uint32_t tid = threadIdx.x;
  const uint32_t gtid = blockIdx.x * blockDim.x + tid;
  const uint32_t gsize = gridDim.x * blockDim.x;
  const bool snapshot = p.rule >= R_SNAP_EXT;

  for (uint32_t r = p.r_begin; r < p.r_end; ++r) {
    const uint32_t cur = r & 1, nxt = cur ^ 1;
    const uint32_t sr = r < STAT_SLOTS - 1 ? r : STAT_SLOTS - 1;
    RoundView<EstT> rv;
    rv.snap = snapshot ? p.est[cur] : p.est[0];
    rv.next = p.est[nxt];
    rv.fcur = p.flag[cur];
    rv.fnxt = p.flag[nxt];
    rv.grab = p.ctl[cur].grab;
    rv.snapshot = snapshot;
    rv.ext = p.rule == R_SNAP_EXT || p.rule == R_REF_EXT;
    unsigned long long* pf = (p.prof && r < PROF_ROUNDS && tid == 0)
                                 ? p.prof + ((size_t)r * gridDim.x + blockIdx.x) * PROF_PHASES
                                 : nullptr;
    if (pf) pf[0] = gtimer();
    // cursors and drop flag of the NEXT round (nobody touches them now)
    if (blockIdx.x == 0 && tid < NCLS + 2) p.ctl[nxt].grab[tid] = 0;
    if (blockIdx.x == 0 && tid == 32) p.anydrop[(r + 1) % 3] = 0;
    if (p.cache_n) {
      // vectorised cache fill: cache_n * sizeof(EstT) is a multiple of 16 bytes
      const uint4* src = reinterpret_cast<const uint4*>(rv.snap);
      uint4* dst = reinterpret_cast<uint4*>(s_cache);
      const uint32_t nvec = (uint32_t)((size_t)p.cache_n * sizeof(EstT) / 16);
      for (uint32_t i = tid; i < nvec; i += SOLVE_THREADS) dst[i] = src[i];
    }
    if (tid < 4) s_acc[tid] = 0;
    if (tid == 0) s_drop = 0;
    __syncthreads();
    Acc acc{0, 0, 0, 0, false};
    if (pf) pf[1] = gtimer();
    eval_huge(p, rv, s_cache, s_hist, s_red, &s_item, acc);
    if (pf) pf[2] = gtimer();
    eval_wstream<CH_BIG>(p, rv, s_cache, C_BIG, w_bins, w_list, acc);
    if (pf) pf[3] = gtimer();
    eval_wstream<CH_WARP>(p, rv, s_cache, C_WARP, w_bins, w_list, acc);
    if (pf) pf[4] = gtimer();
    eval_sub(p, rv, s_cache, w_list, acc);
    if (pf) pf[5] = gtimer();
    eval_thread(p, rv, s_cache, w_list, acc);
    if (pf) pf[6] = gtimer();
    if (__any_sync(FULL, acc.any_drop) && lane_id() == 0) s_drop = 1;
    flush_acc(p, sr, acc, s_acc);  // contains __syncthreads
    if (tid == 0 && s_drop) p.anydrop[r % 3] = 1;
    grid.sync();
    const bool any = *reinterpret_cast<volatile uint32_t*>(&p.anydrop[r % 3]) != 0;
    if (!any) {  // quiescent round: converged (fastk.cpp:109-110)
      if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = r + 1;
        p.status[1] = 1;
        p.status[3] = snapshot ? cur : 0;
      }
      if (pf) pf[7] = gtimer();
      return;
    }
    if (!snapshot) {
      // apply (fastk.cpp:153): est[u] = new value for every dropper
      const uint32_t nw = (p.n_nz + 3) / 4;
      for (uint32_t w = gtid; w < nw; w += gsize) {
        const uint32_t m = reinterpret_cast<const uint32_t*>(p.dropped)[w];
        if (!m) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (m >> (8 * b) & 0xffu) p.est[0][4 * w + b] = p.est[1][4 * w + b];
      }
      grid.sync();
      if (tid < 4) s_acc[tid] = 0;
      __syncthreads();
      Acc nacc{0, 0, 0, 0, false};
      notify_settled(p, rv, w_list, nacc);
      flush_acc(p, sr, nacc, s_acc);
      grid.sync();
    }
    if (pf) pf[7] = gtimer();
    if (blockIdx.x == 0 && tid == 0) {
      p.status[0] = r + 1;
      p.status[3] = snapshot ? nxt : 0;
    }
  }
}

// Round-0 state: est = min(deg, H) in both buffers (identical
// trajectory from round 1; the reference starts at deg, fastk.cpp:67-68),
// every non-isolated vertex flagged active, everything else cleared.
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
    p.est[0][u] = e;
    p.est[1][u] = e;
    p.flag[0][u] = u < p.n_nz ? 1 : 0;
    p.flag[1][u] = 0;
    p.dropped[u] = 0;
  }
  for (uint32_t k = gtid; k < STAT_SLOTS * (uint32_t)(sizeof(RoundStat) / 8); k += gsize)
    reinterpret_cast<unsigned long long*>(p.stats)[k] = 0;
  if (gtid < NCLS + 2) {
    p.ctl[0].grab[gtid] = 0;
    p.ctl[1].grab[gtid] = 0;
  }
  if (gtid < 3) p.anydrop[gtid] = 0;
  if (gtid < 4) p.status[gtid] = 0;
}

template <typename OffT, typename EstT>
P<OffT, EstT> make_params(const SolveBuffers& b) {
  P<OffT, EstT> p{};
  p.off = static_cast<const OffT*>(b.off);
  p.adj = b.adj;
  p.n_nz = b.n_nz;
  for (int c = 0; c <= NCLS; ++c) p.cb[c] = b.cls_begin[c];
  p.est[0] = static_cast<EstT*>(b.est[0]);
  p.est[1] = static_cast<EstT*>(b.est[1]);
  p.old = static_cast<EstT*>(b.old);
  p.flag[0] = b.flag[0];
  p.flag[1] = b.flag[1];
  p.dropped = b.dropped;
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
  const size_t warp_region = (size_t)32 * (WARP_BINS + 64);
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
  dim3 grid(c.num_sms), block(SOLVE_THREADS);
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
  // 227 KB opt-in per CTA: 128 KB of estimates + 40 KB of per-warp bins and
  // lists; the rest stays L1 for the estimate gathers.
  return 128 * 1024;
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
