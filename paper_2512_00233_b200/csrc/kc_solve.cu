// kc_solve.cu — the FastK coreness fixed point as ONE persistent cooperative
// kernel on sm_100a.
//
// Reference path (paths under /root/reference/proj):
//   fastk_run            src/fastk.cpp:57-187  — rounds of process | apply | notify
//   recompute_node       src/fastk.cpp:15-20   — gather est[nb] over the row
//   compute_index_over   include/kcore/kernel.hpp:27-42 — capped h-index
//   should_notify        include/kcore/fastk.hpp:25-27  — extended activation rule
//
// One round (Jacobi: every evaluation reads the round's snapshot, updates are
// applied after a grid barrier, exactly the reference's process/apply split):
//   1. every CTA caches est[0, cache_n) in shared memory (ids are sorted by
//      descending degree, so these are the most-gathered estimates);
//   2. evaluate the frontier, degree class by degree class (kc_internal.h):
//        HUGE/BLOCK  CTA per vertex, windowed shared-memory histogram of
//                    min(est_v, cap) + block suffix scan;
//        WARP        warp per vertex, 32 values per lane in registers (u16x2
//                    packed), counts by __vcmpgeu2 + __reduce_add_sync, search
//                    by bisection;
//        SUB         8-lane tile per vertex, same with shuffle reductions;
//        THREAD      thread per vertex, register h-index by pairwise counts;
//      droppers append (u, t) to the drop list and, under the snapshot rule,
//      push activations with a dedup bitmap + warp-aggregated queue appends;
//   3. grid.sync(); apply the drop list (fastk.cpp:153); reset cursors;
//   4. reference rule only: grid.sync(); notify on settled values
//      (fastk.cpp:156-163);
//   5. grid.sync().  A round with no drop ends the kernel (fastk.cpp:109-110).
// No host synchronisation happens between rounds.
#include <cooperative_groups.h>
#include <cstdint>

#include "kc_internal.h"

namespace cg = cooperative_groups;

namespace kcb {
namespace {

constexpr unsigned FULL = 0xffffffffu;

template <typename OffT, typename EstT>
struct P {
  const OffT* off;
  const uint32_t* adj;
  EstT* est;
  uint32_t n_nz;
  uint32_t cb[NCLS + 1];
  uint32_t* queue[2];
  uint32_t* qcnt;
  uint32_t* bm[2];
  uint32_t* drop_u;
  EstT* drop_t;
  EstT* drop_old;
  Ctl* ctl;
  RoundStat* stats;
  uint32_t* status;
  uint32_t r_begin, r_end;
  int rule;
  uint32_t cache_n;
  uint32_t tail_threshold;
};

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }

template <typename OffT, typename EstT>
__device__ __forceinline__ uint32_t class_of(const P<OffT, EstT>& p, uint32_t v) {
  return (v >= p.cb[1]) + (v >= p.cb[2]) + (v >= p.cb[3]) + (v >= p.cb[4]);
}

// Estimate of v in this round's snapshot: shared-memory cache for the
// highest-degree ids, global (L1/L2) otherwise.
template <typename EstT>
__device__ __forceinline__ uint32_t est_at(const EstT* __restrict__ s_cache, uint32_t cache_n,
                                           const EstT* est, uint32_t v) {
  return v < cache_n ? (uint32_t)s_cache[v] : (uint32_t)est[v];
}

// Snapshot activation predicate for neighbour estimate x after a drop
// cap -> t (t < cap).  SNAP_EXT: should_notify(t, cap, x) (fastk.hpp:25-27);
// SNAP_PLAIN: the plain guard x > t (fastk.cpp:22-24 with extended off).
__device__ __forceinline__ bool snap_fire(int rule, uint32_t t, uint32_t cap, uint32_t x) {
  return rule == R_SNAP_EXT ? (t < x && x <= cap) : (x > t);
}

// Warp-cooperative activation: all 32 lanes must call.  Dedup through the
// next round's bitmap (plain read first, then atomicOr), then one queue
// append per (warp, class) with warp-aggregated atomics.
template <typename OffT, typename EstT>
__device__ __forceinline__ void warp_push(const P<OffT, EstT>& p, uint32_t nxt, uint32_t v,
                                          bool want) {
  if (want) {
    const uint32_t bit = 1u << (v & 31);
    uint32_t* w = p.bm[nxt] + (v >> 5);
    if (*reinterpret_cast<volatile uint32_t*>(w) & bit)
      want = false;
    else
      want = !(atomicOr(w, bit) & bit);
  }
  uint32_t any = __ballot_sync(FULL, want);
  if (!any) return;
  const uint32_t c = want ? class_of(p, v) : NCLS;
  const uint32_t lane = lane_id();
  while (any) {
    const uint32_t leader = __ffs(any) - 1;
    const uint32_t cc = __shfl_sync(FULL, c, leader);
    const uint32_t m = __ballot_sync(FULL, want && c == cc);
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(&p.qcnt[nxt * NCLS + cc], __popc(m));
    base = __shfl_sync(FULL, base, leader);
    if (want && c == cc) p.queue[nxt][p.cb[cc] + base + __popc(m & ((1u << lane) - 1u))] = v;
    any &= ~m;
  }
}

template <typename OffT, typename EstT>
__device__ __forceinline__ void record_drop(const P<OffT, EstT>& p, uint32_t cur, uint32_t u,
                                            uint32_t t, uint32_t cap) {
  const uint32_t k = atomicAdd(&p.ctl[cur].ndrops, 1u);
  p.drop_u[k] = u;
  p.drop_t[k] = (EstT)t;
  p.drop_old[k] = (EstT)cap;
}

// ------------------------------------------------------------------------
// Values held in registers: R per lane.  For 16-bit estimates two values
// share one register and counts use the SIMD compare __vcmpgeu2.
// ------------------------------------------------------------------------
template <typename EstT, int R>
struct Vals;

template <int R>
struct Vals<uint16_t, R> {
  uint32_t w[(R + 1) / 2];
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int j = 0; j < (R + 1) / 2; ++j) w[j] = 0;
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
    for (int j = 0; j < (R + 1) / 2; ++j) c += __popc(__vcmpgeu2(w[j], tt) & 0x00010001u);
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

// ------------------------------------------------------------------------
// Block-wide helpers (blockDim == SOLVE_THREADS)
// ------------------------------------------------------------------------
__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t* s_red) {
  v = __reduce_add_sync(FULL, v);
  if (lane_id() == 0) s_red[warp_id()] = v;
  __syncthreads();
  if (warp_id() == 0) {
    uint32_t w = __reduce_add_sync(FULL, s_red[lane_id()]);
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
    uint32_t w = __reduce_min_sync(FULL, s_red[lane_id()]);
    if (lane_id() == 0) s_red[32] = w;
  }
  __syncthreads();
  return s_red[32];
}

// Exclusive prefix sum over the block (thread order).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_red) {
  const uint32_t lane = lane_id();
  uint32_t incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(FULL, incl, d);
    if (lane >= (uint32_t)d) incl += y;
  }
  if (lane == 31) s_red[warp_id()] = incl;
  __syncthreads();
  if (warp_id() == 0) {
    uint32_t w = s_red[lane];
    uint32_t wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_up_sync(FULL, wi, d);
      if (lane >= (uint32_t)d) wi += y;
    }
    s_red[lane] = wi - w;
  }
  __syncthreads();
  const uint32_t r = s_red[warp_id()] + incl - v;
  __syncthreads();
  return r;
}

struct Acc {  // per-thread counters, flushed per round
  unsigned long long evals, escan, drops, fires;
};

// ------------------------------------------------------------------------
// HUGE / BLOCK classes: one CTA per vertex.  compute_index_over's histogram
// (kernel.hpp:31-41) restricted to a window of HIST_BINS levels below `top`;
// values >= top are counted in registers (no shared atomics on the top bin).
// The first window starts at cap, which resolves "no change" and every drop
// smaller than HIST_BINS in one pass; lower windows re-read the row.
// ------------------------------------------------------------------------
template <typename OffT, typename EstT>
__device__ void eval_block_items(const P<OffT, EstT>& p, uint32_t r, const EstT* s_cache,
                                 uint32_t* s_hist, uint32_t* s_red, uint32_t* s_item, Acc& acc) {
  const uint32_t cur = r & 1, nxt = cur ^ 1;
  const uint32_t tid = threadIdx.x;
  const bool snap = p.rule >= R_SNAP_EXT;
  for (int c = C_HUGE; c <= C_BLOCK; ++c) {
    const uint32_t cnt = p.qcnt[cur * NCLS + c];
    for (;;) {
      if (tid == 0) *s_item = atomicAdd(&p.ctl[cur].grab[c], 1u);
      __syncthreads();
      const uint32_t idx = *s_item;
      __syncthreads();
      if (idx >= cnt) break;
      const uint32_t u = p.queue[cur][p.cb[c] + idx];
      if (tid == 0) p.bm[cur][u >> 5] = 0;  // retire this round's dedup bits
      const OffT ob = p.off[u], oe = p.off[u + 1];
      const uint32_t cap = est_at(s_cache, p.cache_n, p.est, u);
      uint32_t top = cap, t = cap;
      for (int pass = 0;; ++pass) {
        for (int i = tid; i < HIST_BINS; i += SOLVE_THREADS) s_hist[i] = 0;
        __syncthreads();
        const int lo = (int)top - HIST_BINS;  // window holds values in [lo, top)
        uint32_t above = 0;
        for (OffT i = ob + tid; i < oe; i += SOLVE_THREADS) {
          const uint32_t x = est_at(s_cache, p.cache_n, p.est, p.adj[i]);
          if (x >= top) ++above;
          else if ((int)x >= lo) atomicAdd(&s_hist[top - 1 - x], 1u);
        }
        const uint32_t C = block_sum(above, s_red);
        if (pass == 0 && C >= cap) break;  // t = cap: no change
        // smallest bin i (largest level x = top-1-i >= 1) with
        // C + sum(hist[0..i]) >= x
        uint32_t h[HIST_BINS / SOLVE_THREADS];
        uint32_t s = 0;
#pragma unroll
        for (int j = 0; j < HIST_BINS / SOLVE_THREADS; ++j) {
          h[j] = s_hist[tid * (HIST_BINS / SOLVE_THREADS) + j];
          s += h[j];
        }
        uint32_t run = C + block_excl_scan(s, s_red);
        uint32_t found = 0xffffffffu;
#pragma unroll
        for (int j = 0; j < HIST_BINS / SOLVE_THREADS; ++j) {
          run += h[j];
          const int i = tid * (HIST_BINS / SOLVE_THREADS) + j;
          const int x = (int)top - 1 - i;
          if (found == 0xffffffffu && x >= 1 && run >= (uint32_t)x) found = (uint32_t)i;
        }
        found = block_min(found, s_red);
        if (found != 0xffffffffu) {
          t = top - 1 - found;
          break;
        }
        if (lo <= 0) {
          t = 0;
          break;
        }
        top = (uint32_t)lo;
      }
      if (tid == 0) {
        acc.evals += 1;
        acc.escan += (unsigned long long)(oe - ob);
      }
      if (t < cap) {
        if (tid == 0) {
          acc.drops += 1;
          record_drop(p, cur, u, t, cap);
        }
        if (snap) {
          // re-read the row (L2-resident: just streamed) and activate
          const uint32_t lane = lane_id();
          for (OffT base = ob + warp_id() * 32; base < oe; base += SOLVE_THREADS) {
            const OffT i = base + lane;
            bool want = false;
            uint32_t v = 0;
            if (i < oe) {
              v = p.adj[i];
              want = snap_fire(p.rule, t, cap, est_at(s_cache, p.cache_n, p.est, v));
            }
            acc.fires += want;
            warp_push(p, nxt, v, want);
          }
          if (p.rule == R_SNAP_EXT && warp_id() == 0) warp_push(p, nxt, u, lane == 0);
        }
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------------
// WARP class: warp per vertex, up to 32 values per lane (entry lane + 32 j).
// ------------------------------------------------------------------------
template <typename OffT, typename EstT>
__device__ void eval_warp_items(const P<OffT, EstT>& p, uint32_t r, const EstT* s_cache,
                                Acc& acc) {
  constexpr int R = DEG_WARP_MAX / 32;
  const uint32_t cur = r & 1, nxt = cur ^ 1;
  const uint32_t lane = lane_id();
  const bool snap = p.rule >= R_SNAP_EXT;
  const uint32_t cnt = p.qcnt[cur * NCLS + C_WARP];
  for (;;) {
    uint32_t idx = 0;
    if (lane == 0) idx = atomicAdd(&p.ctl[cur].grab[C_WARP], 1u);
    idx = __shfl_sync(FULL, idx, 0);
    if (idx >= cnt) break;
    const uint32_t u = p.queue[cur][p.cb[C_WARP] + idx];
    if (lane == 0) p.bm[cur][u >> 5] = 0;
    const OffT ob = p.off[u];
    const uint32_t deg = (uint32_t)(p.off[u + 1] - ob);
    const uint32_t cap = est_at(s_cache, p.cache_n, p.est, u);
    Vals<EstT, R> vals;
    vals.clear();
    {
      uint32_t ids[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const uint32_t i = lane + 32 * j;
        ids[j] = i < deg ? p.adj[ob + i] : 0xffffffffu;
      }
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (ids[j] != 0xffffffffu) vals.set(j, est_at(s_cache, p.cache_n, p.est, ids[j]));
    }
    uint32_t t;
    if (__reduce_add_sync(FULL, vals.count_ge(cap)) >= cap) {
      t = cap;
    } else {  // invariant: count(>= lo) >= lo, count(>= hi) < hi
      uint32_t lo = 0, hi = cap;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__reduce_add_sync(FULL, vals.count_ge(mid)) >= mid) lo = mid; else hi = mid;
      }
      t = lo;
    }
    if (lane == 0) {
      acc.evals += 1;
      acc.escan += deg;
    }
    if (t < cap) {
      if (lane == 0) {
        acc.drops += 1;
        record_drop(p, cur, u, t, cap);
      }
      if (snap) {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if (32 * j >= deg) break;  // warp-uniform
          const uint32_t i = lane + 32 * j;
          bool want = false;
          uint32_t v = 0;
          if (i < deg) {
            v = p.adj[ob + i];
            want = snap_fire(p.rule, t, cap, vals.get(j));
          }
          acc.fires += want;
          warp_push(p, nxt, v, want);
        }
        if (p.rule == R_SNAP_EXT) warp_push(p, nxt, u, lane == 0);
      }
    }
  }
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
__device__ void eval_sub_items(const P<OffT, EstT>& p, uint32_t r, const EstT* s_cache,
                               Acc& acc) {
  constexpr int R = DEG_SUB_MAX / 8;
  const uint32_t cur = r & 1, nxt = cur ^ 1;
  const uint32_t lane = lane_id(), g = lane >> 3, k = lane & 7;
  const bool snap = p.rule >= R_SNAP_EXT;
  const uint32_t cnt = p.qcnt[cur * NCLS + C_SUB];
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(&p.ctl[cur].grab[C_SUB], 4u);
    base = __shfl_sync(FULL, base, 0);
    if (base >= cnt) break;
    const uint32_t idx = base + g;
    const bool has = idx < cnt;
    uint32_t u = 0, deg = 0, cap = 0;
    OffT ob = 0;
    if (has) {
      u = p.queue[cur][p.cb[C_SUB] + idx];
      ob = p.off[u];
      deg = (uint32_t)(p.off[u + 1] - ob);
      cap = est_at(s_cache, p.cache_n, p.est, u);
      if (k == 0) p.bm[cur][u >> 5] = 0;
    }
    uint32_t ids[R];
    Vals<EstT, R> vals;
    vals.clear();
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const uint32_t i = k + 8 * j;
      ids[j] = i < deg ? p.adj[ob + i] : 0xffffffffu;
    }
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (ids[j] != 0xffffffffu) vals.set(j, est_at(s_cache, p.cache_n, p.est, ids[j]));
    // capped h-index by bisection, all four tiles in lockstep
    uint32_t t;
    const bool keep = tile8_sum(vals.count_ge(cap)) >= cap;
    uint32_t lo = 0, hi = cap;
#pragma unroll 1
    for (int s = 0; s < 7; ++s) {  // cap <= 64
      const uint32_t mid = (lo + hi) >> 1;
      const bool ok = tile8_sum(vals.count_ge(mid)) >= mid;
      if (hi - lo > 1) {
        if (ok) lo = mid; else hi = mid;
      }
    }
    t = keep ? cap : lo;
    const bool dropped = has && t < cap;
    if (has && k == 0) {
      acc.evals += 1;
      acc.escan += deg;
      if (dropped) {
        acc.drops += 1;
        record_drop(p, cur, u, t, cap);
      }
    }
    if (snap && __any_sync(FULL, dropped)) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const bool want = dropped && ids[j] != 0xffffffffu && snap_fire(p.rule, t, cap, vals.get(j));
        acc.fires += want;
        warp_push(p, nxt, ids[j], want);
      }
      if (p.rule == R_SNAP_EXT) warp_push(p, nxt, u, dropped && k == 0);
    }
  }
}

// ------------------------------------------------------------------------
// THREAD class: one thread per vertex (deg <= 8), h-index = max_i min(x_i,
// #{j : x_j >= x_i}) — the classic h-index identity, capped at est[u].
// ------------------------------------------------------------------------
template <typename OffT, typename EstT>
__device__ void eval_thread_items(const P<OffT, EstT>& p, uint32_t r, const EstT* s_cache,
                                  Acc& acc) {
  constexpr int R = DEG_THREAD_MAX;
  const uint32_t cur = r & 1, nxt = cur ^ 1;
  const uint32_t lane = lane_id();
  const bool snap = p.rule >= R_SNAP_EXT;
  const uint32_t cnt = p.qcnt[cur * NCLS + C_THREAD];
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(&p.ctl[cur].grab[C_THREAD], 32u);
    base = __shfl_sync(FULL, base, 0);
    if (base >= cnt) break;
    const uint32_t idx = base + lane;
    const bool has = idx < cnt;
    uint32_t u = 0, deg = 0, cap = 0;
    OffT ob = 0;
    if (has) {
      u = p.queue[cur][p.cb[C_THREAD] + idx];
      ob = p.off[u];
      deg = (uint32_t)(p.off[u + 1] - ob);
      cap = est_at(s_cache, p.cache_n, p.est, u);
      p.bm[cur][u >> 5] = 0;
    }
    uint32_t ids[R], x[R];
#pragma unroll
    for (int j = 0; j < R; ++j) ids[j] = (uint32_t)j < deg ? p.adj[ob + j] : 0xffffffffu;
#pragma unroll
    for (int j = 0; j < R; ++j)
      x[j] = ids[j] != 0xffffffffu ? est_at(s_cache, p.cache_n, p.est, ids[j]) : 0u;
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
    const bool dropped = has && t < cap;
    if (has) {
      acc.evals += 1;
      acc.escan += deg;
      if (dropped) {
        acc.drops += 1;
        record_drop(p, cur, u, t, cap);
      }
    }
    if (snap && __any_sync(FULL, dropped)) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const bool want = dropped && ids[j] != 0xffffffffu && snap_fire(p.rule, t, cap, x[j]);
        acc.fires += want;
        warp_push(p, nxt, ids[j], want);
      }
      if (p.rule == R_SNAP_EXT) warp_push(p, nxt, u, dropped);
    }
  }
}

// ------------------------------------------------------------------------
// Reference notify phase on SETTLED estimates (fastk.cpp:156-163): each
// dropper's row is re-scanned after the apply barrier; a warp per dropper.
// ------------------------------------------------------------------------
template <typename OffT, typename EstT>
__device__ void notify_settled(const P<OffT, EstT>& p, uint32_t r, uint32_t nd, Acc& acc) {
  const uint32_t nxt = (r & 1) ^ 1;
  const uint32_t lane = lane_id();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const bool ext = p.rule == R_REF_EXT;
  for (uint32_t k = gw; k < nd; k += nw) {
    const uint32_t u = p.drop_u[k];
    const uint32_t t = p.drop_t[k], oc = p.drop_old[k];
    const OffT ob = p.off[u], oe = p.off[u + 1];
    for (OffT base = ob; base < oe; base += 32) {
      const OffT i = base + lane;
      bool want = false;
      uint32_t v = 0;
      if (i < oe) {
        v = p.adj[i];
        const uint32_t x = p.est[v];
        want = ext ? (t < x && oc >= x) : (x > t);
      }
      acc.fires += want;
      warp_push(p, nxt, v, want);
    }
  }
}

template <typename OffT, typename EstT>
__global__ void __launch_bounds__(SOLVE_THREADS, 1) rounds_kernel(P<OffT, EstT> p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem[];
  EstT* s_cache = reinterpret_cast<EstT*>(smem);
  const size_t cache_bytes = ((size_t)p.cache_n * sizeof(EstT) + 15) & ~(size_t)15;
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(smem + cache_bytes);
  __shared__ uint32_t s_red[33];
  __shared__ uint32_t s_item;
  __shared__ unsigned long long s_acc[4];
  const uint32_t tid = threadIdx.x;
  const uint32_t gtid = blockIdx.x * blockDim.x + tid;
  const uint32_t gsize = gridDim.x * blockDim.x;

  for (uint32_t r = p.r_begin; r < p.r_end; ++r) {
    const uint32_t cur = r & 1, nxt = cur ^ 1;
    const uint32_t sr = r < STAT_SLOTS - 1 ? r : STAT_SLOTS - 1;
    if (p.cache_n) {
      // vectorised cache fill: cache_n is a multiple of 8 (16 bytes)
      const uint4* src = reinterpret_cast<const uint4*>(p.est);
      uint4* dst = reinterpret_cast<uint4*>(s_cache);
      const uint32_t nvec = (uint32_t)((size_t)p.cache_n * sizeof(EstT) / 16);
      for (uint32_t i = tid; i < nvec; i += SOLVE_THREADS) dst[i] = src[i];
    }
    if (tid < 4) s_acc[tid] = 0;
    if (blockIdx.x == 0 && tid == 32) {
      unsigned long long fr = 0;
      for (int c = 0; c < NCLS; ++c) fr += p.qcnt[cur * NCLS + c];
      p.stats[sr].frontier = fr;
    }
    __syncthreads();
    Acc acc{0, 0, 0, 0};
    eval_block_items(p, r, s_cache, s_hist, s_red, &s_item, acc);
    eval_warp_items(p, r, s_cache, acc);
    eval_sub_items(p, r, s_cache, acc);
    eval_thread_items(p, r, s_cache, acc);
    // flush counters: warp reduce, then one shared atomic per warp
    {
      unsigned long long v[4] = {acc.evals, acc.escan, acc.drops, acc.fires};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        unsigned long long x = v[q];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(FULL, x, d);
        if (lane_id() == 0 && x) atomicAdd(&s_acc[q], x);
      }
    }
    __syncthreads();
    if (tid == 0) {
      if (s_acc[0]) atomicAdd(&p.stats[sr].evals, s_acc[0]);
      if (s_acc[1]) atomicAdd(&p.stats[sr].escan, s_acc[1]);
      if (s_acc[2]) atomicAdd(&p.stats[sr].drops, s_acc[2]);
      if (s_acc[3]) atomicAdd(&p.stats[sr].fires, s_acc[3]);
    }
    grid.sync();
    const uint32_t nd = *reinterpret_cast<volatile uint32_t*>(&p.ctl[cur].ndrops);
    if (nd == 0) {
      if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = r + 1;
        p.status[1] = 1;
      }
      return;
    }
    // apply (fastk.cpp:153)
    for (uint32_t k = gtid; k < nd; k += gsize) p.est[p.drop_u[k]] = p.drop_t[k];
    if (blockIdx.x == 0) {
      if (tid < NCLS) {
        p.ctl[nxt].grab[tid] = 0;
        p.qcnt[cur * NCLS + tid] = 0;  // becomes round r+1's push target
      }
      if (tid == NCLS) p.ctl[nxt].ndrops = 0;
    }
    if (p.rule <= R_REF_PLAIN) {
      grid.sync();
      if (tid < 4) s_acc[tid] = 0;
      __syncthreads();
      Acc nacc{0, 0, 0, 0};
      notify_settled(p, r, nd, nacc);
      unsigned long long x = nacc.fires;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(FULL, x, d);
      if (lane_id() == 0 && x) atomicAdd(&s_acc[3], x);
      __syncthreads();
      if (tid == 0 && s_acc[3]) atomicAdd(&p.stats[sr].fires, s_acc[3]);
    }
    grid.sync();
    if (blockIdx.x == 0 && tid == 0) {
      unsigned long long act = 0;
      for (int c = 0; c < NCLS; ++c) act += p.qcnt[nxt * NCLS + c];
      p.stats[sr].active_after = act;
      p.status[0] = r + 1;
    }
  }
}

// Round-0 state: est = min(deg, H) (identical trajectory
// from round 1; the reference starts at deg, fastk.cpp:67-68), frontier =
// every non-isolated vertex in id order, bitmaps and counters cleared.
template <typename OffT, typename EstT>
__global__ void init_kernel(P<OffT, EstT> p, uint32_t h_graph, uint32_t nwords) {
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t gsize = gridDim.x * blockDim.x;
  for (uint32_t u = gtid; u < p.n_nz; u += gsize) {
    const uint32_t d = (uint32_t)(p.off[u + 1] - p.off[u]);
    p.est[u] = (EstT)(d < h_graph ? d : h_graph);
    p.queue[0][u] = u;
  }
  for (uint32_t w = gtid; w < nwords; w += gsize) {
    p.bm[0][w] = 0;
    p.bm[1][w] = 0;
  }
  for (uint32_t k = gtid; k < STAT_SLOTS * (uint32_t)(sizeof(RoundStat) / 8); k += gsize)
    reinterpret_cast<unsigned long long*>(p.stats)[k] = 0;
  if (gtid < NCLS) {
    p.qcnt[gtid] = p.cb[gtid + 1] - p.cb[gtid];
    p.qcnt[NCLS + gtid] = 0;
    p.ctl[0].grab[gtid] = 0;
    p.ctl[1].grab[gtid] = 0;
  }
  if (gtid == 0) {
    p.ctl[0].ndrops = 0;
    p.ctl[1].ndrops = 0;
    p.status[0] = 0;
    p.status[1] = 0;
    p.status[2] = 0;
  }
}

template <typename OffT, typename EstT>
P<OffT, EstT> make_params(const SolveBuffers& b) {
  P<OffT, EstT> p{};
  p.off = static_cast<const OffT*>(b.off);
  p.adj = b.adj;
  p.est = static_cast<EstT*>(b.est);
  p.n_nz = b.n_nz;
  for (int c = 0; c <= NCLS; ++c) p.cb[c] = b.cls_begin[c];
  p.queue[0] = b.queue[0];
  p.queue[1] = b.queue[1];
  p.qcnt = b.qcnt;
  p.bm[0] = b.bm[0];
  p.bm[1] = b.bm[1];
  p.drop_u = b.drop_u;
  p.drop_t = static_cast<EstT*>(b.drop_t);
  p.drop_old = static_cast<EstT*>(b.drop_old);
  p.ctl = b.ctl;
  p.stats = b.stats;
  p.status = b.status;
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
  p.tail_threshold = c.tail_threshold;
  const size_t smem = (((size_t)c.cache_n * sizeof(EstT) + 15) & ~(size_t)15) +
                      (size_t)HIST_BINS * sizeof(uint32_t);
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
cudaError_t launch_init_t(const SolveBuffers& b, uint32_t h_graph, uint32_t max_rounds,
                          cudaStream_t stream) {
  P<OffT, EstT> p = make_params<OffT, EstT>(b);
  const uint32_t nwords = (b.n_nz + 31) / 32;
  (void)max_rounds;
  init_kernel<OffT, EstT><<<148 * 4, 256, 0, stream>>>(p, h_graph, nwords);
  return cudaGetLastError();
}

}  // namespace

size_t solver_cache_bytes_max() {
  // 227 KB opt-in per CTA: keep HIST_BINS * 4 + static scratch + headroom for L1.
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
  if (est16)
    return off64 ? launch_init_t<uint64_t, uint16_t>(b, h_graph, max_rounds, stream)
                 : launch_init_t<uint32_t, uint16_t>(b, h_graph, max_rounds, stream);
  return off64 ? launch_init_t<uint64_t, uint32_t>(b, h_graph, max_rounds, stream)
               : launch_init_t<uint32_t, uint32_t>(b, h_graph, max_rounds, stream);
}

}  // namespace kcb
