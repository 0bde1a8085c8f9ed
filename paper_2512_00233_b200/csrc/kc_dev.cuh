// kc_dev.cuh — device building blocks shared by the two solvers:
// kc_solve.cu (reference activation rule, byte-flag frontier) and
// kc_count.cu (counting rule, direct queues, relevant-neighbour lists).
//
// The h-index pieces restate include/kcore/kernel.hpp:27-42
// (compute_index_over): values are capped at `cap`, counted per level, and
// the answer is the largest level t >= 1 with count(>= t) >= t.
#pragma once
#include <cstdint>
#include <cstdio>

#include "kc_internal.h"

namespace kcb {
namespace dev {

constexpr unsigned FULL = 0xffffffffu;

// KC_DEBUG_BOUNDS=1 (scripts/build_debug_bounds.sh): every queue, list,
// long-scan-queue, histogram and per-vertex index the solvers write is
// checked; a violation prints its site and traps (the launch fails with a
// CUDA error, the C-ABI returns KC_ERR_CUDA).  compute-sanitizer is closed on
// this pool, so this build stands in for its bounds checks.
#ifndef KC_DEBUG_BOUNDS
#define KC_DEBUG_BOUNDS 0
#endif
#if KC_DEBUG_BOUNDS
#define KC_BOUNDS(cond)                                                                  \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      printf("KC_BOUNDS %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, blockIdx.x, \
             threadIdx.x, #cond);                                                        \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define KC_BOUNDS(cond) \
  do {                  \
  } while (0)
#endif
constexpr uint32_t NWARPS = SOLVE_THREADS / 32;

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint32_t lanemask_lt() { return (1u << lane_id()) - 1u; }
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Estimate of v: shared-memory cache for the highest-degree ids, global
// (L1/L2) otherwise.  One generic load per gather keeps the inlined gather
// sites small for the instruction cache.
// The estimate cache's generic address, opaque to the compiler.  Left as a
// pointer the compiler knows to be shared, it rebuilds the generic address
// of the shared window (S2R SR_CgaCtaId + S2R SR_SWINHI + LEA + MOVs) at
// every gather site instead of keeping it in a register: ~9 extra
// instructions, two of them slow special-register reads, per gathered
// estimate (SASS of the notify scans).  KC_OPAQUE_CACHE=0 restores that.
#ifndef KC_OPAQUE_CACHE
#define KC_OPAQUE_CACHE 1
#endif
template <typename T>
__device__ __forceinline__ T* opaque_ptr(T* p) {
#if KC_OPAQUE_CACHE
  T* r;
  asm volatile("mov.b64 %0, %1;" : "=l"(r) : "l"(p));
  return r;
#else
  return p;
#endif
}

#ifndef KC_EST_CACHE
#define KC_EST_CACHE 1   // 0: every gather from global memory (A/B: R-MAT 22 -1.5%,
                         // R-MAT 26 +1.6%; explicit LDS/LDG pairs cost more)
#endif
template <typename EstT>
__device__ __forceinline__ uint32_t est_at(const EstT* __restrict__ s_cache, uint32_t cache_n,
                                           const EstT* snap, uint32_t v) {
#if KC_EST_CACHE
  const EstT* base = v < cache_n ? s_cache : snap;
  return (uint32_t)base[v];
#else
  (void)s_cache;
  (void)cache_n;
  __builtin_assume(__isGlobal(snap));
  return (uint32_t)snap[v];
#endif
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
// RO: the array is immutable for the kernel's lifetime (the CSR) — non-
// coherent path, no L1 allocation (L1 is left to the estimate gathers).
// Otherwise (lists rewritten inside the kernel): L2 only.
// The id streams are read once per phase: with KC_L2_STREAM_FIRST (default) they carry
// an L2 evict-first policy so they do not push the gathered estimates out of
// L2 (the estimates of R-MAT 26 alone are 134 MB): -2.4% on R-MAT 22, -2.2% on R-MAT 26.
#ifndef KC_L2_STREAM_FIRST
#define KC_L2_STREAM_FIRST 1
#endif
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

template <bool RO>
__device__ __forceinline__ uint4 ld_ids4(const uint32_t* src, uint64_t a) {  // 4 ids at src + a
  uint4 r;
#if KC_L2_STREAM_FIRST
  const uint64_t pol = l2_evict_first_policy();
  if (RO)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(src + a), "l"(pol));
  else
    asm volatile("ld.global.cg.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(src + a), "l"(pol));
#else
  if (RO)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(src + a));
  else
    asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(src + a));
#endif
  return r;
}
// Bulk L2 prefetch of a row / list by the copy engine (cp.async.bulk.prefetch,
// sm_90+): one instruction per item, no registers held while it is in flight.
// The solver's chains start with a DRAM round trip for each queued vertex's
// first ids (the CSR and the lists do not fit L2); issuing the prefetch for
// every item of a grab as soon as its metadata is known turns those into L2
// hits.  KC_L2_PREFETCH=0 disables (A/B).
#ifndef KC_L2_PREFETCH
#define KC_L2_PREFETCH 1
#endif
__device__ __forceinline__ void l2_prefetch_ids(const uint32_t* p, uint64_t n) {
#if KC_L2_PREFETCH
  const uint64_t a = reinterpret_cast<uint64_t>(p) & ~(uint64_t)15;
  const uint64_t b = (reinterpret_cast<uint64_t>(p + n) + 15) & ~(uint64_t)15;
  uint64_t bytes = b - a;
  if (bytes > (1u << 20)) bytes = 1u << 20;  // the head of a hub row is enough
  if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)bytes)
                      : "memory");
#else
  (void)p;
  (void)n;
#endif
}

__device__ __forceinline__ uint32_t u4_get(const uint4& q, int e) {
  return e == 0 ? q.x : e == 1 ? q.y : e == 2 ? q.z : q.w;
}

// ------------------------------------------------------------------------
// Block-wide helpers (blockDim == SOLVE_THREADS)
// ------------------------------------------------------------------------
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

// Tally one gathered value into the window [top - NB, top): bin i counts
// x == top-1-i, `above` counts x >= top (the capped top bin of
// compute_index_over, kernel.hpp:31-35, kept in registers).
// Values below `floor` cannot change the answer (it is known to be >= floor)
// and are skipped.
template <int NB>
__device__ __forceinline__ void tally(uint32_t x, uint32_t top, uint32_t floor, uint32_t& above,
                                      uint32_t* bins) {
  if (x >= top) ++above;
  else if ((int)x >= (int)top - NB && x >= floor) {
    KC_BOUNDS(top - 1 - x < (uint32_t)NB);
    atomicAdd(&bins[top - 1 - x], 1u);
  }
}

// Suffix scan of one window (kernel.hpp:36-41): the smallest bin i whose
// level x = top-1-i >= minlvl (>= 1) has count(>= x) = C + sum(bins[0..i])
// >= x.  Levels below the tally floor are not complete, so minlvl must be
// >= the floor.  Warp version, lane l owns bins [8l, 8l+8).  Returns the
// level and, in `cnt`, count(>= level).
__device__ __forceinline__ bool warp_resolve(const uint32_t* bins, uint32_t C, uint32_t top,
                                             uint32_t& level, uint32_t& cnt,
                                             uint32_t minlvl = 1) {
  static_assert(WARP_BINS == 256, "8 bins per lane");
  const uint32_t lane = lane_id();
  const uint4 b0 = reinterpret_cast<const uint4*>(bins)[2 * lane];
  const uint4 b1 = reinterpret_cast<const uint4*>(bins)[2 * lane + 1];
  const uint32_t b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += b[j];
  uint32_t run = C + warp_incl_scan(s) - s;
  uint32_t found = 0xffffffffu, frun = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    run += b[j];
    const int i = (int)lane * 8 + j;
    const int x = (int)top - 1 - i;
    if (found == 0xffffffffu && x >= (int)minlvl && run >= (uint32_t)x) {
      found = (uint32_t)i;
      frun = run;
    }
  }
  const uint32_t g = __reduce_min_sync(FULL, found);
  if (g == 0xffffffffu) return false;
  cnt = __shfl_sync(FULL, frun, g >> 3);
  level = top - 1 - g;
  return true;
}

// Coarse windows.  The levels [L, top) are split into bins of width w, bin i
// covering [low_i, top - i*w) with low_i = max(top - (i+1)*w, L), i = 0 at
// the top; C = count(>= top).  count(>= low_i) = C + bins[0..i] =: run_i,
// so the largest qualifying level (count(>= x) >= x) lies in the first bin
// with run_i >= low_i, and no level above it qualifies.  Warp version, lane l
// owns bins [8l, 8l+8).  Returns that bin and run_i.
__device__ __forceinline__ uint32_t bin_low(uint32_t top, uint32_t w, uint32_t L, uint32_t i) {
  const uint64_t d = (uint64_t)(i + 1) * w;
  return d >= (uint64_t)(top - L) ? L : top - (uint32_t)d;
}

__device__ __forceinline__ bool warp_resolve_w(const uint32_t* bins, uint32_t C, uint32_t top,
                                               uint32_t w, uint32_t L, uint32_t& bin,
                                               uint32_t& run_at) {
  static_assert(WARP_BINS == 256, "8 bins per lane");
  const uint32_t lane = lane_id();
  const uint4 b0 = reinterpret_cast<const uint4*>(bins)[2 * lane];
  const uint4 b1 = reinterpret_cast<const uint4*>(bins)[2 * lane + 1];
  const uint32_t b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += b[j];
  uint32_t run = C + warp_incl_scan(s) - s;
  const uint32_t nb = (top - L + w - 1) / w;  // bins in use
  uint32_t found = 0xffffffffu, frun = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    run += b[j];
    const uint32_t i = lane * 8 + j;
    if (found == 0xffffffffu && i < nb && run >= bin_low(top, w, L, i)) {
      found = i;
      frun = run;
    }
  }
  const uint32_t g = __reduce_min_sync(FULL, found);
  if (g == 0xffffffffu) return false;
  run_at = __shfl_sync(FULL, frun, g >> 3);
  bin = g;
  return true;
}

__device__ __forceinline__ void warp_zero_bins(uint32_t* bins) {
  const uint32_t lane = lane_id();
  reinterpret_cast<uint4*>(bins)[2 * lane] = make_uint4(0, 0, 0, 0);
  reinterpret_cast<uint4*>(bins)[2 * lane + 1] = make_uint4(0, 0, 0, 0);
  __syncwarp();
}

__device__ __forceinline__ uint32_t tile8_sum(uint32_t v) {
  v += __shfl_xor_sync(FULL, v, 4, 8);
  v += __shfl_xor_sync(FULL, v, 2, 8);
  v += __shfl_xor_sync(FULL, v, 1, 8);
  return v;
}

// ------------------------------------------------------------------------
// Streaming over a row with 128-bit id loads: each of NT cooperating threads
// takes 8 entries per step (two 16-byte loads, software-pipelined one step
// ahead), gathers their 8 estimates, then hands (valid mask, ids, estimates)
// to the callback.  Rows need not be 16-byte aligned: the stream starts at
// the 16-byte granule holding ob and masks positions outside [ob, oe) (id
// arrays have ADJ_PAD spare entries).  Position arithmetic is 32-bit,
// relative to that granule (a row is < 2^32 entries): one 64-bit base.
//
// `cut`: ids >= cut are masked without a gather (with degree-descending ids,
// id >= cut(x) means degree < x, so the estimate is < x too).  `stop`: the
// source is sorted ascending, so once a warp's step holds an id >= cut every
// later step of that warp does too — the warp leaves the stream.
// `ro`: the immutable CSR via the non-coherent path; else lists rewritten
// inside the kernel (L2 only).
// ------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_ids4_rt(const uint32_t* p, bool ro) {
  return ro ? ld_ids4<true>(p, 0) : ld_ids4<false>(p, 0);
}

// KC_STREAM_K: entries per thread per step (8: two 128-bit id loads, 4: one);
// KC_STREAM_PREFETCH: the next step's ids are loaded before this step's
// gathers are consumed (8 more live registers); 2 (4-entry streams only): also
// the next step's gathers are issued before this step is consumed (measured
// 4% slower: profiles/r02/stream_pf2_ab.txt).  The per-phase kernels
// (kc_count_split.cu) trade both for resident warps.  The callback always
// sees 8 slots; with K = 4 the upper four are never valid (compile-time
// zero bits of `ok`, so their code folds away).
#ifndef KC_STREAM_K
#define KC_STREAM_K 8
#endif
#ifndef KC_STREAM_PREFETCH
#define KC_STREAM_PREFETCH 1
#endif
template <int NT, typename EstT, typename F>
__device__ __forceinline__ void stream_row_rt(const uint32_t* src, bool ro, const EstT* snap,
                                              uint32_t me, uint64_t ob, uint64_t oe,
                                              const EstT* s_cache, uint32_t cache_n, F&& f,
                                              uint32_t cut = 0xffffffffu, bool stop = false) {
  constexpr int K = KC_STREAM_K;
  constexpr bool PF = KC_STREAM_PREFETCH != 0;
  static_assert(K == 4 || K == 8, "one or two 128-bit id loads per step");
  constexpr uint32_t STEP = (uint32_t)NT * K;
  const uint32_t* base = src + (ob & ~(uint64_t)3) + 4 * me;  // this thread's first granule
  const uint32_t head = (uint32_t)(ob & 3);   // masked entries before the row
  const uint32_t len = (uint32_t)(oe - ob);
  const uint32_t end = head + len;            // relative end
  const uint32_t l0 = 4 * me, l1 = 4 * me + 4 * NT;
#if KC_STREAM_PREFETCH == 2
  if constexpr (K == 4) {
    // Two-deep pipeline: the gathers of step a + 1 are issued before step a is
    // consumed (and the ids of step a + 2 are loaded), so a step waits for
    // max(gather, the consumer's own round trips) instead of their sum.
    auto gather4 = [&](const uint4& q, uint32_t a, uint32_t (&xx)[4], uint32_t& okk, bool& pst) {
      okk = 0;
      pst = false;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t id = u4_get(q, k);
        const bool in = a + l0 + k - head < len;
        const bool v = in && id < cut;
        pst |= in && !v;
        okk |= (uint32_t)v << k;
        xx[k] = v ? est_at(s_cache, cache_n, snap, id) : 0u;
      }
    };
    uint4 qa = make_uint4(0, 0, 0, 0), qb = qa;
    if (l0 < end) qa = ld_ids4_rt(base, ro);
    if (STEP + l0 < end) qb = ld_ids4_rt(base + STEP, ro);
    uint32_t xa[4], oka;
    bool pasta;
    gather4(qa, 0, xa, oka, pasta);
    for (uint32_t a = 0; a < end; a += STEP) {
      const uint32_t nb = a + STEP;
      uint32_t xb[4] = {0, 0, 0, 0}, okb = 0;
      bool pastb = false;
      if (nb < end) gather4(qb, nb, xb, okb, pastb);
      uint4 qc = make_uint4(0, 0, 0, 0);
      if (nb + STEP + l0 < end) qc = ld_ids4_rt(base + nb + STEP, ro);
      uint32_t ids[8], x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        ids[k] = k < 4 ? u4_get(qa, k & 3) : 0u;
        x[k] = k < 4 ? xa[k & 3] : 0u;
      }
      f(oka, ids, x);
      if (stop && __any_sync(FULL, pasta)) break;
      qa = qb;
      qb = qc;
#pragma unroll
      for (int k = 0; k < 4; ++k) xa[k] = xb[k];
      oka = okb;
      pasta = pastb;
    }
    return;
  }
#endif
  uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0;
  if (PF) {
    if (l0 < end) q0 = ld_ids4_rt(base, ro);
    if (K == 8 && l1 < end) q1 = ld_ids4_rt(base + 4 * NT, ro);
  }
  for (uint32_t a = 0; a < end; a += STEP) {
    uint4 n0 = make_uint4(0, 0, 0, 0), n1 = n0;
    if (PF) {
      const uint32_t nb = a + STEP;
      if (nb + l0 < end) n0 = ld_ids4_rt(base + nb, ro);
      if (K == 8 && nb + l1 < end) n1 = ld_ids4_rt(base + nb + 4 * NT, ro);
    } else {
      q0 = q1 = make_uint4(0, 0, 0, 0);
      if (a + l0 < end) q0 = ld_ids4_rt(base + a, ro);
      if (K == 8 && a + l1 < end) q1 = ld_ids4_rt(base + a + 4 * NT, ro);
    }
    uint32_t ids[8], x[8];
    uint32_t ok = 0;
    bool past = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= K) {
        ids[k] = 0;
        x[k] = 0;
        continue;
      }
      const uint32_t pos = a + (k < 4 ? l0 : l1) + (k & 3);
      ids[k] = u4_get(k < 4 ? q0 : q1, k & 3);
      const bool in = pos - head < len;  // head <= pos < end
      const bool v = in && ids[k] < cut;
      past |= in && !v;
      ok |= (uint32_t)v << k;
      x[k] = v ? est_at(s_cache, cache_n, snap, ids[k]) : 0u;
    }
    f(ok, ids, x);
    if (stop && __any_sync(FULL, past)) break;
    if (PF) {
      q0 = n0;
      q1 = n1;
    }
  }
}

// The immutable CSR (RO) or a list, fixed at compile time.
template <int NT, bool RO, typename EstT, typename F>
__device__ __forceinline__ void stream_row(const uint32_t* src, const EstT* snap, uint32_t me,
                                           uint64_t ob, uint64_t oe, const EstT* s_cache,
                                           uint32_t cache_n, F&& f, uint32_t cut = 0xffffffffu,
                                           bool stop = false) {
  stream_row_rt<NT>(src, RO, snap, me, ob, oe, s_cache, cache_n, static_cast<F&&>(f), cut, stop);
}

// Round 0 on a degree-sorted row (`dcut`: the degree cut table, kc_count.cu
// DegCut): the snapshot is E = min(deg, H), non-increasing along the row, so d_i >= i (1-based positions) holds
// exactly on a prefix and the capped h-index is t = #{i <= cap : row[i-1] <
// cut(i)}; count(E >= t) = #{j : row[j] < cut(t)}, a prefix of length >= t.
// Both read the row and the contiguous cut table only — no gathers — and
// stop at the first position that fails.  Returns (t, count(>= t)).
__device__ __forceinline__ uint2 r0_sorted_warp(const uint32_t* adj, const uint32_t* dcut,
                                                uint64_t ob, uint32_t deg, uint32_t cap,
                                                uint32_t& scanned) {
  const uint32_t lane = lane_id();
  const uint32_t m = cap < deg ? cap : deg;
  uint32_t h = 0, i0 = 0;
  for (; i0 < m; i0 += 256) {
    uint32_t id[8], ct[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t i = i0 + 32 * k + lane;  // 0-based position
      id[k] = i < m ? __ldg(adj + ob + i) : 0xffffffffu;
      ct[k] = i < m ? __ldg(dcut + i + 1) : 0u;
    }
    bool miss = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool in = i0 + 32 * k + lane < m;
      h += in && id[k] < ct[k];
      miss |= in && !(id[k] < ct[k]);
    }
    if (__any_sync(FULL, miss)) break;
  }
  const uint32_t t = __reduce_add_sync(FULL, h);
  const uint32_t ctt = __ldg(dcut + t);
  uint32_t c = 0, j0 = t;
  for (; j0 < deg; j0 += 256) {
    uint32_t id[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t j = j0 + 32 * k + lane;
      id[k] = j < deg ? __ldg(adj + ob + j) : 0xffffffffu;
    }
    bool miss = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      c += id[k] < ctt;
      miss |= j0 + 32 * k + lane < deg && !(id[k] < ctt);
    }
    if (__any_sync(FULL, miss)) break;
  }
  scanned = (i0 < m ? i0 + 256 : m) + (j0 < deg ? j0 + 256 - t : deg - t);
  return make_uint2(t, t + __reduce_add_sync(FULL, c));
}

// The same rule by one lane: both quantities are monotone along a sorted row
// (row ids ascend, the cut table descends), so t is the last position i <= cap
// with row[i-1] < cut(i) and count(E >= t) the first position j >= t with
// row[j] >= cut(t) — two binary searches, ~2 log2(deg) probes of one sector
// each instead of streaming the row (count(E >= t) is nearly the whole row for
// most vertices).  A warp evaluates 32 vertices at once.  `probes`: entries
// read.
__device__ __forceinline__ uint2 r0_sorted_lane(const uint32_t* adj, const uint32_t* dcut,
                                                uint64_t ob, uint32_t deg, uint32_t cap,
                                                uint32_t& probes) {
  const uint32_t* row = adj + ob;
  uint32_t lo = 0, hi = cap < deg ? cap : deg, np = 0;
  while (lo < hi) {  // largest i with row[i-1] < cut(i) (holds on a prefix; i = 0: vacuous)
    const uint32_t mid = (lo + hi + 1) >> 1;
    const uint32_t id = __ldg(row + mid - 1), ct = __ldg(dcut + mid);
    ++np;
    if (id < ct) lo = mid; else hi = mid - 1;
  }
  const uint32_t t = lo;
  const uint32_t ctt = __ldg(dcut + t);
  hi = deg;
  while (lo < hi) {  // first j >= t with row[j] >= cut(t)
    const uint32_t mid = (lo + hi) >> 1;
    ++np;
    if (__ldg(row + mid) < ctt) lo = mid + 1; else hi = mid;
  }
  probes = np;
  return make_uint2(t, lo);
}

template <typename EstT>
__device__ __forceinline__ void fill_cache(EstT* s_cache, const EstT* src, uint32_t cache_n) {
  // cache_n * sizeof(EstT) is a multiple of 16 bytes; 8 loads in flight per
  // thread so the fill costs ~2 memory round trips, not nvec / SOLVE_THREADS
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(s_cache);
  const uint32_t nvec = (uint32_t)((size_t)cache_n * sizeof(EstT) / 16);
  for (uint32_t i0 = threadIdx.x; i0 < nvec; i0 += 8 * SOLVE_THREADS) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t i = i0 + k * SOLVE_THREADS;
      if (i < nvec) v[k] = s[i];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t i = i0 + k * SOLVE_THREADS;
      if (i < nvec) d[i] = v[k];
    }
  }
}

// The same fill as one TMA bulk copy (cp.async.bulk global -> shared,
// completion on an mbarrier; UBLKCP in SASS): one thread issues it, every
// thread waits on the barrier's phase.  No registers, no LSU instructions and
// no shared-memory stores per thread.  `smem_cache` is the 16-byte aligned
// start of the cache, cache_n * sizeof(EstT) a multiple of 16 bytes.  The
// previous readers of the cache are behind a CTA or grid barrier (every call
// site); the proxy fence orders their generic-proxy reads before the async
// proxy's writes.
#ifndef KC_TMA_FILL
#define KC_TMA_FILL 1
#endif
__device__ __forceinline__ void mbar_init(unsigned long long* mbar) {  // one thread, before a CTA barrier
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(mbar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
template <typename EstT>
__device__ __forceinline__ void fill_cache_bulk(void* smem_cache, EstT* s_cache, const EstT* src,
                                                uint32_t cache_n, unsigned long long* mbar,
                                                uint32_t& phase) {
#if KC_TMA_FILL
  (void)s_cache;
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)((size_t)cache_n * sizeof(EstT));
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem_cache);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(mb)
        : "memory");
  }
  uint32_t done;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(mb), "r"(phase)
        : "memory");
  } while (!done);
  phase ^= 1u;
#else
  (void)smem_cache;
  (void)mbar;
  (void)phase;
  fill_cache(s_cache, src, cache_n);
#endif
}

}  // namespace dev
}  // namespace kcb
