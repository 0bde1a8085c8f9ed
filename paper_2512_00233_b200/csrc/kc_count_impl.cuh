// kc_count_impl.cuh — the counting-rule FastK solver (KC_RULE_COUNTING, the
// default) on sm_100a.  Included by two translation units, each with its own
// register budget and CTA shape (everything below lives in an anonymous
// namespace, so each unit gets its own copies):
//   kc_count.cu        KC_TU_SPLIT=0  the persistent cooperative kernel (every
//                                     round in one launch, grid barriers)
//   kc_count_split.cu  KC_TU_SPLIT=1  one kernel per phase (EVALUATE, NOTIFY)
//                                     for the large rounds, phase functions
//                                     inlined, more resident warps per SM
//
// Reference path (paths under /root/reference/proj):
//   fastk_run            src/fastk.cpp:57-187  — rounds of process | apply | notify
//   compute_index_over   include/kcore/kernel.hpp:27-42 — capped h-index
//   should_notify        include/kcore/fastk.hpp:25-27  — extended activation rule
//
// Same Jacobi trajectory as the reference (and as kc_solve.cu), organised
// around three facts of the counting rule:
//
//  1. Support counters.  cnt[v] = #{w in N(v) : est_w >= est_v}.  A drop
//     u: cap -> t passes should_notify(t, cap, N[w]) exactly when it removes
//     u from w's count; the one decrement that takes cnt[w] below N[w] makes
//     w unstable.  So a vertex is evaluated iff it drops, and the decrement
//     that activates it is unique: it is appended to the next round's queue
//     directly (per-warp shared-memory buffers, one global atomic per 32
//     activations) — no frontier flags, no compaction pass.
//
//  2. The answer is bracketed.  An active u has lo = cnt[u] = count(>= cap)
//     < cap, and its new level t satisfies lo <= t < cap.  Only neighbour
//     values in [lo, cap) are binned.
//
//  3. Relevant-neighbour lists.  After its first drop, u keeps in `radj` the
//     neighbours w with est_w >= L_u (L_u = ceil(t/2) at build time).
//     Estimates only fall, so every neighbour left out stays below L_u
//     forever.  While t >= L_u, both the h-index (levels >= L_u) and the
//     notify test (N[w] > t) are decided by the list alone; a hub with 160 K
//     neighbours and t ~ 900 scans a few thousand entries per round instead
//     of its whole row.  If the answer falls below L_u (lo < L_u and t < L_u)
//     the evaluation scans the CSR row, and the notify pass that follows
//     rebuilds the list.  E_scan is still reported as the sum of degrees
//     (the algorithmic convention of SURVEY §8(d)).
//
// Round r:
//   EVALUATE  every queued u (round 0: every vertex) computes t and
//             c = count(E >= t); writes N[u] = t, cnt[u] = c.
//   --- grid.sync (round 0 without a drop ends here, fastk.cpp:109-110) ---
//   NOTIFY    every dropper streams its list (or row) against the settled
//             values N, decrements cnt[w] where should_notify holds,
//             enqueues the w whose counter crossed below N[w], applies
//             E[u] = t (fastk.cpp:153).
//   --- grid.sync ---
// An empty queue at a round start is the quiescent round: converged.
#include <cooperative_groups.h>
#include <cstdint>
#include <mutex>

#include "kc_dev.cuh"
#include "kc_internal.h"

namespace cg = cooperative_groups;

#ifndef KC_TU_SPLIT
#define KC_TU_SPLIT 0
#endif
// Phase functions: out of line in the persistent kernel (one body per phase,
// small kernel text), inlined into the per-phase kernels.
#ifndef KC_PHASE_INLINE
#define KC_PHASE_INLINE 0
#endif
#if KC_PHASE_INLINE
#define KC_PHASE_FN __forceinline__
#else
#define KC_PHASE_FN __noinline__
#endif

namespace kcb {
namespace {
using namespace dev;

#ifndef KC_GMAX_BIG
#define KC_GMAX_BIG 8
#endif
#ifndef KC_GMAX_WARP
#define KC_GMAX_WARP 16
#endif
#ifndef KC_CACHE_MIN_ACTIVE
#define KC_CACHE_MIN_ACTIVE 4096
#endif
#ifndef KC_GMAX_SMALL
#define KC_GMAX_SMALL 32
#endif
constexpr uint32_t GMAX_BIG = KC_GMAX_BIG, GMAX_WARP = KC_GMAX_WARP, GMAX_SMALL = KC_GMAX_SMALL;  // items per grab (max)
static_assert(GMAX_BIG <= 32 && GMAX_WARP <= 32 && GMAX_SMALL <= 32,
              "a grab's items are held one per lane");
constexpr uint32_t CACHE_MIN_ACTIVE = KC_CACHE_MIN_ACTIVE;  // smaller rounds skip the shared-memory cache
#ifndef KC_LIST_MIN_DEG
#define KC_LIST_MIN_DEG 64
#endif
constexpr uint32_t LIST_MIN_DEG = KC_LIST_MIN_DEG;  // rows longer than this keep a list
#ifndef KC_WARP_MAX_LEN
#define KC_WARP_MAX_LEN DEG_BIG_MAX
#endif
constexpr uint32_t WARP_MAX_LEN = KC_WARP_MAX_LEN;  // longest scan a single warp takes
// ... in a small round (fewer than WML_SMALL_ACTIVE active vertices) only
// WML_SMALL: most warps are idle there and a hub's 8 K-entry list on one warp
// is the round's critical path (64 dependent steps); CTA-wide it is 3.
// Chung-Lu's rounds 10-72 (0.5-2 K hubs, nothing else): 13.0 -> 11.9 ms.
#ifndef KC_WML_SMALL
#define KC_WML_SMALL 2048
#endif
#ifndef KC_WML_SMALL_ACTIVE
#define KC_WML_SMALL_ACTIVE 8192
#endif
constexpr uint32_t WML_SMALL = KC_WML_SMALL, WML_SMALL_ACTIVE = KC_WML_SMALL_ACTIVE;
constexpr int HREG = HIST_BINS > (int)NWARPS * WARP_BINS ? HIST_BINS : (int)NWARPS * WARP_BINS;
#ifndef KC_WQ
#define KC_WQ 64
#endif
constexpr int WQ = KC_WQ;          // per-warp, per-class enqueue buffer (flushed at WQ - 32)
#ifndef KC_FLAT_EVAL
#define KC_FLAT_EVAL 1             // rounds >= 1: batched flat streams for BIG / WARP evaluate
#endif
#ifndef KC_FLAT_NOTIFY
#define KC_FLAT_NOTIFY 0           // ... and notify (slower: per-entry segment lookups)
#endif
#ifndef KC_SPEC
#define KC_SPEC 1                  // notify scans evaluate droppers for the next round
#endif
#ifndef KC_SPEC_CTA
#define KC_SPEC_CTA HIST_BINS      // next-round window of the CTA-wide (hub) notify scans
#endif
#ifndef KC_SPEC_BINS
#define KC_SPEC_BINS 256           // spec window width (levels below t), <= WARP_BINS
#endif
#ifndef KC_R0_PASSA
#define KC_R0_PASSA 0              // 1: round 0 first counts values >= cap (one pass when
#endif                             //    nothing drops); 0: straight to the window
#ifndef KC_LIST_COMPACT
#define KC_LIST_COMPACT 0          // 1: notify filters lists in place (warp scans)
#endif
#ifndef KC_FLAT_META
#define KC_FLAT_META 1             // per-vertex metadata loaded in one level (see eval_item)
#endif
#ifndef KC_R0_LISTS
#define KC_R0_LISTS 0              // 1: round-0 droppers build their lists in round 0's notify
#endif
#ifndef KC_DCUT
#define KC_DCUT 1                  // degree cut table on sorted layouts (DegCut)
#endif
#ifndef KC_CUT_EVAL
#define KC_CUT_EVAL 1              // windowed evaluations skip / stop at ids below their floor
#endif
#ifndef KC_CUT_NOTIFY
#define KC_CUT_NOTIFY 1            // notify row scans likewise, in their own function
#endif
#ifndef KC_ROW_FLOOR_BUILD
#define KC_ROW_FLOOR_BUILD 1       // a row scan that builds a list resolves its next-round
                                   // window only down to the list threshold L (a level below L
                                   // needs the row again anyway), so the scan needs no value
                                   // below L and on sorted rows stops at the degree cut dcut[L]
#endif
#ifndef KC_CUT_LISTS
#define KC_CUT_LISTS 1             // ... also on (unsorted) lists: mask only
#endif
#ifndef KC_R0_SORTED
#define KC_R0_SORTED 1             // round 0 on sorted rows without gathers (r0_sorted_warp)
#endif
#ifndef KC_R0_LANE
#define KC_R0_LANE 1               // ... BIG / WARP rows by a lane each, binary searches (r0_sorted_lane)
#endif
#ifndef KC_LIST_SHIFT
#define KC_LIST_SHIFT 1            // list threshold L = t - (t >> KC_LIST_SHIFT)
#endif

// Degree cut table.  New ids are assigned in order of non-increasing degree,
// so cut(x) = #{ids of degree >= x} splits the ids: id < cut(x) iff degree
// >= x.  Estimates never exceed degrees, hence id >= cut(x) implies estimate
// < x — those entries can be skipped without a gather, and in a row sorted
// ascending (sorted layouts) they form its suffix.
struct DegCut {
  const uint32_t* t;  // [n]; nullptr: no table
  uint32_t n;         // max degree + 2
  bool sorted;        // rows sorted ascending: prefix rules and early exits apply
  __device__ __forceinline__ uint32_t at(uint32_t x) const {
    return !t ? 0xffffffffu : x < n ? t[x] : 0u;
  }
};

template <typename OffT, typename EstT>
struct CP {
  const OffT* off;
  const uint32_t* adj;  // CSR rows (immutable)
  uint32_t* radj;       // relevant-neighbour lists, row u at off[u]
  uint32_t* rlen;       // list lengths
  EstT* rthr;           // list thresholds L_u (0: no list, use the CSR row)
  uint32_t* spec_r;     // speculative next-round evaluation: round it is valid for,
  uint32_t* spec_t;     //   its level and
  uint32_t* spec_c;     //   count(>= level) (computed by the notify scan, see NOTIFY)
  uint8_t* pflag;       // PULL: round-1 droppers (compacted into round 1's queue)
  DegCut dc;
  uint32_t n_nz;
  uint32_t cb[NCLS + 1];
  EstT* E;  // snapshot
  EstT* N;  // settled
  uint32_t* cnt;
  uint32_t* queue[2];  // queue[r & 1]: round r's active ids, class c at offset cb[c]
  uint32_t* lq[2];     // long-scan queues (evaluate, notify); empty slots 0xffffffff
  Ctl* ctl;            // [2] per round parity: qcnt (queue sizes), grab / grab2 cursors
  uint32_t* anydrop;   // [0]: some estimate dropped in round 0
  RoundStat* stats;
  uint32_t* status;
  unsigned long long* prof;
  uint32_t r_begin, r_end, cache_n, clamp_drop;
  uint32_t prof_ctas;   // CTAs per profile row (the persistent kernel's grid)
  bool pull;            // round 0 ends with the PULL phase (see the kernel)
};
constexpr uint32_t R_RESUME = 0xffffffffu;  // r_begin: carry on at round status[0]
#ifndef KC_SPLIT_CTAS
#define KC_SPLIT_CTAS 1            // per-phase kernels: CTAs per SM (kc_count_split.cu)
#endif

// The solver's parameters in constant memory, for the out-of-line phase
// functions: a `const CP&` argument is a generic pointer there, and every
// field it reads (the counter array of each atomic, the estimate arrays of
// each stream) was a generic load with a uniform-descriptor move (LD.E +
// R2UR pairs in SASS).  From the constant bank they are LDC / ULDC.  Written
// by launch_t right before the launch, ordered after the previous solve's
// kernel on any stream (c_done), so concurrent solves never see each
// other's copy.
template <typename OffT, typename EstT>
__constant__ CP<OffT, EstT> c_params;

template <typename EstT>
struct View {
  const EstT* snap;      // gathered estimates: E (evaluate) or N (notify)
  const uint32_t* q;     // this round's queue; nullptr in round 0 (ids implicit)
  const uint32_t* qcnt;  // this round's class sizes
  uint32_t* grab;        // cursors of the current phase
  uint32_t* qn;          // next round's class sizes
  uint32_t* qnext;       // next round's queue
  uint32_t cache_n;      // ids cached in shared memory this phase (0: none)
  bool r0;
  bool pull;             // the PULL phase: every vertex evaluated against N
  uint32_t round;
  uint32_t wml;          // longest hub scan a single warp takes this round (see WML_SMALL)
};

struct Acc {  // per-thread counters of one round (one phase in the per-phase kernels), flushed
              // into 64-bit sums per round; 32 bits each: a thread's own share of a round's
              // entries (six registers less than 64-bit counters, live through the whole kernel)
  uint32_t evals, escan, drops, fires, nscan, ascan;
  bool any_drop;
};

struct Acc32 {  // the same, per phase call, in registers (32-bit: one phase's share)
  uint32_t evals, escan, drops, fires, nscan, ascan;
  bool any_drop;
};

__device__ __forceinline__ void merge_acc(Acc& to, const Acc32& a) {
  to.evals += a.evals;
  to.escan += a.escan;
  to.drops += a.drops;
  to.fires += a.fires;
  to.nscan += a.nscan;
  to.ascan += a.ascan;
  to.any_drop |= a.any_drop;
}

struct Shared {  // per-CTA bookkeeping (static shared memory)
  uint32_t red[33];
  uint32_t item;
  uint32_t drop;
  uint32_t ticket;            // long-scan queue ticket held across the phase
  uint32_t cursor;            // CTA list-build cursor
  uint32_t out[2];
  unsigned long long acc[6];
};

template <typename OffT, typename EstT>
__device__ __forceinline__ int cls_of(const CP<OffT, EstT>& p, uint32_t id) {
  return (int)(id >= p.cb[1]) + (int)(id >= p.cb[2]) + (int)(id >= p.cb[3]) +
         (int)(id >= p.cb[4]);
}

// Grab size for class c this round: up to gmax items per atomic, fewer when
// the queue is short so that every warp gets work.
__device__ __forceinline__ uint32_t grab_size(uint32_t cnt, uint32_t gmax) {
  const uint32_t per = cnt / (gridDim.x * NWARPS * 2u);
  return per < 1u ? 1u : per > gmax ? gmax : per;
}

// The warp's next slice [base, base + G) of a class queue (>= cnt: drained).
// KC_STATIC_FIRST: the first slice is assigned statically — warp w takes
// slice w, no atomic and no round trip (a small round's whole critical path
// is a few dependent round trips) — and the atomic cursor hands out the rest,
// counting past the static range.
#ifndef KC_STATIC_FIRST
#define KC_STATIC_FIRST 1
#endif
#ifndef KC_STATIC_MAXQ
#define KC_STATIC_MAXQ 16          // static first slice only for queues <= this many slices per warp
#endif
__device__ __forceinline__ uint32_t next_slice(uint32_t* cursor, uint32_t cnt, uint32_t G,
                                               bool& first) {
  uint32_t stat = 0;
  // (big queues: the dynamic grabs balance better, and one round trip per
  // phase is noise there)
  if (KC_STATIC_FIRST && cnt <= gridDim.x * NWARPS * G * KC_STATIC_MAXQ) {
    const uint32_t nw = gridDim.x * NWARPS;
    if (first) {
      first = false;
      const uint32_t b = (blockIdx.x * NWARPS + warp_id()) * G;
      return b < cnt ? b : cnt;
    }
    stat = nw * G;
    if (stat >= cnt) return cnt;  // the static slices covered the queue
  }
  uint32_t base = 0;
  if (lane_id() == 0)  // plain read first: no atomic once the queue is drained
    base = *reinterpret_cast<volatile uint32_t*>(cursor) + stat >= cnt ? cnt
                                                                       : stat + atomicAdd(cursor, G);
  return __shfl_sync(FULL, base, 0);
}

// Warp-level queue walk: `proc(u, n)` gets the warp's slice, lane i holding
// item i (i < n).
template <typename OffT, typename EstT, typename F>
__device__ __forceinline__ void for_class(const CP<OffT, EstT>& p, const View<EstT>& v, int c,
                                          uint32_t gmax, F&& proc) {
  const uint32_t cnt = v.qcnt[c];
  if (cnt == 0) return;
  const uint32_t G = grab_size(cnt, gmax);
  uint32_t* cursor = &v.grab[c];
  const uint32_t lane = lane_id();
  bool first = true;
  for (;;) {
    const uint32_t base = next_slice(cursor, cnt, G, first);
    if (base >= cnt) break;
    const uint32_t n = cnt - base < G ? cnt - base : G;
    uint32_t u = 0;
    if (lane < n) u = v.q ? v.q[p.cb[c] + base + lane] : p.cb[c] + base + lane;
    proc(u, n);
  }
}

// ------------------------------------------------------------------------
// Enqueue (notify phase, warp-converged): lanes' activations `act` (bit k:
// ids[k]) go to the warp's shared buffer of their class; a buffer holding
// >= 32 ids is flushed with one global atomicAdd.
// ------------------------------------------------------------------------
struct Enq {            // the warp's view of the next round's queue
  uint32_t* qn;         // next round's class sizes
  uint32_t* qnext;      // next round's queue
  uint32_t* wbuf;       // this warp's buffers [NCLS][WQ] (shared memory)
  uint32_t* wn;         // this warp's buffer fill levels [NCLS] (shared memory)
};

template <typename OffT, typename EstT>
__device__ __noinline__ void wq_flush(const CP<OffT, EstT>& p_arg, const Enq& q, int c) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  const uint32_t n = q.wn[c];
  if (n == 0) return;
  uint32_t base = 0;
  if (lane_id() == 0) base = atomicAdd(&q.qn[c], n);
  base = __shfl_sync(FULL, base, 0);
  KC_BOUNDS(p.cb[c] + base + n <= p.cb[c + 1]);  // a class never holds more than its ids
  KC_BOUNDS(n <= (uint32_t)WQ);
  for (uint32_t i = lane_id(); i < n; i += 32) q.qnext[p.cb[c] + base + i] = q.wbuf[c * WQ + i];
  __syncwarp();
  if (lane_id() == 0) q.wn[c] = 0;
  __syncwarp();
}

// End of the notify phase: every class buffer of the warp flushed with the
// atomics of all classes in flight together (lane c reserves class c), one
// round trip instead of one per non-empty class.
template <typename OffT, typename EstT>
__device__ __noinline__ void wq_flush_all(const CP<OffT, EstT>& p_arg, const Enq& q) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  const uint32_t lane = lane_id();
  uint32_t n = lane < (uint32_t)NCLS ? q.wn[lane] : 0u;
  uint32_t base = 0;
  if (n) base = atomicAdd(&q.qn[lane], n);
#pragma unroll 1
  for (int c = 0; c < NCLS; ++c) {
    const uint32_t nc = __shfl_sync(FULL, n, c);
    if (!nc) continue;
    const uint32_t bc = __shfl_sync(FULL, base, c);
    KC_BOUNDS(nc <= (uint32_t)WQ && p.cb[c] + bc + nc <= p.cb[c + 1]);
    for (uint32_t i = lane; i < nc; i += 32) q.qnext[p.cb[c] + bc + i] = q.wbuf[c * WQ + i];
  }
  __syncwarp();
  if (lane < (uint32_t)NCLS) q.wn[lane] = 0;
  __syncwarp();
}

// One activation per lane at most (a: this lane activates `id`).
template <typename OffT, typename EstT>
__device__ __noinline__ void wq_push(const CP<OffT, EstT>& p_arg, const Enq& q, bool a, uint32_t id) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  const int c = a ? cls_of(p, id) : NCLS;
#pragma unroll 1
  for (int cc = 0; cc < NCLS; ++cc) {
    const uint32_t m = __ballot_sync(FULL, c == cc);
    if (!m) continue;
    const uint32_t n0 = q.wn[cc];
    KC_BOUNDS(n0 + __popc(m) <= (uint32_t)WQ);
    KC_BOUNDS(c != cc || id < p.n_nz);
    if (c == cc) q.wbuf[cc * WQ + n0 + __popc(m & lanemask_lt())] = id;
    __syncwarp();
    if (lane_id() == 0) q.wn[cc] = n0 + __popc(m);
    __syncwarp();
    if (n0 + __popc(m) >= (uint32_t)(WQ - 32)) wq_flush(p, q, cc);
  }
}

// What a dropper u (cap -> t) does to 8 neighbours ids[k] with settled levels
// x[k] (valid where bit k of ok): decrement cnt[w] where should_notify(t,
// cap, N[w]) holds (fastk.hpp:25-27); the decrement that takes cnt[w] below
// N[w] activates w.  All atomics are issued before any result is consumed.
// Warp-converged.
template <typename OffT, typename EstT>
__device__ __forceinline__ void notify8(const CP<OffT, EstT>& p, const Enq& q, uint32_t ok,
                                        const uint32_t (&ids)[8], const uint32_t (&x)[8],
                                        uint32_t t, uint32_t cap, uint32_t& fires) {
  uint32_t fire = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) fire |= (uint32_t)((ok >> k & 1) && t < x[k] && x[k] <= cap) << k;
  uint32_t act = 0;
  if (fire) {
    fires += __popc(fire);
    uint32_t old[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) old[k] = (fire >> k & 1) ? atomicSub(&p.cnt[ids[k]], 1u) : 0u;
#pragma unroll
    for (int k = 0; k < 8; ++k) act |= (uint32_t)((fire >> k & 1) && old[k] == x[k]) << k;
  }
  if (__any_sync(FULL, act)) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (__any_sync(FULL, act >> k & 1)) wq_push(p, q, (act >> k & 1) != 0, ids[k]);
  }
}

// ------------------------------------------------------------------------
// Windowed h-index over one row or list (kernel.hpp:31-41), values >= top
// counted in registers, [top - NB, top) binned in shared memory, levels
// below `lo` skipped (the answer is >= lo).  Returns (t, count(>= t)).
// ------------------------------------------------------------------------
// Windowed h-index over one row or list (kernel.hpp:31-41) for the levels
// [max(lo, 1), cap]: values >= top are counted in registers, values in
// [L, top) are binned in shared memory in coarse bins when the range is
// wider than the bin count, then the qualifying bin is refined — at most two
// passes for 16-bit estimates.  Values below lo are skipped (the answer is
// known to be >= lo, or only levels >= lo are asked for).  Returns (t,
// count(>= t)), (cap, count(>= cap)) when nothing drops, or (0, deg) when no
// level >= lo qualifies.
template <typename EstT>
__device__ __forceinline__ uint2 warp_window(const uint32_t* src, bool ro, const EstT* snap,
                                          const EstT* s_cache, uint32_t cache_n, uint32_t* bins,
                                          uint64_t ob, uint64_t oe, uint32_t cap, uint32_t lo,
                                          uint32_t deg, bool fine_first, DegCut dc) {
  uint32_t top = cap;
  const uint32_t L0 = lo > 1u ? lo : 1u;
  uint32_t L = L0;
  bool fine = fine_first;
  for (;;) {
    uint32_t range = top > L ? top - L : 0u;
    if (fine && range > (uint32_t)WARP_BINS) {  // small drops first: one exact top window
      L = top - WARP_BINS;
      range = WARP_BINS;
    }
    fine = false;
    const uint32_t w = range > (uint32_t)WARP_BINS ? (range + WARP_BINS - 1) / WARP_BINS : 1u;
    warp_zero_bins(bins);
    uint32_t above = 0;
    stream_row_rt<32>(src, ro, snap, lane_id(), ob, oe, s_cache, cache_n,
                       [&](uint32_t ok, const uint32_t(&)[8], const uint32_t(&x)[8]) {
#pragma unroll
                         for (int k = 0; k < 8; ++k) {
                           if (!(ok >> k & 1)) continue;
                           if (x[k] >= top) ++above;
                           else if (x[k] >= L) {
                             KC_BOUNDS((top - 1 - x[k]) / w < (uint32_t)WARP_BINS);
                             atomicAdd(&bins[(top - 1 - x[k]) / w], 1u);
                           }
                         }
                       }, KC_CUT_EVAL && (KC_CUT_LISTS || ro) ? dc.at(L) : 0xffffffffu, KC_CUT_EVAL && ro && dc.sorted);
    __syncwarp();
    const uint32_t C = __reduce_add_sync(FULL, above);
    if (top == cap && C >= cap) return make_uint2(cap, C);  // no drop (round 0 only)
    uint32_t b = 0, run = 0;
    const bool hit = range > 0 && warp_resolve_w(bins, C, top, w, L, b, run);
    __syncwarp();
    if (!hit) {
      if (L > L0) {  // the top window missed: search the rest
        top = L;
        L = L0;
        continue;
      }
      return make_uint2(0u, deg);
    }
    const uint32_t low = bin_low(top, w, L, b);
    if (w == 1) return make_uint2(low, run);
    // refine inside bin b: levels [low, top - b*w); level low qualifies
    top -= b * w;
    L = low;
  }
}

template <typename EstT>
__device__ __noinline__ void cta_window(const uint32_t* src, bool ro, const EstT* snap, const EstT* s_cache,
                                        uint32_t cache_n, uint32_t* s_hist, uint32_t* s_red,
                                        uint64_t ob, uint64_t oe, uint32_t cap, uint32_t lo,
                                        uint32_t deg, bool fine_first, uint32_t* out, DegCut dc) {
  const uint32_t tid = threadIdx.x;
  uint32_t top = cap;
  const uint32_t L0 = lo > 1u ? lo : 1u;
  uint32_t L = L0;
  bool fine = fine_first;
  for (;;) {
    uint32_t range = top > L ? top - L : 0u;
    if (fine && range > (uint32_t)HIST_BINS) {  // small drops first: one exact top window
      L = top - HIST_BINS;
      range = HIST_BINS;
    }
    fine = false;
    const uint32_t w = range > (uint32_t)HIST_BINS ? (range + HIST_BINS - 1) / HIST_BINS : 1u;
    for (int i = tid; i < HIST_BINS; i += SOLVE_THREADS) s_hist[i] = 0;
    __syncthreads();
    uint32_t above = 0;
    stream_row_rt<SOLVE_THREADS>(src, ro, snap, tid, ob, oe, s_cache, cache_n,
                                  [&](uint32_t ok, const uint32_t(&)[8], const uint32_t(&x)[8]) {
#pragma unroll
                                    for (int k = 0; k < 8; ++k) {
                                      if (!(ok >> k & 1)) continue;
                                      if (x[k] >= top) ++above;
                                      else if (x[k] >= L) {
                                        KC_BOUNDS((top - 1 - x[k]) / w < (uint32_t)HIST_BINS);
                                        atomicAdd(&s_hist[(top - 1 - x[k]) / w], 1u);
                                      }
                                    }
                                  }, KC_CUT_EVAL && (KC_CUT_LISTS || ro) ? dc.at(L) : 0xffffffffu, KC_CUT_EVAL && ro && dc.sorted);
    const uint32_t C = block_sum(above, s_red);
    if (top == cap && C >= cap) {  // no drop (round 0 only)
      if (tid == 0) {
        out[0] = cap;
        out[1] = C;
      }
      __syncthreads();
      return;
    }
    constexpr int PER = (HIST_BINS + SOLVE_THREADS - 1) / SOLVE_THREADS;  // bins per thread
    uint32_t h[PER];
    uint32_t sm = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      h[j] = tid * PER + j < HIST_BINS ? s_hist[tid * PER + j] : 0u;
      sm += h[j];
    }
    uint32_t run = C + block_excl_scan(sm, s_red);
    const uint32_t nb = range ? (range + w - 1) / w : 0u;
    uint32_t found = 0xffffffffu, frun = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      run += h[j];
      const uint32_t i = tid * PER + j;
      if (found == 0xffffffffu && i < nb && run >= bin_low(top, w, L, i)) {
        found = i;
        frun = run;
      }
    }
    const uint32_t g = block_min(found, s_red);
    if (g == 0xffffffffu) {
      if (L > L0) {  // the top window missed: search the rest
        top = L;
        L = L0;
        __syncthreads();
        continue;
      }
      if (tid == 0) {
        out[0] = 0;
        out[1] = deg;
      }
      __syncthreads();
      return;
    }
    const uint32_t low = bin_low(top, w, L, g);
    if (w == 1) {
      if (found == g) {
        out[0] = low;
        out[1] = frun;
      }
      __syncthreads();
      return;
    }
    top -= g * w;
    L = low;
    __syncthreads();
  }
}

// count(x >= cap) over a row (round 0's "no change" test), warp / CTA.
template <typename EstT>
__device__ __forceinline__ uint32_t warp_count_ge(const uint32_t* adj, const EstT* snap,
                                                  const EstT* s_cache, uint32_t cache_n,
                                                  uint64_t ob, uint64_t oe, uint32_t cap) {
  uint32_t c = 0;
  stream_row<32, true>(adj, snap, lane_id(), ob, oe, s_cache, cache_n,
                       [&](uint32_t ok, const uint32_t(&)[8], const uint32_t(&x)[8]) {
#pragma unroll
                         for (int k = 0; k < 8; ++k) c += (ok >> k & 1) && x[k] >= cap;
                       });
  return __reduce_add_sync(FULL, c);
}

// ------------------------------------------------------------------------
// One evaluation (vertex u, estimate cap, lower bound lo = cnt[u] in rounds
// >= 1).  Round 0 first counts values >= cap ("no change" = one pass).
// ------------------------------------------------------------------------
struct Item {
  uint32_t u, cap, lo, thr, len, deg;
  uint64_t ob;
  bool list;
  bool spec;               // evaluated in advance by last round's notify scan
  uint32_t spec_t, spec_c;
};

// A vertex with a list (thr != 0) is first evaluated on it: levels >= thr
// are decided by the list alone.  Only if no level >= max(lo, thr)
// qualifies does the CSR row get scanned.
template <bool PULL, typename OffT, typename EstT>
__device__ __forceinline__ Item eval_item(const CP<OffT, EstT>& p, const View<EstT>& v,
                                          const EstT* s_cache, uint32_t u) {
  Item it;
  it.u = u;
#if KC_FLAT_META
  // every per-vertex field in one level of independent loads (the unused
  // ones are cheap; a second dependent level per item is not)
  it.ob = p.off[u];
  const uint64_t oe = p.off[u + 1];
  it.cap = est_at(s_cache, v.cache_n, v.snap, u);
  uint32_t lo = 0, thr = 0, sr = 0, st = 0, sc = 0, rl = 0;
  if (!v.r0 && !PULL) {
    lo = p.cnt[u];
    thr = p.rthr[u];
    sr = p.spec_r[u];
    st = p.spec_t[u];
    sc = p.spec_c[u];
    rl = p.rlen[u];
  }
  it.deg = (uint32_t)(oe - it.ob);
  it.lo = lo;
  const bool big = !v.r0 && !PULL && it.deg > LIST_MIN_DEG;
  it.thr = big ? thr : 0u;
  it.list = it.thr != 0;
  it.spec = big && sr == v.round;
  it.spec_t = it.spec ? st : 0u;
  it.spec_c = it.spec ? sc : 0u;
  it.len = it.spec ? 0u : it.list ? rl : it.deg;
#else
  it.ob = p.off[u];
  it.deg = (uint32_t)(p.off[u + 1] - it.ob);
  it.cap = est_at(s_cache, v.cache_n, v.snap, u);
  it.lo = v.r0 ? 0u : p.cnt[u];
  it.thr = (v.r0 || it.deg <= LIST_MIN_DEG) ? 0u : (uint32_t)p.rthr[u];
  it.list = it.thr != 0;
  it.spec = !v.r0 && it.deg > LIST_MIN_DEG && p.spec_r[u] == v.round;
  it.spec_t = it.spec ? p.spec_t[u] : 0u;
  it.spec_c = it.spec ? p.spec_c[u] : 0u;
  it.len = it.spec ? 0u : it.list ? p.rlen[u] : it.deg;
#endif
  return it;
}

template <bool PULL, typename OffT, typename EstT, typename A>
__device__ __forceinline__ void finish_eval(const CP<OffT, EstT>& p, const View<EstT>& v,
                                            const Item& it, uint32_t t, uint32_t c,
                                            uint32_t scanned, A& acc) {
  if (PULL) {  // PULL (see the kernel): round 1's evaluation, round 0's apply
    acc.nscan += scanned;
    p.cnt[it.u] = c;
    p.E[it.u] = (EstT)it.cap;  // E <- N (fastk.cpp:153); N is read by others this phase
    if (t < it.cap) {
      p.spec_t[it.u] = t;      // N <- t by the compaction, after the barrier
      p.pflag[it.u] = 1;
    }
    return;
  }
  KC_BOUNDS(it.u < p.n_nz);
  acc.evals += 1;
  acc.escan += it.deg;
  acc.ascan += scanned;
  p.cnt[it.u] = c;
  if (t < it.cap) {
    p.N[it.u] = (EstT)t;
    acc.drops += 1;
    acc.any_drop = true;
  }
  // the answer fell below the list threshold: the list is no longer
  // sufficient for the notify test; the notify pass rebuilds it
  if (it.thr != 0 && t < it.thr) p.rthr[it.u] = 0;
}


template <bool PULL, typename OffT, typename EstT, typename A>
__device__ __forceinline__ void eval_warp(const CP<OffT, EstT>& p, const View<EstT>& v, const EstT* s_cache,
                          uint32_t* bins, const Item& it, A& acc) {
  if (it.spec) {
    if (lane_id() == 0) finish_eval<PULL>(p, v, it, it.spec_t, it.spec_c, 0u, acc);
    return;
  }
  if (KC_R0_SORTED && v.r0 && p.dc.sorted) {
    uint32_t scanned = 0;
    const uint2 tc = r0_sorted_warp(p.adj, p.dc.t, it.ob, it.deg, it.cap, scanned);
    if (lane_id() == 0) finish_eval<PULL>(p, v, it, tc.x, tc.y, scanned, acc);
    return;
  }
  const EstT* snap = v.snap;
  const uint32_t cache_n = v.cache_n;
  uint32_t lo = it.lo;
  if (KC_R0_PASSA && v.r0) {
    const uint32_t cA = warp_count_ge(p.adj, snap, s_cache, cache_n, it.ob, it.ob + it.deg, it.cap);
    if (cA >= it.cap) {
      if (lane_id() == 0) finish_eval<PULL>(p, v, it, it.cap, cA, it.deg, acc);
      return;
    }
    lo = cA;  // count(>= cA) >= count(>= cap) = cA: the answer is >= cA
  }
  // pass 0: the list (levels >= max(lo, thr)); pass 1: the CSR row
  uint2 tc = make_uint2(0, 0);
  uint32_t scanned = 0;
#pragma unroll 1
  for (int pass = it.list ? 0 : 1; pass < 2; ++pass) {
    const bool lst = pass == 0;
    const uint32_t len = lst ? it.len : it.deg;
    tc = warp_window(lst ? (const uint32_t*)p.radj : p.adj, !lst, snap, s_cache, cache_n, bins,
                     it.ob, it.ob + len, it.cap, lst && it.thr > lo ? it.thr : lo, it.deg, !v.r0, p.dc);
    scanned += len;
    if (tc.x != 0) break;  // found (a list miss falls through to the row)
  }
  if (lane_id() == 0) finish_eval<PULL>(p, v, it, tc.x, tc.y, scanned, acc);
}

template <bool PULL, typename OffT, typename EstT>
__device__ __noinline__ void eval_cta(const CP<OffT, EstT>& p_arg, const View<EstT>& v, const EstT* s_cache,
                         uint32_t* s_hist, Shared& sh, uint32_t u, Acc& acc) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  const Item it = eval_item<PULL>(p, v, s_cache, u);
  if (it.spec) {
    if (threadIdx.x == 0) finish_eval<PULL>(p, v, it, it.spec_t, it.spec_c, 0u, acc);
    __syncthreads();
    return;
  }
  const EstT* snap = v.snap;
  const uint32_t cache_n = v.cache_n;
  uint32_t lo = it.lo;
  if (KC_R0_PASSA && v.r0) {
    uint32_t c = 0;
    stream_row<SOLVE_THREADS, true>(p.adj, snap, threadIdx.x, it.ob, it.ob + it.deg, s_cache,
                                    cache_n,
                                    [&](uint32_t ok, const uint32_t(&)[8], const uint32_t(&x)[8]) {
#pragma unroll
                                      for (int k = 0; k < 8; ++k) c += (ok >> k & 1) && x[k] >= it.cap;
                                    });
    const uint32_t cA = block_sum(c, sh.red);
    if (cA >= it.cap) {
      if (threadIdx.x == 0) finish_eval<PULL>(p, v, it, it.cap, cA, it.deg, acc);
      __syncthreads();
      return;
    }
    lo = cA;
  }
  uint32_t scanned = 0;
  if (it.list) {
    cta_window(p.radj, false, snap, s_cache, cache_n, s_hist, sh.red, it.ob, it.ob + it.len,
                      it.cap, lo > it.thr ? lo : it.thr, it.deg, !v.r0, sh.out, p.dc);
    scanned = it.len;
  } else if (threadIdx.x == 0) {
    sh.out[0] = 0;
  }
  __syncthreads();
  if (sh.out[0] == 0) {
    cta_window(p.adj, true, snap, s_cache, cache_n, s_hist, sh.red, it.ob, it.ob + it.deg, it.cap,
                     lo, it.deg, !v.r0, sh.out, p.dc);
    scanned += it.deg;
  }
  if (threadIdx.x == 0) finish_eval<PULL>(p, v, it, sh.out[0], sh.out[1], scanned, acc);
  __syncthreads();
}

// HUGE class.  Warps grab hubs one at a time and take those whose scan
// (list or row) is at most WARP_MAX_LEN; longer ones are appended to the
// phase's global long-scan queue, which CTAs drain one hub at a time
// (CTA-wide scan).  consume_long(false) takes what is already queued;
// consume_long(true) — at the end of the phase — keeps taking tickets until
// every CTA has finished appending and no ticket is left.
constexpr uint32_t NONE = 0xffffffffu;

template <typename OffT, typename EstT, typename WarpF>
__device__ void huge_warps(const CP<OffT, EstT>& p, const View<EstT>& v, Shared& sh, Ctl& ctl,
                           int ph, WarpF&& warp_fn) {
  const uint32_t cnt = v.qcnt[C_HUGE];
  if (cnt == 0) return;  // CTA- and grid-uniform
  uint32_t* cursor = &v.grab[C_HUGE];
  bool first = true;
  for (;;) {
    const uint32_t k = next_slice(cursor, cnt, 1u, first);
    if (k >= cnt) break;
    const uint32_t u = v.q ? v.q[p.cb[C_HUGE] + k] : p.cb[C_HUGE] + k;
    if (!warp_fn(u)) {  // too long for a warp: to the CTA-wide queue
      if (lane_id() == 0) {
        const uint32_t slot = atomicAdd(&ctl.lqn[ph], 1u);
        KC_BOUNDS(slot < p.cb[1] + 1);
        atomicExch(&p.lq[ph][slot], u);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&ctl.lqd[ph], 1u);
  }
}

template <typename OffT, typename EstT, typename CtaF>
__device__ void consume_long(const CP<OffT, EstT>& p, const View<EstT>& v, Shared& sh, Ctl& ctl,
                             int ph, bool wait, CtaF&& cta_fn) {
  if (v.qcnt[C_HUGE] == 0) return;
  volatile uint32_t* lqn = &ctl.lqn[ph];
  volatile uint32_t* lqc = &ctl.lqc[ph];
  volatile uint32_t* lqd = &ctl.lqd[ph];
  volatile uint32_t* lq = p.lq[ph];
  for (;;) {
    if (threadIdx.x == 0) {
      uint32_t k = sh.ticket, u = NONE;
      if (k == NONE && (wait || *lqc < *lqn)) k = atomicAdd(const_cast<uint32_t*>(lqc), 1u);
      while (k != NONE) {
        if (k < *lqn) {
          while ((u = lq[k]) == NONE) {}  // the appender's store is in flight
          lq[k] = NONE;
          k = NONE;
        } else if (!wait) {
          break;  // keep the ticket for the final drain
        } else if (*lqd == gridDim.x) {
          __threadfence();
          if (k >= *lqn) k = NONE;  // every hub is taken: done
        } else {
          __nanosleep(256);
        }
      }
      sh.ticket = k;
      sh.item = u;
    }
    __syncthreads();
    const uint32_t u = sh.item;
    __syncthreads();
    if (u == NONE) break;
    cta_fn(u);
  }
}

// WARP and BIG classes: warp per vertex; metadata of a grab loaded one lane
// per item, then walked.
template <bool PULL, typename OffT, typename EstT, typename A>
__device__ __forceinline__ void eval_wclass_impl(const CP<OffT, EstT>& p, const View<EstT>& v, const EstT* s_cache,
                            uint32_t* bins, int c, uint32_t gmax, A& acc) {
#if KC_R0_LANE
  if (KC_R0_SORTED && !PULL && v.r0 && p.dc.sorted) {
    // round 0 on sorted rows: a lane per vertex, two binary searches (r0_sorted_lane)
    for_class(p, v, c, 32u, [&](uint32_t u, uint32_t n) {
      if (lane_id() < n) {
        const Item it = eval_item<PULL>(p, v, s_cache, u);
        uint32_t probes = 0;
        const uint2 tc = r0_sorted_lane(p.adj, p.dc.t, it.ob, it.deg, it.cap, probes);
        finish_eval<PULL>(p, v, it, tc.x, tc.y, probes, acc);
      }
    });
    return;
  }
#endif
  for_class(p, v, c, gmax, [&](uint32_t u, uint32_t n) {
    Item mine{};
    if (lane_id() < n) {
      mine = eval_item<PULL>(p, v, s_cache, u);
      if (!mine.spec && !(KC_R0_SORTED && v.r0 && p.dc.sorted))  // (round 0 sorted: a prefix)
        l2_prefetch_ids((mine.list ? (const uint32_t*)p.radj : p.adj) + mine.ob, mine.len);
    }
    for (uint32_t i = 0; i < n; ++i) {
      Item it;
      it.u = __shfl_sync(FULL, mine.u, i);
      it.cap = __shfl_sync(FULL, mine.cap, i);
      it.lo = __shfl_sync(FULL, mine.lo, i);
      it.thr = __shfl_sync(FULL, mine.thr, i);
      it.len = __shfl_sync(FULL, mine.len, i);
      it.deg = __shfl_sync(FULL, mine.deg, i);
      it.ob = __shfl_sync(FULL, mine.ob, i);
      it.list = __shfl_sync(FULL, (uint32_t)mine.list, i) != 0;
      it.spec = __shfl_sync(FULL, (uint32_t)mine.spec, i) != 0;
      it.spec_t = __shfl_sync(FULL, mine.spec_t, i);
      it.spec_c = __shfl_sync(FULL, mine.spec_c, i);
      eval_warp<PULL>(p, v, s_cache, bins, it, acc);
    }
  });
}

// Counters in registers for the whole phase (an Acc& into the kernel's
// frame would be local-memory traffic per evaluation).
template <bool PULL, typename OffT, typename EstT>
__device__ KC_PHASE_FN void eval_wclass(const CP<OffT, EstT>& p_arg, const View<EstT>& v, const EstT* s_cache,
                            uint32_t* bins, int c, uint32_t gmax, Acc& acc) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  Acc32 a{0, 0, 0, 0, 0, 0, false};
  eval_wclass_impl<PULL>(p, v, s_cache, bins, c, gmax, a);
  merge_acc(acc, a);
}

// ------------------------------------------------------------------------
// Batched flat streams (rounds >= 1, BIG and WARP classes).  A warp takes G
// queued vertices and streams their lists / rows CONCATENATED, 256 entries
// per step, 8 consecutive entries per lane: every step keeps 8 id loads and
// 8 gathers in flight per lane however short the rows are, and the per-vertex
// work (window resolve, bookkeeping) is one lane's, not the warp's.
//
// Evaluate: for an active u, count(>= cap) = cnt[u] exactly (list or row) and
// lo <= t < cap, so only values in [L, cap) are binned, L = max(lo, thr,
// cap - FB); one lane per vertex then runs the suffix scan of
// kernel.hpp:36-41 over its FB bins.  A vertex whose level lies below its
// window takes the per-vertex windowed path afterwards.
// Notify: the same stream over the droppers' lists against N.  Droppers
// without a list (their first drop after round 0) take the per-vertex path,
// which builds the list.
// ------------------------------------------------------------------------
struct FlatW {                // per-warp batch state (shared memory)
  uint32_t pre[33];           // exclusive prefix of the segment lengths; pre[n] = total
  uint32_t hi[32];            // evaluate: cap; notify: cap (old estimate)
  uint32_t lo[32];            // evaluate: window floor L; notify: t (new estimate)
  uint32_t list[32];          // segment reads radj (1) or adj (0)
  unsigned long long ob[32];  // segment start in adj / radj
  uint32_t above[32];         // notify: count(N >= t) per segment (next-round evaluation)
  uint32_t slo[32];           // notify: floor of the segment's next-round window
};

__device__ __forceinline__ uint32_t flat_fb(uint32_t G) {  // bins per vertex
  return G <= 1u ? (uint32_t)WARP_BINS : (uint32_t)WARP_BINS >> (32 - __clz(G - 1u));
}

// Stream the batch: f(seg[8], ids[8], x[8], ok) per step.
template <typename OffT, typename EstT, typename F>
__device__ __forceinline__ void flat_stream(const CP<OffT, EstT>& p, const FlatW& fw, uint32_t n,
                                            const EstT* snap, const EstT* s_cache,
                                            uint32_t cache_n, F&& f) {
  const uint32_t lane = lane_id();
  const uint32_t total = fw.pre[n];
  for (uint32_t base = 0; base < total; base += 256) {
    const uint32_t first = base + 8 * lane;
    uint32_t s = 0;
    if (first < total) {  // segment of `first`: largest s with pre[s] <= first
      uint32_t a = 0, b = n;
      while (b - a > 1) {
        const uint32_t mid = (a + b) >> 1;
        if (fw.pre[mid] <= first) a = mid; else b = mid;
      }
      s = a;
    }
    uint32_t seg[8], ids[8], x[8], ok = 0;
    uint32_t s_pre = fw.pre[s], s_end = fw.pre[s + 1];
    const uint32_t* s_src = fw.list[s] ? p.radj : p.adj;
    uint64_t s_ob = fw.ob[s];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t e = first + j;
      const bool val = e < total;
      if (val && e >= s_end) {  // next non-empty segment
        do { ++s; } while (e >= fw.pre[s + 1]);
        s_pre = fw.pre[s];
        s_end = fw.pre[s + 1];
        s_src = fw.list[s] ? p.radj : p.adj;
        s_ob = fw.ob[s];
      }
      seg[j] = s;
      ok |= (uint32_t)val << j;
      ids[j] = val ? __ldcg(s_src + s_ob + (e - s_pre)) : 0u;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = (ok >> j & 1) ? est_at(s_cache, cache_n, snap, ids[j]) : 0u;
    f(seg, ids, x, ok);
  }
}

template <typename OffT, typename EstT, typename A>
__device__ __forceinline__ void flat_eval_impl(const CP<OffT, EstT>& p, const View<EstT>& v,
                                       const EstT* s_cache, uint32_t* bins, FlatW& fw, int c,
                                       uint32_t gmax, A& acc) {
  const uint32_t lane = lane_id();
  const EstT* snap = v.snap;
  const uint32_t cache_n = v.cache_n;
  const uint32_t fb = flat_fb(grab_size(v.qcnt[c], gmax));
  for_class(p, v, c, gmax, [&](uint32_t u, uint32_t n) {
    Item it{};
    uint32_t L = 0;
    if (lane < n) {
      it = eval_item<false>(p, v, s_cache, u);
      if (!it.spec) l2_prefetch_ids((it.list ? (const uint32_t*)p.radj : p.adj) + it.ob, it.len);
      L = it.lo;
      if (it.list && it.thr > L) L = it.thr;
      if (it.cap > fb && it.cap - fb > L) L = it.cap - fb;
      if (L < 1u) L = 1u;
    }
    if (lane < n && it.spec) finish_eval<false>(p, v, it, it.spec_t, it.spec_c, 0u, acc);
    const bool pending = lane < n && !it.spec;
    const uint32_t len = pending ? it.len : 0u;
    const uint32_t incl = warp_incl_scan(len);
    fw.pre[lane] = incl - len;
    if (lane == 31) fw.pre[32] = incl;
    fw.hi[lane] = it.cap;
    fw.lo[lane] = L;
    fw.list[lane] = it.list ? 1u : 0u;
    fw.ob[lane] = it.ob;
    for (uint32_t i = lane; i < (uint32_t)WARP_BINS; i += 32) bins[i] = 0;
    __syncwarp();
    if (n < 32 && lane == 0) fw.pre[n] = fw.pre[32];
    __syncwarp();
    flat_stream(p, fw, n, snap, s_cache, cache_n,
                [&](const uint32_t(&seg)[8], const uint32_t(&)[8], const uint32_t(&x)[8],
                    uint32_t ok) {
#pragma unroll
                  for (int j = 0; j < 8; ++j) {
                    if (!(ok >> j & 1)) continue;
                    const uint32_t sj = seg[j];
                    const uint32_t cp = fw.hi[sj];
                    if (x[j] < cp && x[j] >= fw.lo[sj]) {
                      KC_BOUNDS(sj < 32 && cp - 1 - x[j] < fb && sj * fb + (cp - 1 - x[j]) < (uint32_t)WARP_BINS);
                      atomicAdd(&bins[sj * fb + (cp - 1 - x[j])], 1u);
                    }
                  }
                });
    __syncwarp();
    // one lane per vertex: suffix scan of its window (C = count(>= cap) = lo)
    bool deep = false;
    if (pending) {
      uint32_t run = it.lo, t = 0;
      for (uint32_t k = 0; k < fb && it.cap - k > L; ++k) {
        const uint32_t level = it.cap - 1 - k;
        run += bins[lane * fb + k];
        if (run >= level) {
          t = level;
          break;
        }
      }
      if (t) finish_eval<false>(p, v, it, t, run, it.len, acc);
      else deep = true;  // below the window: per-vertex passes
    }
    uint32_t dm = __ballot_sync(FULL, deep);
    __syncwarp();
    while (dm) {
      const int i = __ffs(dm) - 1;
      dm &= dm - 1;
      Item d;
      d.u = __shfl_sync(FULL, it.u, i);
      d.cap = __shfl_sync(FULL, it.cap, i);
      d.lo = __shfl_sync(FULL, it.lo, i);
      d.thr = __shfl_sync(FULL, it.thr, i);
      d.len = __shfl_sync(FULL, it.len, i);
      d.deg = __shfl_sync(FULL, it.deg, i);
      d.ob = __shfl_sync(FULL, it.ob, i);
      d.list = __shfl_sync(FULL, (uint32_t)it.list, i) != 0;
      d.spec = false;
      eval_warp<false>(p, v, s_cache, bins, d, acc);
    }
  });
}

template <typename OffT, typename EstT>
__device__ KC_PHASE_FN void flat_eval(const CP<OffT, EstT>& p_arg, const View<EstT>& v,
                                       const EstT* s_cache, uint32_t* bins, FlatW& fw, int c,
                                       uint32_t gmax, Acc& acc) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  Acc32 a{0, 0, 0, 0, 0, 0, false};
  flat_eval_impl(p, v, s_cache, bins, fw, c, gmax, a);
  merge_acc(acc, a);
}

// SUB class (deg <= 64): 8-lane tile per vertex, 8 values per lane,
// bisection on [lo, cap).
// Round 0 on sorted rows (s_dcut: the cut table's first DEG_SUB_MAX + 2
// entries in shared memory) takes r0_sorted_warp's rule: no gathers.
template <bool PULL, typename OffT, typename EstT, typename A>
__device__ __forceinline__ void eval_sub_impl(const CP<OffT, EstT>& p, const View<EstT>& v, const EstT* s_cache,
                         const uint32_t* s_dcut, A& acc) {
  constexpr int R = DEG_SUB_MAX / 8;
  const uint32_t g = lane_id() >> 3, k = lane_id() & 7;
  const EstT* snap = v.snap;
  const uint32_t cache_n = v.cache_n;
  const bool r0 = v.r0;
  const bool r0s = KC_R0_SORTED && r0 && p.dc.sorted;
  for_class(p, v, C_SUB, GMAX_SMALL, [&](uint32_t mu, uint32_t n) {
    // metadata of the grab, one lane per item, loaded in parallel
    uint64_t mob = 0;
    uint32_t mdeg = 0, mcap = 0, mlo = 0;
    if (lane_id() < n) {
      mob = p.off[mu];
      mdeg = (uint32_t)(p.off[mu + 1] - mob);
      mcap = est_at(s_cache, cache_n, snap, mu);
      mlo = (r0 || PULL) ? 0u : p.cnt[mu];
    }
    for (uint32_t i0 = 0; i0 < n; i0 += 4) {
      // every lane runs the shuffles; tiles beyond n idle
      const int src = (int)(i0 + g) & 31;
      const uint32_t u = __shfl_sync(FULL, mu, src);
      const bool has = i0 + g < n;
      const uint64_t ob = __shfl_sync(FULL, mob, src);
      const uint32_t sdeg = __shfl_sync(FULL, mdeg, src);  // shuffles by every lane
      const uint32_t scap = __shfl_sync(FULL, mcap, src);
      const uint32_t deg = has ? sdeg : 0u;
      const uint32_t cap = has ? scap : 0u;
      const uint32_t lo = __shfl_sync(FULL, mlo, src);
      Vals<EstT, R> vals;
      vals.clear();
      {
        uint32_t ids[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const uint32_t q = k + 8 * j;
          ids[j] = q < deg ? p.adj[ob + q] : 0xffffffffu;
        }
        if (r0s) {
          const uint32_t m = deg < cap ? deg : cap;
          uint32_t hc = 0;
#pragma unroll
          for (int j = 0; j < R; ++j) hc += k + 8 * j < m && ids[j] < s_dcut[k + 8 * j + 1];
          const uint32_t t = tile8_sum(hc);
          const uint32_t ct = s_dcut[t];
          uint32_t cc = 0;
#pragma unroll
          for (int j = 0; j < R; ++j) cc += ids[j] < ct;
          const uint32_t c = tile8_sum(cc);
          if (has && k == 0) {
            Item it;
            it.u = u; it.cap = cap; it.deg = deg; it.len = deg; it.thr = 0;
            finish_eval<PULL>(p, v, it, t, t ? c : deg, deg, acc);
          }
          continue;
        }
#pragma unroll
        for (int j = 0; j < R; ++j)
          if (ids[j] != 0xffffffffu) vals.set(j, est_at(s_cache, cache_n, snap, ids[j]));
      }
      const uint32_t cA = tile8_sum(vals.count_ge(cap));
      uint32_t lo_b = lo, hi = cap;  // invariant: count(>= lo_b) >= lo_b
#pragma unroll 1
      for (int s = 0; s < 7; ++s) {  // cap <= 64
        const uint32_t mid = (lo_b + hi) >> 1;
        const bool okm = tile8_sum(vals.count_ge(mid)) >= mid;
        if (hi - lo_b > 1) {
          if (okm) lo_b = mid; else hi = mid;
        }
      }
      const uint32_t t = cA >= cap ? cap : lo_b;
      const uint32_t c = tile8_sum(vals.count_ge(t));
      if (has && k == 0) {
        Item it;
        it.u = u; it.cap = cap; it.deg = deg; it.len = deg; it.thr = 0;
        finish_eval<PULL>(p, v, it, t, c, deg, acc);
      }
    }
  });
}

template <bool PULL, typename OffT, typename EstT>
__device__ KC_PHASE_FN void eval_sub(const CP<OffT, EstT>& p_arg, const View<EstT>& v, const EstT* s_cache,
                         const uint32_t* s_dcut, Acc& acc) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  Acc32 a{0, 0, 0, 0, 0, 0, false};
  eval_sub_impl<PULL>(p, v, s_cache, s_dcut, a);
  merge_acc(acc, a);
}

// THREAD class (deg <= 8): thread per vertex, h = max_i min(x_i, #{x_j >= x_i}).
// A warp grabs up to GMAX_THREAD ids per atomic and each lane works TU
// vertices at a time, their loads issued level by level (offsets, ids,
// gathers) so that one lane keeps up to 8 * TU gathers in flight: a round
// of millions of degree-3 vertices (the road-like grid) is bound by memory
// parallelism, not by per-vertex latency or by the shared grab cursor.
#ifndef KC_TU
#define KC_TU 2
#endif
constexpr int TU = KC_TU;                       // evaluate: vertices per lane per pass
#ifndef KC_TUN
#define KC_TUN 2
#endif
constexpr int TUN = KC_TUN;                     // notify: droppers per lane per pass
constexpr uint32_t GMAX_THREAD = 32u * TU * 4u;  // ids per grab (max)

__device__ __forceinline__ uint32_t warp_grab(uint32_t* cursor, uint32_t cnt, uint32_t G) {
  uint32_t base = 0;
  if (lane_id() == 0)  // plain read first: no atomic once the queue is drained
    base = *reinterpret_cast<volatile uint32_t*>(cursor) >= cnt ? cnt : atomicAdd(cursor, G);
  return __shfl_sync(FULL, base, 0);
}

// Lane-level walk of class c's queue: proc(u[K], valid mask) per pass.
template <int K, typename OffT, typename EstT, typename F>
__device__ __forceinline__ void for_class_lanes(const CP<OffT, EstT>& p, const View<EstT>& v, int c,
                                                uint32_t gmax, F&& proc) {
  const uint32_t cnt = v.qcnt[c];
  if (cnt == 0) return;
  const uint32_t G = grab_size(cnt, gmax);
  const uint32_t lane = lane_id();
  bool first = true;
  for (;;) {
    const uint32_t base = next_slice(&v.grab[c], cnt, G, first);
    if (base >= cnt) break;
    const uint32_t n = cnt - base < G ? cnt - base : G;
    for (uint32_t s0 = 0; s0 < n; s0 += 32u * K) {
      uint32_t u[K], valid = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t i = s0 + lane + 32u * k;
        u[k] = 0;
        if (i < n) {
          u[k] = v.q ? v.q[p.cb[c] + base + i] : p.cb[c] + base + i;
          valid |= 1u << k;
        }
      }
      proc(u, valid);
    }
  }
}

template <bool PULL, typename OffT, typename EstT, typename A>
__device__ __forceinline__ void eval_thread_impl(const CP<OffT, EstT>& p, const View<EstT>& v, const EstT* s_cache,
                            const uint32_t* s_dcut, A& acc) {
  constexpr int R = DEG_THREAD_MAX;
  const EstT* snap = v.snap;
  const uint32_t cache_n = v.cache_n;
  const bool r0s = KC_R0_SORTED && v.r0 && p.dc.sorted;
  for_class_lanes<TU>(p, v, C_THREAD, GMAX_THREAD, [&](const uint32_t(&u)[TU], uint32_t valid) {
    uint64_t ob[TU];
    uint32_t deg[TU], cap[TU], x[TU][R];
#pragma unroll
    for (int k = 0; k < TU; ++k) {
      ob[k] = 0;
      deg[k] = cap[k] = 0;
      if (valid >> k & 1) {
        ob[k] = p.off[u[k]];
        deg[k] = (uint32_t)(p.off[u[k] + 1] - ob[k]);
        cap[k] = est_at(s_cache, cache_n, snap, u[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < TU; ++k)
#pragma unroll
      for (int j = 0; j < R; ++j) x[k][j] = (uint32_t)j < deg[k] ? p.adj[ob[k] + j] : 0xffffffffu;
    if (r0s) {  // round 0, sorted rows: r0_sorted_warp's rule on the ids (no gathers)
#pragma unroll
      for (int k = 0; k < TU; ++k) {
        if (!(valid >> k & 1)) continue;
        const uint32_t m = deg[k] < cap[k] ? deg[k] : cap[k];
        uint32_t t = 0;
#pragma unroll
        for (int j = 0; j < R; ++j) t += (uint32_t)j < m && x[k][j] < s_dcut[j + 1];
        const uint32_t ct = s_dcut[t];
        uint32_t c = 0;
#pragma unroll
        for (int j = 0; j < R; ++j) c += x[k][j] < ct;
        Item it;
        it.u = u[k]; it.cap = cap[k]; it.deg = deg[k]; it.len = deg[k]; it.thr = 0;
        finish_eval<PULL>(p, v, it, t, t ? c : deg[k], deg[k], acc);
      }
      return;
    }
#pragma unroll
    for (int k = 0; k < TU; ++k)
#pragma unroll
      for (int j = 0; j < R; ++j)
        x[k][j] = x[k][j] != 0xffffffffu ? est_at(s_cache, cache_n, snap, x[k][j]) : 0u;
#pragma unroll
    for (int k = 0; k < TU; ++k) {
      if (!(valid >> k & 1)) continue;
      uint32_t h = 0;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        uint32_t c = 0;
#pragma unroll
        for (int j = 0; j < R; ++j) c += x[k][j] >= x[k][i];
        const uint32_t m = x[k][i] < c ? x[k][i] : c;
        h = m > h ? m : h;
      }
      const uint32_t t = h < cap[k] ? h : cap[k];
      uint32_t c = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) c += x[k][j] >= t;
      Item it;
      it.u = u[k]; it.cap = cap[k]; it.deg = deg[k]; it.len = deg[k]; it.thr = 0;
      finish_eval<PULL>(p, v, it, t, t ? c : deg[k], deg[k], acc);
    }
  });
}

template <bool PULL, typename OffT, typename EstT>
__device__ KC_PHASE_FN void eval_thread(const CP<OffT, EstT>& p_arg, const View<EstT>& v, const EstT* s_cache,
                            const uint32_t* s_dcut, Acc& acc) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  Acc32 a{0, 0, 0, 0, 0, 0, false};
  eval_thread_impl<PULL>(p, v, s_cache, s_dcut, a);
  merge_acc(acc, a);
}

// ------------------------------------------------------------------------
// NOTIFY.  A dropper scans its list (or its CSR row, building the list when
// the row is longer than LIST_MIN_DEG) against the settled values N.
// ------------------------------------------------------------------------
__device__ __forceinline__ uint32_t list_threshold(uint32_t t) {
  const uint32_t L = t - (t >> KC_LIST_SHIFT);
  return L ? L : 1u;
}

// The notify scan gathers N over u's list — exactly the snapshot u's next
// evaluation would read (E of round r+1 = N of round r; N is not written
// during notify).  So the scan also evaluates u for round r+1 (`tag`):
// values >= t counted, [max(t - NB, floor), t) binned, suffix scan; the
// result is kept in spec_* and the next evaluate phase takes it instead of
// rescanning (it is used only if u is activated, which happens iff the
// level is below t).  floor = the list threshold (levels below it are not
// decided by the list) or 1.

// Returns the notifications fired by this lane (counted once per warp in
// `acc` by the callers).
template <bool CUT, typename OffT, typename EstT>
__device__ __forceinline__ uint32_t notify_warp(const CP<OffT, EstT>& p, const Enq& q,
                                             const EstT* s_cache, uint32_t cache_n,
                                             uint32_t* bins, const uint32_t* src, bool ro, uint32_t u,
                                             uint64_t ob, uint32_t len, uint32_t t, uint32_t cap,
                                             uint32_t build, uint32_t tag, uint32_t floor) {
  uint32_t cursor = 0;  // warp-uniform
  uint32_t fires = 0;
  uint32_t above = 0;
  const uint32_t sl = t > (uint32_t)KC_SPEC_BINS ? t - KC_SPEC_BINS : 1u;
  const uint32_t slo = floor > sl ? floor : sl;  // spec window [slo, t)
  // lowest value this scan looks at: t + 1 (notify), slo (spec), build (list)
  uint32_t need = t + 1;
  if (tag && slo < need) need = slo;
  if (build && build < need) need = build;
  if (tag) warp_zero_bins(bins);
  stream_row_rt<32>(src, ro, p.N, lane_id(), ob, ob + len, s_cache, cache_n,
                     [&](uint32_t ok, const uint32_t(&ids)[8], const uint32_t(&x)[8]) {
                       notify8(p, q, ok, ids, x, t, cap, fires);
                       if (tag) {
#pragma unroll
                         for (int k = 0; k < 8; ++k) {
                           if (!(ok >> k & 1)) continue;
                           if (x[k] >= t) ++above;
                           else if (x[k] >= slo) {
                             KC_BOUNDS(t - 1 - x[k] < (uint32_t)KC_SPEC_BINS);
                             atomicAdd(&bins[t - 1 - x[k]], 1u);
                           }
                         }
                       }
                       if (build) {
                         uint32_t keep = 0;
#pragma unroll
                         for (int k = 0; k < 8; ++k) keep |= (uint32_t)((ok >> k & 1) && x[k] >= build) << k;
                         const uint32_t nk = __popc(keep);
                         const uint32_t incl = warp_incl_scan(nk);
                         uint32_t pos = cursor + incl - nk;
#pragma unroll
                         for (int k = 0; k < 8; ++k)
                           if (keep >> k & 1) {
                             KC_BOUNDS(pos < len);  // a list is a subset of its row
                             p.radj[ob + pos++] = ids[k];
                           }
                         cursor += __shfl_sync(FULL, incl, 31);
                       }
                     }, CUT ? p.dc.at(need) : 0xffffffffu, CUT && ro && p.dc.sorted);
  if (tag) {
    __syncwarp();
    const uint32_t C = __reduce_add_sync(FULL, above);
    uint32_t lvl = t, cnt = C, b = 0, run = 0;
    bool ok = C >= t;  // no drop next round (u will not be activated)
    if (!ok && t > slo && warp_resolve_w(bins, C, t, 1u, slo, b, run)) {
      ok = true;
      lvl = t - 1 - b;
      cnt = run;
    }
    if (ok && lane_id() == 0) {
      p.spec_t[u] = lvl;
      p.spec_c[u] = cnt;
      p.spec_r[u] = tag;
    }
    __syncwarp();
  }
  if (lane_id() == 0) {
    if (build) {
      p.rlen[u] = cursor;
      p.rthr[u] = (EstT)build;
    }
    p.E[u] = (EstT)t;  // apply (fastk.cpp:153)
  }
  return fires;
}

template <typename OffT, typename EstT>
__device__ __noinline__ uint32_t notify_cta(const CP<OffT, EstT>& p_arg, const Enq& q,
                                            const EstT* s_cache, uint32_t cache_n, Shared& sh,
                                            uint32_t* s_hist, const uint32_t* src, bool ro, uint32_t u,
                                            uint64_t ob, uint32_t len, uint32_t t, uint32_t cap,
                                            uint32_t build, uint32_t tag, uint32_t floor) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  const uint32_t tid = threadIdx.x;
  if (tid == 0) sh.cursor = 0;
  // the CTA has HIST_BINS bins: a hub's next-round window reaches that far
  // below t (hubs drop by more than a warp window early on)
  const uint32_t sl = t > (uint32_t)KC_SPEC_CTA ? t - KC_SPEC_CTA : 1u;
  const uint32_t slo = floor > sl ? floor : sl;
  uint32_t need = t + 1;  // lowest value this scan looks at (see notify_warp)
  if (tag && slo < need) need = slo;
  if (build && build < need) need = build;
  if (tag)
    for (int i = tid; i < HIST_BINS; i += SOLVE_THREADS) s_hist[i] = 0;
  __syncthreads();
  uint32_t fires = 0, above = 0;
  stream_row_rt<SOLVE_THREADS>(src, ro, p.N, tid, ob, ob + len, s_cache, cache_n,
                                [&](uint32_t ok, const uint32_t(&ids)[8], const uint32_t(&x)[8]) {
                                  notify8(p, q, ok, ids, x, t, cap, fires);
                                  if (tag) {
#pragma unroll
                                    for (int k = 0; k < 8; ++k) {
                                      if (!(ok >> k & 1)) continue;
                                      if (x[k] >= t) ++above;
                                      else if (x[k] >= slo) {
                                        KC_BOUNDS(t - 1 - x[k] < (uint32_t)HIST_BINS);
                                        atomicAdd(&s_hist[t - 1 - x[k]], 1u);
                                      }
                                    }
                                  }
                                  if (build) {
                                    uint32_t keep = 0;
#pragma unroll
                                    for (int k = 0; k < 8; ++k)
                                      keep |= (uint32_t)((ok >> k & 1) && x[k] >= build) << k;
                                    const uint32_t nk = __popc(keep);
                                    const uint32_t incl = warp_incl_scan(nk);
                                    const uint32_t tot = __shfl_sync(FULL, incl, 31);
                                    uint32_t base = 0;
                                    if (lane_id() == 0 && tot) base = atomicAdd(&sh.cursor, tot);
                                    uint32_t pos = __shfl_sync(FULL, base, 0) + incl - nk;
#pragma unroll
                                    for (int k = 0; k < 8; ++k)
                                      if (keep >> k & 1) {
                                        KC_BOUNDS(pos < len);
                                        p.radj[ob + pos++] = ids[k];
                                      }
                                  }
                                }, KC_CUT_NOTIFY && (KC_CUT_LISTS || ro) ? p.dc.at(need) : 0xffffffffu, KC_CUT_NOTIFY && ro && p.dc.sorted);
  if (tag) {  // CTA suffix scan of the spec window (one pass, no refinement)
    const uint32_t C = block_sum(above, sh.red);
    constexpr int PER = (HIST_BINS + SOLVE_THREADS - 1) / SOLVE_THREADS;
    uint32_t h[PER];
    uint32_t sm = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      h[j] = tid * PER + j < HIST_BINS ? s_hist[tid * PER + j] : 0u;
      sm += h[j];
    }
    uint32_t run = C + block_excl_scan(sm, sh.red);
    uint32_t found = 0xffffffffu, frun = 0;
    if (C < t) {
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        run += h[j];
        const uint32_t i = tid * PER + j;
        if (found == 0xffffffffu && i < t - slo && run >= t - 1 - i) {
          found = i;
          frun = run;
        }
      }
    }
    const uint32_t g = block_min(found, sh.red);
    if (C >= t) {
      if (tid == 0) {
        p.spec_t[u] = t;
        p.spec_c[u] = C;
        p.spec_r[u] = tag;
      }
    } else if (g != 0xffffffffu && found == g) {
      p.spec_t[u] = t - 1 - g;
      p.spec_c[u] = frun;
      p.spec_r[u] = tag;
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (build) {
      p.rlen[u] = sh.cursor;
      p.rthr[u] = (EstT)build;
    }
    p.E[u] = (EstT)t;
  }
  __syncthreads();
  return fires;
}

struct Drop {
  uint32_t u, t, cap, thr, len, deg;
  uint64_t ob;
};

template <typename OffT, typename EstT>
__device__ __noinline__ uint32_t notify_row_warp(const CP<OffT, EstT>& p_arg, const Enq& q,
                                                 const EstT* s_cache, uint32_t cache_n,
                                                 uint32_t* bins, uint32_t u, uint64_t ob,
                                                 uint32_t len, uint32_t t, uint32_t cap,
                                                 uint32_t build, uint32_t tag) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  return notify_warp<true>(p, q, s_cache, cache_n, bins, p.adj, true, u, ob, len, t, cap, build,
                           tag, KC_ROW_FLOOR_BUILD && build ? build : 1u);
}

template <typename OffT, typename EstT>
__device__ __forceinline__ Drop drop_item(const CP<OffT, EstT>& p, uint32_t u) {
  Drop d;
  d.u = u;
  d.t = p.N[u];
  d.cap = p.E[u];
  d.ob = p.off[u];
  d.deg = (uint32_t)(p.off[u + 1] - d.ob);
  d.thr = 0;
  d.len = d.deg;
#if KC_FLAT_META
  const uint32_t thr = p.rthr[u], rl = p.rlen[u];  // same level as the loads above
  if (d.t < d.cap && d.deg > LIST_MIN_DEG && thr) {
    d.thr = thr;
    d.len = rl;
  }
#else
  if (d.t < d.cap && d.deg > LIST_MIN_DEG) {
    d.thr = p.rthr[u];
    if (d.thr) d.len = p.rlen[u];
  }
#endif
  return d;
}

__device__ __forceinline__ uint32_t list_build(bool r0, const Drop& d) {
  return ((KC_R0_LISTS || !r0) && d.deg > LIST_MIN_DEG) ? list_threshold(d.t) : 0u;
}

template <typename OffT, typename EstT>
__device__ __forceinline__ uint32_t notify_drop_warp(const CP<OffT, EstT>& p, const Enq& q,
                                                     const EstT* s_cache, uint32_t cache_n,
                                                     uint32_t* bins, uint32_t round,
                                                     const Drop& d) {
  const uint32_t tag = KC_SPEC ? round + 1 : 0u;
  // a list (optionally filtered in place), or the CSR row (building the list)
  const bool lst = d.thr != 0;
  if (KC_CUT_NOTIFY && !lst)  // CSR row: its own code (and register budget), cut at `need`
    return notify_row_warp(p, q, s_cache, cache_n, bins, d.u, d.ob, d.len, d.t, d.cap,
                           list_build(round == 0, d), tag);
  return notify_warp<false>(p, q, s_cache, cache_n, bins, lst ? (const uint32_t*)p.radj : p.adj,
                            !lst, d.u, d.ob, d.len, d.t, d.cap,
                            lst ? (KC_LIST_COMPACT ? d.thr : 0u) : list_build(round == 0, d), tag,
                            lst ? d.thr : 1u);
}

template <typename OffT, typename EstT, typename A>
__device__ __forceinline__ void notify_wclass_impl(const CP<OffT, EstT>& p, const View<EstT>& v,
                                           const Enq& q, const EstT* s_cache, uint32_t* bins,
                                           int c, uint32_t gmax, A& acc) {
  const uint32_t cache_n = v.cache_n;
  const bool r0 = v.r0;
  uint32_t fires = 0;
  uint32_t nscan = 0;
  for_class(p, v, c, gmax, [&](uint32_t u, uint32_t n) {
    Drop mine{};
    if (lane_id() < n) {
      mine = drop_item(p, u);
      if (mine.t < mine.cap)
        l2_prefetch_ids((mine.thr ? (const uint32_t*)p.radj : p.adj) + mine.ob, mine.len);
    }
    for (uint32_t i = 0; i < n; ++i) {
      Drop d;
      d.t = __shfl_sync(FULL, mine.t, i);
      d.cap = __shfl_sync(FULL, mine.cap, i);
      if (d.t >= d.cap) continue;  // round 0: evaluated, no drop (warp-uniform)
      d.u = __shfl_sync(FULL, mine.u, i);
      d.thr = __shfl_sync(FULL, mine.thr, i);
      d.len = __shfl_sync(FULL, mine.len, i);
      d.deg = __shfl_sync(FULL, mine.deg, i);
      d.ob = __shfl_sync(FULL, mine.ob, i);
      fires += notify_drop_warp(p, q, s_cache, cache_n, bins, v.round, d);
      nscan += d.len;
    }
  });
  acc.fires += fires;
  if (lane_id() == 0) acc.nscan += nscan;
}

template <typename OffT, typename EstT>
__device__ KC_PHASE_FN void notify_wclass(const CP<OffT, EstT>& p_arg, const View<EstT>& v,
                                           const Enq& q, const EstT* s_cache, uint32_t* bins,
                                           int c, uint32_t gmax, Acc& acc) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  Acc32 a{0, 0, 0, 0, 0, 0, false};
  notify_wclass_impl(p, v, q, s_cache, bins, c, gmax, a);
  merge_acc(acc, a);
}

template <typename OffT, typename EstT, typename A>
__device__ __forceinline__ void flat_notify_impl(const CP<OffT, EstT>& p, const View<EstT>& v,
                                         const Enq& q, const EstT* s_cache, uint32_t* bins,
                                         FlatW& fw, int c, uint32_t gmax, A& acc) {
  const uint32_t lane = lane_id();
  const uint32_t cache_n = v.cache_n;
  uint32_t fires = 0, nscan = 0;
  for_class(p, v, c, gmax, [&](uint32_t u, uint32_t n) {
    Drop d{};
    if (lane < n) d = drop_item(p, u);  // rounds >= 1: every queued vertex dropped
    const bool flat = lane < n && d.thr != 0;  // has a list: stream it in the batch
    const uint32_t len = flat ? d.len : 0u;
    const uint32_t incl = warp_incl_scan(len);
    fw.pre[lane] = incl - len;
    if (lane == 31) fw.pre[32] = incl;
    fw.hi[lane] = d.cap;
    fw.lo[lane] = d.t;
    fw.list[lane] = 1u;
    fw.ob[lane] = d.ob;
    __syncwarp();
    if (n < 32 && lane == 0) fw.pre[n] = fw.pre[32];
    __syncwarp();
    // next-round evaluation of each listed dropper (as notify_warp's spec):
    // values >= t counted, the FB levels below t binned, floor = the list
    // threshold (levels below it are not decided by the list)
    const uint32_t FB = flat_fb(grab_size(v.qcnt[c], gmax));
    {
      const uint32_t sl = d.t > FB ? d.t - FB : 1u;
      fw.slo[lane] = d.thr > sl ? d.thr : sl;
      fw.above[lane] = 0;
      for (uint32_t i = lane; i < (uint32_t)WARP_BINS; i += 32) bins[i] = 0;
    }
    __syncwarp();
    nscan += len;
    flat_stream(p, fw, n, (const EstT*)p.N, s_cache, cache_n,
                [&](const uint32_t(&seg)[8], const uint32_t(&ids)[8], const uint32_t(&x)[8],
                    uint32_t ok) {
                  uint32_t fire = 0;
                  uint32_t cs = seg[0], cc = 0;  // run of this lane's entries in one segment
#pragma unroll
                  for (int j = 0; j < 8; ++j) {
                    const uint32_t sj = seg[j];
                    const uint32_t tj = fw.lo[sj];
                    const bool v = ok >> j & 1;
                    const bool f = v && tj < x[j] && x[j] <= fw.hi[sj];
                    fire |= (uint32_t)f << j;
                    if (sj != cs) {
                      if (cc) atomicAdd(&fw.above[cs], cc);
                      cs = sj;
                      cc = 0;
                    }
                    if (v && x[j] >= tj) ++cc;
                    else if (v && x[j] >= fw.slo[sj]) {
                      KC_BOUNDS(tj - 1 - x[j] < FB && sj * FB + (tj - 1 - x[j]) < (uint32_t)WARP_BINS);
                      atomicAdd(&bins[sj * FB + (tj - 1 - x[j])], 1u);
                    }
                  }
                  if (cc) atomicAdd(&fw.above[cs], cc);
                  uint32_t act = 0;
                  if (fire) {
                    fires += __popc(fire);
                    uint32_t old[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                      old[j] = (fire >> j & 1) ? atomicSub(&p.cnt[ids[j]], 1u) : 0u;
#pragma unroll
                    for (int j = 0; j < 8; ++j) act |= (uint32_t)((fire >> j & 1) && old[j] == x[j]) << j;
                  }
                  if (__any_sync(FULL, act)) {
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                      if (__any_sync(FULL, act >> j & 1)) wq_push(p, q, (act >> j & 1) != 0, ids[j]);
                  }
                });
    __syncwarp();
    if (KC_SPEC && flat) {  // lane = segment: resolve the window (kernel.hpp:36-41)
      const uint32_t C = fw.above[lane];
      uint32_t lvl = d.t, run = C;
      bool found = C >= d.t;  // no drop next round
      for (uint32_t k = 0; !found && k < FB && d.t - 1 - k >= fw.slo[lane]; ++k) {
        run += bins[lane * FB + k];
        if (run >= d.t - 1 - k) {
          lvl = d.t - 1 - k;
          found = true;
        }
      }
      if (found) {
        p.spec_t[d.u] = lvl;
        p.spec_c[d.u] = run;
        p.spec_r[d.u] = v.round + 1;
      }
    }
    __syncwarp();
    if (flat) p.E[d.u] = (EstT)d.t;  // apply (fastk.cpp:153)
    // droppers without a list: per-vertex pass that builds it
    uint32_t rest = __ballot_sync(FULL, lane < n && !flat);
    while (rest) {
      const int i = __ffs(rest) - 1;
      rest &= rest - 1;
      Drop e;
      e.u = __shfl_sync(FULL, d.u, i);
      e.t = __shfl_sync(FULL, d.t, i);
      e.cap = __shfl_sync(FULL, d.cap, i);
      e.thr = __shfl_sync(FULL, d.thr, i);
      e.len = __shfl_sync(FULL, d.len, i);
      e.deg = __shfl_sync(FULL, d.deg, i);
      e.ob = __shfl_sync(FULL, d.ob, i);
      fires += notify_drop_warp(p, q, s_cache, cache_n, bins, v.round, e);
      if (lane == 0) nscan += e.len;
    }
  });
  acc.fires += fires;
  acc.nscan += nscan;
}

template <typename OffT, typename EstT>
__device__ KC_PHASE_FN void flat_notify(const CP<OffT, EstT>& p_arg, const View<EstT>& v,
                                         const Enq& q, const EstT* s_cache, uint32_t* bins,
                                         FlatW& fw, int c, uint32_t gmax, Acc& acc) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  Acc32 a{0, 0, 0, 0, 0, 0, false};
  flat_notify_impl(p, v, q, s_cache, bins, fw, c, gmax, a);
  merge_acc(acc, a);
}

// SUB and THREAD droppers: 8-lane tile per dropper, up to 8 neighbours per lane.
template <typename OffT, typename EstT, typename A>
__device__ __forceinline__ void notify_small_impl(const CP<OffT, EstT>& p, const View<EstT>& v,
                                          const Enq& q, const EstT* s_cache, int c, A& acc) {
  const uint32_t g = lane_id() >> 3, k = lane_id() & 7;
  const uint32_t cache_n = v.cache_n;
  uint32_t fires = 0, nscan = 0;
  for_class(p, v, c, GMAX_SMALL, [&](uint32_t mu, uint32_t n) {
    // the slice's estimates and offsets, one lane per item, in one level of
    // loads for all of its items (not one round trip per 4-item step)
    uint32_t mt = 0, mcap = 0, mdeg = 0;
    uint64_t mob = 0;
    if (lane_id() < n) {
      mt = p.N[mu];
      mcap = p.E[mu];
      mob = p.off[mu];
      mdeg = (uint32_t)(p.off[mu + 1] - mob);
      if (!(mt < mcap)) mdeg = 0;
    }
    for (uint32_t i0 = 0; i0 < n; i0 += 4) {
      const int src = (int)(i0 + g) & 31;
      const uint32_t u = __shfl_sync(FULL, mu, src);
      const bool has = i0 + g < n;
      const uint32_t st = __shfl_sync(FULL, mt, src), scap = __shfl_sync(FULL, mcap, src);
      const uint32_t sdeg = __shfl_sync(FULL, mdeg, src);
      const uint64_t sob = __shfl_sync(FULL, mob, src);
      const uint32_t t = has ? st : 0u, cap = has ? scap : 0u, deg = has ? sdeg : 0u;
      const uint64_t ob = has ? sob : 0ull;
      uint32_t ids[8], x[8], ok = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bool val = k + 8u * j < deg;
        ids[j] = val ? p.adj[ob + k + 8u * j] : 0u;
        ok |= (uint32_t)val << j;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        x[j] = (ok >> j & 1) ? est_at(s_cache, cache_n, (const EstT*)p.N, ids[j]) : 0u;
      notify8(p, q, ok, ids, x, t, cap, fires);  // warp-converged
      if (k == 0 && t < cap) {
        nscan += deg;
        p.E[u] = (EstT)t;
      }
    }
  });
  acc.fires += fires;
  acc.nscan += nscan;
}

template <typename OffT, typename EstT>
__device__ KC_PHASE_FN void notify_small(const CP<OffT, EstT>& p_arg, const View<EstT>& v,
                                          const Enq& q, const EstT* s_cache, int c, Acc& acc) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  Acc32 a{0, 0, 0, 0, 0, 0, false};
  notify_small_impl(p, v, q, s_cache, c, a);
  merge_acc(acc, a);
}

// THREAD droppers: lane per dropper, TUN droppers per lane per pass, loads
// issued level by level (estimates, offsets, ids, gathers, counters).
template <typename OffT, typename EstT, typename A>
__device__ __forceinline__ void notify_thread_impl(const CP<OffT, EstT>& p, const View<EstT>& v,
                                           const Enq& q, const EstT* s_cache, A& acc) {
  constexpr int R = DEG_THREAD_MAX;
  const uint32_t cache_n = v.cache_n;
  uint32_t fires = 0, nscan = 0;
  for_class_lanes<TUN>(p, v, C_THREAD, GMAX_THREAD, [&](const uint32_t(&u)[TUN], uint32_t valid) {
    uint32_t t[TUN], cap[TUN], deg[TUN], ids[TUN][R], x[TUN][R];
    uint64_t ob[TUN];
    // estimates and offsets in one level (offsets of non-droppers are
    // loaded for nothing: cheaper than another dependent round trip)
#pragma unroll
    for (int k = 0; k < TUN; ++k) {
      t[k] = cap[k] = 0;
      ob[k] = 0;
      deg[k] = 0;
      if (valid >> k & 1) {
        t[k] = p.N[u[k]];
        cap[k] = p.E[u[k]];
        ob[k] = p.off[u[k]];
        deg[k] = (uint32_t)(p.off[u[k] + 1] - ob[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < TUN; ++k)
      if (!(t[k] < cap[k])) deg[k] = 0;  // not dropped this round
#pragma unroll
    for (int k = 0; k < TUN; ++k)
#pragma unroll
      for (int j = 0; j < R; ++j) ids[k][j] = (uint32_t)j < deg[k] ? p.adj[ob[k] + j] : 0u;
#pragma unroll
    for (int k = 0; k < TUN; ++k)
#pragma unroll
      for (int j = 0; j < R; ++j)
        x[k][j] = (uint32_t)j < deg[k] ? est_at(s_cache, cache_n, (const EstT*)p.N, ids[k][j]) : 0u;
    // should_notify(t, cap, N[w]) (fastk.hpp:25-27) == the drop removes u
    // from w's support count; the decrement that crosses N[w] activates w
    uint32_t act[TUN];
#pragma unroll
    for (int k = 0; k < TUN; ++k) {
      uint32_t fire = 0;
#pragma unroll
      for (int j = 0; j < R; ++j)
        fire |= (uint32_t)((uint32_t)j < deg[k] && t[k] < x[k][j] && x[k][j] <= cap[k]) << j;
      fires += __popc(fire);
      uint32_t old[R];
#pragma unroll
      for (int j = 0; j < R; ++j) old[j] = (fire >> j & 1) ? atomicSub(&p.cnt[ids[k][j]], 1u) : 0u;
      act[k] = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) act[k] |= (uint32_t)((fire >> j & 1) && old[j] == x[k][j]) << j;
      if (t[k] < cap[k]) {
        nscan += deg[k];
        p.E[u[k]] = (EstT)t[k];  // apply (fastk.cpp:153)
      }
    }
#pragma unroll
    for (int k = 0; k < TUN; ++k)
      if (__any_sync(FULL, act[k])) {
#pragma unroll
        for (int j = 0; j < R; ++j)
          if (__any_sync(FULL, act[k] >> j & 1)) wq_push(p, q, (act[k] >> j & 1) != 0, ids[k][j]);
      }
  });
  acc.fires += fires;
  acc.nscan += nscan;
}

template <typename OffT, typename EstT>
__device__ KC_PHASE_FN void notify_thread(const CP<OffT, EstT>& p_arg, const View<EstT>& v,
                                           const Enq& q, const EstT* s_cache, Acc& acc) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  Acc32 a{0, 0, 0, 0, 0, 0, false};
  notify_thread_impl(p, v, q, s_cache, a);
  merge_acc(acc, a);
}

template <typename OffT, typename EstT>
__device__ __forceinline__ void flush_acc(const CP<OffT, EstT>& p, uint32_t sr, const Acc& acc,
                                          unsigned long long* s_acc) {
  const unsigned long long val[6] = {acc.evals, acc.escan, acc.drops, acc.fires, acc.nscan, acc.ascan};
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    unsigned long long x = val[q];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(FULL, x, d);
    if (lane_id() == 0 && x) atomicAdd(&s_acc[q], x);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    RoundStat& st = p.stats[sr];
    unsigned long long* dst[6] = {&st.evals, &st.escan, &st.drops, &st.fires, &st.nscan, &st.ascan};
#pragma unroll
    for (int q = 0; q < 6; ++q)
      if (s_acc[q]) atomicAdd(dst[q], s_acc[q]);
  }
}

// The EVALUATE phase (every class; the long-scan queue of slot `ph`), inline
// in the kernel body; its PULL instance runs out of line (pull_phase).
template <bool PULL, typename OffT, typename EstT>
__device__ __forceinline__ void eval_phase(const CP<OffT, EstT>& p, const View<EstT>& v, Shared& sh,
                                        Ctl& ctl, int ph, const EstT* s_cache, uint32_t* s_hist,
                                        uint32_t* w_bins, FlatW& fw, const uint32_t* s_dcut,
                                        unsigned long long* pf, Acc& acc) {
  auto eval_long = [&](uint32_t u) { eval_cta<PULL>(p, v, s_cache, s_hist, sh, u, acc); };
  huge_warps(p, v, sh, ctl, ph, [&](uint32_t u) {
    const Item it = eval_item<PULL>(p, v, s_cache, u);  // metadata loaded once
    // (round 0 on sorted rows reads a prefix only: always a warp's)
    if (it.len > v.wml && !(KC_R0_SORTED && v.r0 && p.dc.sorted)) return false;
    eval_warp<PULL>(p, v, s_cache, w_bins, it, acc);
    return true;
  });
  consume_long(p, v, sh, ctl, ph, false, eval_long);
  if (pf) pf[2] = gtimer();
  KC_BOUNDS(blockDim.x == SOLVE_THREADS);
  // (empty classes skip the out-of-line calls: their prologues and epilogues
  // cost ~1 us each in the small rounds, scripts/round_overhead.py)
  if (v.r0 || PULL || !KC_FLAT_EVAL) {
    if (v.qcnt[C_BIG]) eval_wclass<PULL>(p, v, s_cache, w_bins, C_BIG, GMAX_BIG, acc);
    if (v.qcnt[C_WARP]) eval_wclass<PULL>(p, v, s_cache, w_bins, C_WARP, GMAX_WARP, acc);
  } else {
    if (v.qcnt[C_BIG]) flat_eval(p, v, s_cache, w_bins, fw, C_BIG, GMAX_BIG, acc);
    if (v.qcnt[C_WARP]) flat_eval(p, v, s_cache, w_bins, fw, C_WARP, GMAX_WARP, acc);
  }
  if (pf) pf[3] = gtimer();
  if (v.qcnt[C_SUB]) eval_sub<PULL>(p, v, s_cache, s_dcut, acc);
  if (v.qcnt[C_THREAD]) eval_thread<PULL>(p, v, s_cache, s_dcut, acc);
  consume_long(p, v, sh, ctl, ph, true, eval_long);
  if (pf) pf[4] = gtimer();
}

template <typename OffT, typename EstT>
__device__ __noinline__ void pull_phase(const CP<OffT, EstT>& p_arg, const View<EstT>& v, Shared& sh,
                                        Ctl& ctl, const EstT* s_cache, uint32_t* s_hist,
                                        uint32_t* w_bins, FlatW& fw, const uint32_t* s_dcut,
                                        Acc& acc) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  // phase stamps of PULL (debug): the last profile row, slots 1-4
  unsigned long long* pf = (p.prof && threadIdx.x == 0)
                               ? p.prof + ((size_t)(PROF_ROUNDS - 1) * gridDim.x + blockIdx.x) * PROF_PHASES
                               : nullptr;
  if (pf) pf[1] = gtimer();
  eval_phase<true>(p, v, sh, ctl, 1, s_cache, s_hist, w_bins, fw, s_dcut, pf, acc);
}

// After PULL: the flagged round-1 droppers become round 1's queue (class
// segments, ids ascending within a CTA block), their new level moves from
// spec_t into N, and round 1's evaluation counters are added.  CTAs take
// interleaved blocks of PULL_IDS ids; each thread reads 16 flags with one
// 128-bit load; one block scan and one atomicAdd per CTA block.
constexpr uint32_t PULL_IDS = SOLVE_THREADS * 16;

template <typename OffT, typename EstT>
__device__ __noinline__ void compact_pull(const CP<OffT, EstT>& p_arg, uint32_t* qcnt, uint32_t* queue,
                             Shared& sh, RoundStat& st) {
  const CP<OffT, EstT>& p = c_params<OffT, EstT>;  // constant bank, not p_arg
  (void)p_arg;
  const uint32_t tid = threadIdx.x;
  unsigned long long evals = 0, escan = 0;
  for (int c = 0; c < NCLS; ++c) {
    const uint32_t b0 = p.cb[c], b1 = p.cb[c + 1];
    const uint32_t a0 = b0 & ~15u;
    const uint32_t nblk = (b1 - a0 + PULL_IDS - 1) / PULL_IDS;
    for (uint32_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
      const uint32_t a = a0 + blk * PULL_IDS + 16 * tid;
      uint4 w = make_uint4(0, 0, 0, 0);
      if (a < b1) w = *reinterpret_cast<const uint4*>(p.pflag + a);
      uint32_t m = 0;  // bit j: id a+j dropped and inside the class
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t word = j < 4 ? w.x : j < 8 ? w.y : j < 12 ? w.z : w.w;
        const uint32_t id = a + j;
        if ((word >> (8 * (j & 3)) & 0xffu) && id >= b0 && id < b1) m |= 1u << j;
      }
      const uint32_t mine = __popc(m);
      const uint32_t off = block_excl_scan(mine, sh.red);
      if (tid == SOLVE_THREADS - 1) {
        const uint32_t tot = off + mine;
        sh.item = tot ? atomicAdd(&qcnt[c], tot) : 0u;
      }
      __syncthreads();
      uint32_t pos = b0 + sh.item + off;
      __syncthreads();
      if (m) {
#pragma unroll 1
        for (int j = 0; j < 16; ++j)
          if (m >> j & 1) {
            const uint32_t u = a + j;
            KC_BOUNDS(pos < b1);
            queue[pos++] = u;
            p.pflag[u] = 0;
            p.N[u] = (EstT)p.spec_t[u];
            evals += 1;
            escan += (uint64_t)(p.off[u + 1] - p.off[u]);
          }
      }
    }
  }
  evals = __reduce_add_sync(FULL, (uint32_t)evals);
  for (int d = 16; d > 0; d >>= 1) escan += __shfl_xor_sync(FULL, escan, d);
  if (lane_id() == 0 && evals) {
    atomicAdd(&st.evals, evals);
    atomicAdd(&st.drops, evals);
    atomicAdd(&st.escan, escan);
  }
}

// The NOTIFY + APPLY phase of round v.round (every class; the long-scan queue
// of slot 1), shared by the persistent kernel and the per-phase kernel.
template <typename OffT, typename EstT>
__device__ __forceinline__ void notify_phase(const CP<OffT, EstT>& p, const View<EstT>& v,
                                             const Enq& q, Shared& sh, Ctl& ctl,
                                             const EstT* s_cache, uint32_t* s_hist,
                                             uint32_t* w_bins, FlatW& fw, uint32_t* wn, Acc& acc) {
  const uint32_t tid = threadIdx.x;
  const uint32_t cache_n = v.cache_n;
  const uint32_t r = v.round;
  auto notify_long = [&](uint32_t u) {
    const Drop d = drop_item(p, u);  // a long-queued hub always dropped
    const uint32_t f =
        d.thr ? notify_cta(p, q, s_cache, cache_n, sh, s_hist, p.radj, false, d.u, d.ob, d.len,
                           d.t, d.cap, 0u, KC_SPEC ? r + 1 : 0u, d.thr)
              : notify_cta(p, q, s_cache, cache_n, sh, s_hist, p.adj, true, d.u, d.ob, d.len,
                           d.t, d.cap, list_build(v.r0, d), KC_SPEC ? r + 1 : 0u,
                           KC_ROW_FLOOR_BUILD && list_build(v.r0, d) ? list_build(v.r0, d) : 1u);
    acc.fires += f;
    if (tid == 0) acc.nscan += d.len;
  };
  huge_warps(p, v, sh, ctl, 1, [&](uint32_t u) {
    const Drop d = drop_item(p, u);  // metadata loaded once
    if (d.t >= d.cap) return true;   // round 0: evaluated, no drop
    if (d.len > v.wml) return false;
    acc.fires += notify_drop_warp(p, q, s_cache, cache_n, w_bins, r, d);
    if (lane_id() == 0) acc.nscan += d.len;
    return true;
  });
  consume_long(p, v, sh, ctl, 1, false, notify_long);
  if (v.r0 || !KC_FLAT_NOTIFY) {
    if (v.qcnt[C_BIG]) notify_wclass(p, v, q, s_cache, w_bins, C_BIG, GMAX_BIG, acc);
    if (v.qcnt[C_WARP]) notify_wclass(p, v, q, s_cache, w_bins, C_WARP, GMAX_WARP, acc);
  } else {
    if (v.qcnt[C_BIG]) flat_notify(p, v, q, s_cache, w_bins, fw, C_BIG, GMAX_BIG, acc);
    if (v.qcnt[C_WARP]) flat_notify(p, v, q, s_cache, w_bins, fw, C_WARP, GMAX_WARP, acc);
  }
  if (v.qcnt[C_SUB]) notify_small(p, v, q, s_cache, C_SUB, acc);
  if (v.qcnt[C_THREAD]) notify_thread(p, v, q, s_cache, acc);
  consume_long(p, v, sh, ctl, 1, true, notify_long);
  if (__any_sync(FULL, lane_id() < (uint32_t)NCLS && wn[lane_id()] != 0u)) wq_flush_all(p, q);
}

// Round-start bookkeeping by CTA 0: the next round's queue sizes and cursors
// (idle until the notify phase) and this round's queue sizes for the stats.
template <typename OffT, typename EstT>
__device__ __forceinline__ void round_start_ctl(const CP<OffT, EstT>& p, uint32_t nxt, uint32_t sr,
                                                const uint32_t* qcnt) {
  const uint32_t tid = threadIdx.x;
  if (blockIdx.x != 0) return;
  if (tid < NCLS) {
    p.ctl[nxt].grab[tid] = 0;
    p.ctl[nxt].grab2[tid] = 0;
    p.ctl[nxt].qcnt[tid] = 0;
    if (tid < 2) p.ctl[nxt].lqn[tid] = p.ctl[nxt].lqc[tid] = p.ctl[nxt].lqd[tid] = 0;
  }
  if (tid == 32) {
    p.stats[sr].q01 = qcnt[0] | (unsigned long long)qcnt[1] << 32;
    p.stats[sr].q23 = qcnt[2] | (unsigned long long)qcnt[3] << 32;
    p.stats[sr].q4 = qcnt[4];
  }
}

#if !KC_TU_SPLIT
template <typename OffT, typename EstT>
__global__ void __launch_bounds__(SOLVE_THREADS, 1) count_rounds_kernel(const __grid_constant__ CP<OffT, EstT> p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem[];
  EstT* s_cache = opaque_ptr(reinterpret_cast<EstT*>(smem));  // see opaque_ptr
  const size_t cache_bytes = ((size_t)p.cache_n * sizeof(EstT) + 15) & ~(size_t)15;
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(smem + cache_bytes);  // CTA window / warp bins
  uint32_t* w_bins = s_hist + WARP_BINS * warp_id();
  uint32_t* s_wq = s_hist + HREG;  // per-warp enqueue buffers
  __shared__ uint32_t s_wn[NWARPS][NCLS];
  __shared__ FlatW s_flat[(KC_FLAT_EVAL || KC_FLAT_NOTIFY) ? NWARPS : 1];
  __shared__ Shared sh;
  __shared__ uint32_t s_qcnt[NCLS];
  __shared__ uint32_t s_dcut[DEG_SUB_MAX + 2];  // head of the degree cut table (round 0)
  // the phase's view, published in shared memory: the noinline phase
  // functions read it through a reference (a stack copy would be local
  // memory, which misses L1 under this kernel's stack footprint)
  __shared__ View<EstT> s_view;
  __shared__ __align__(8) unsigned long long s_mbar;  // the cache fills' TMA barrier
  uint32_t fill_phase = 0;
  const View<EstT>& v = s_view;
  uint32_t* wn = s_wn[warp_id()];
  const uint32_t tid = threadIdx.x;
  Enq q;
  q.wbuf = s_wq + (size_t)warp_id() * NCLS * WQ;
  q.wn = wn;
  if (tid == 0) mbar_init(&s_mbar);
  if (tid == 0) sh.ticket = 0xffffffffu;
  if (lane_id() < NCLS) wn[lane_id()] = 0;
  if (tid < DEG_SUB_MAX + 2) s_dcut[tid] = p.dc.at(tid);
  __syncthreads();
  bool evaluated = false;  // this round's evaluation already ran (PULL did round 1's)
  uint32_t r_first = p.r_begin;
  if (p.r_begin == R_RESUME) {
    // after the per-phase kernels (kc_count_split.cu): carry on at the round
    // they stopped before (nobody writes status before the first grid barrier)
    if (p.status[1]) return;  // they ran to convergence
    r_first = p.status[0];
    evaluated = r_first == 1 && p.pull;  // PULL ran, round 1's notify did not
  }

  for (uint32_t r = r_first; r < p.r_end; ++r) {
    const uint32_t cur = r & 1, nxt = cur ^ 1;
    const uint32_t sr = r < STAT_SLOTS - 1 ? r : STAT_SLOTS - 1;
    View<EstT> vl;
    vl.snap = p.E;
    vl.q = r == 0 ? nullptr : p.queue[cur];
    // this round's class sizes, final since the last grid barrier: one
    // global read per CTA, then shared memory for every grab loop
    if (tid < NCLS) s_qcnt[tid] = p.ctl[cur].qcnt[tid];
    __syncthreads();
    vl.qcnt = s_qcnt;
    vl.grab = p.ctl[cur].grab;
    vl.qn = p.ctl[nxt].qcnt;
    vl.qnext = p.queue[nxt];
    q.qn = vl.qn;
    q.qnext = vl.qnext;
    vl.r0 = r == 0;
    vl.pull = false;
    vl.round = r;
    vl.wml = WARP_MAX_LEN;
    unsigned long long* pf = (p.prof && r < PROF_ROUNDS && tid == 0)
                                 ? p.prof + ((size_t)r * gridDim.x + blockIdx.x) * PROF_PHASES
                                 : nullptr;
    if (pf) pf[0] = gtimer();
    uint32_t active = 0;
#pragma unroll
    for (int c = 0; c < NCLS; ++c) active += vl.qcnt[c];
    if (r > 0 && active == 0) {  // quiescent round: converged (fastk.cpp:109-110)
      if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = r + 1;
        p.status[1] = 1;
        p.status[3] = 0;
      }
      if (pf) pf[1] = pf[2] = pf[3] = pf[4] = pf[5] = pf[6] = pf[7] = gtimer();
      return;
    }
    round_start_ctl(p, nxt, sr, vl.qcnt);
    if (tid < 6) sh.acc[tid] = 0;
    if (tid == 0) sh.drop = 0;
    const uint32_t cache_n = active >= CACHE_MIN_ACTIVE ? p.cache_n : 0u;
    vl.cache_n = cache_n;
    if (r > 0 && active < WML_SMALL_ACTIVE) vl.wml = WML_SMALL;
    if (cache_n && !evaluated) fill_cache_bulk(smem, s_cache, (const EstT*)p.E, cache_n, &s_mbar, fill_phase);
    if (tid == 0) s_view = vl;
    __syncthreads();
    Acc acc{0, 0, 0, 0, 0, 0, false};
    if (pf) pf[1] = gtimer();
    // ---------------- EVALUATE ----------------
    Ctl& ctl = p.ctl[cur];
    if (!evaluated) {
    eval_phase<false>(p, v, sh, ctl, 0, s_cache, s_hist, w_bins, s_flat[warp_id()], s_dcut, pf, acc);
    if (v.r0) {
      if (__any_sync(FULL, acc.any_drop) && lane_id() == 0) sh.drop = 1;
      __syncthreads();
      if (tid == 0 && sh.drop) p.anydrop[0] = 1;
    }
    grid.sync();
    }  // !evaluated
    evaluated = false;
    // The reference starts at est = deg (fastk.cpp:67-68); the solver starts
    // at min(deg, H), so round 0 "changed" also when some degree exceeds H
    // (that drop is already applied).  Keeps iterations equal to the reference.
    if (v.r0 && !(*reinterpret_cast<volatile uint32_t*>(&p.anydrop[0]) != 0 || p.clamp_drop)) {
      flush_acc(p, sr, acc, sh.acc);
      if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = 1;
        p.status[1] = 1;
        p.status[3] = 0;
      }
      if (pf) pf[5] = pf[6] = pf[7] = gtimer();
      return;
    }
    if (pf) pf[5] = gtimer();
    if (v.r0 && p.pull) {
      // ---------------- PULL (round 0's notify + round 1's evaluate) ----------------
      // Round 1's snapshot is N (round 0's settled levels).  Instead of every
      // round-0 dropper pushing counter decrements to its neighbours (one
      // atomic per fire: 176 M on R-MAT 26) and round 1 then evaluating the
      // vertices the decrements activated, every vertex evaluates itself
      // against N once: cap = N[v], t = capped h-index over N, c = count(N
      // >= t).  cnt[v] = c is exactly the counter the decrements would have
      // left (count(N >= N[v]) when v does not drop) or round 1's evaluation
      // stores; a vertex drops (t < cap) iff its counter would have crossed
      // below N[v], i.e. iff round 0's notify would have activated it.  So
      // the Jacobi trajectory, the evaluations (V_eval, E_scan) and round 1's
      // queue are unchanged; only round 0's push (and its decrements) goes.
      // The apply E[v] = N[v] is done here; the new levels wait in spec_t
      // until the compaction (N is being read).
      vl.snap = p.N;
      vl.grab = p.ctl[cur].grab2;
      vl.r0 = false;
      vl.pull = true;
      if (cache_n) fill_cache_bulk(smem, s_cache, (const EstT*)p.N, cache_n, &s_mbar, fill_phase);
      if (tid == 0) s_view = vl;
      __syncthreads();
      if (pf) pf[6] = gtimer();
      pull_phase(p, v, sh, ctl, s_cache, s_hist, w_bins, s_flat[warp_id()], s_dcut, acc);
      flush_acc(p, sr, acc, sh.acc);
      grid.sync();
      compact_pull(p, p.ctl[nxt].qcnt, p.queue[nxt], sh, p.stats[1 < STAT_SLOTS - 1 ? 1 : STAT_SLOTS - 1]);
      grid.sync();
      if (pf) pf[7] = gtimer();
      if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = r + 1;
        p.status[3] = 0;
      }
      evaluated = true;  // round 1 starts at its notify phase
      continue;
    }
    // ---------------- NOTIFY + APPLY ----------------
    vl.snap = p.N;
    vl.grab = p.ctl[cur].grab2;
    if (cache_n) fill_cache_bulk(smem, s_cache, (const EstT*)p.N, cache_n, &s_mbar, fill_phase);
    if (tid == 0) s_view = vl;
    __syncthreads();
    if (pf) pf[6] = gtimer();
    notify_phase(p, v, q, sh, ctl, s_cache, s_hist, w_bins, s_flat[warp_id()], wn, acc);
    flush_acc(p, sr, acc, sh.acc);
    grid.sync();
    if (pf) pf[7] = gtimer();
    if (blockIdx.x == 0 && tid == 0) {
      p.status[0] = r + 1;
      p.status[3] = 0;
    }
  }
}
#endif  // !KC_TU_SPLIT

#if KC_TU_SPLIT
// ------------------------------------------------------------------------
// One phase of one round per launch (the large rounds): PH 0 = round start +
// EVALUATE, PH 1 = NOTIFY + APPLY.  The kernel boundary is the grid barrier.
// Each kernel has the register budget of its own phase (the phase functions
// are inlined here: no ABI calls, no callee-save spills) and KC_SPLIT_CTAS
// CTAs per SM, i.e. more resident warps than the persistent kernel's one CTA:
// the phases are chains of dependent memory round trips per vertex, bound by
// how many of them an SM keeps in flight.
//
// No host round trip: the host queues the kernels of rounds [r_lo, r_hi] and
// then the persistent kernel (R_RESUME).  The EVALUATE kernel of a round that
// starts with fewer than `split_min` active vertices (or none: converged)
// sets status[ST_HANDOFF]; every later per-phase kernel then returns at once
// and the persistent kernel carries on at round status[0].  All CTAs of a
// kernel take the same decision from the (final) queue sizes.
// ------------------------------------------------------------------------
template <int PH, typename OffT, typename EstT>
__global__ void __launch_bounds__(SOLVE_THREADS, KC_SPLIT_CTAS)
    count_phase_kernel(const __grid_constant__ CP<OffT, EstT> p, const uint32_t r,
                       const uint32_t skip_eval, const uint32_t split_min) {
  if (p.status[1] | p.status[ST_HANDOFF]) return;
  extern __shared__ __align__(16) unsigned char smem[];
  EstT* s_cache = opaque_ptr(reinterpret_cast<EstT*>(smem));  // see opaque_ptr
  const size_t cache_bytes = ((size_t)p.cache_n * sizeof(EstT) + 15) & ~(size_t)15;
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(smem + cache_bytes);  // CTA window / warp bins
  uint32_t* w_bins = s_hist + WARP_BINS * warp_id();
  uint32_t* s_wq = s_hist + HREG;  // per-warp enqueue buffers (PH 1)
  __shared__ uint32_t s_wn[NWARPS][NCLS];
  constexpr bool FLAT = PH == 0 ? KC_FLAT_EVAL != 0 : KC_FLAT_NOTIFY != 0;
  __shared__ FlatW s_flat[FLAT ? NWARPS : 1];
  FlatW& fw = s_flat[FLAT ? warp_id() : 0];
  __shared__ Shared sh;
  __shared__ uint32_t s_qcnt[NCLS];
  __shared__ View<EstT> s_view;
  __shared__ __align__(8) unsigned long long s_mbar;  // the cache fill's TMA barrier
  uint32_t fill_phase = 0;
  const View<EstT>& v = s_view;
  uint32_t* wn = s_wn[warp_id()];
  const uint32_t tid = threadIdx.x;
  const uint32_t cur = r & 1, nxt = cur ^ 1;
  const uint32_t sr = r < STAT_SLOTS - 1 ? r : STAT_SLOTS - 1;
  if (tid == 0) mbar_init(&s_mbar);
  if (tid == 0) sh.ticket = 0xffffffffu;
  if (lane_id() < NCLS) wn[lane_id()] = 0;
  if (tid < NCLS) s_qcnt[tid] = p.ctl[cur].qcnt[tid];
  if (tid < 6) sh.acc[tid] = 0;
  __syncthreads();
  uint32_t active = 0;
#pragma unroll
  for (int c = 0; c < NCLS; ++c) active += s_qcnt[c];
  // stamps: the first prof_ctas CTAs only (the profile rows are that wide)
  unsigned long long* pf = (p.prof && r < PROF_ROUNDS && tid == 0 && blockIdx.x < p.prof_ctas)
                               ? p.prof + ((size_t)r * p.prof_ctas + blockIdx.x) * PROF_PHASES
                               : nullptr;
  View<EstT> vl;
  vl.q = p.queue[cur];
  vl.qcnt = s_qcnt;
  vl.qn = p.ctl[nxt].qcnt;
  vl.qnext = p.queue[nxt];
  vl.r0 = false;
  vl.pull = false;
  vl.round = r;
  vl.wml = active < WML_SMALL_ACTIVE ? WML_SMALL : WARP_MAX_LEN;
  const uint32_t cache_n = active >= CACHE_MIN_ACTIVE ? p.cache_n : 0u;
  vl.cache_n = cache_n;
  Ctl& ctl = p.ctl[cur];
  Acc acc{0, 0, 0, 0, 0, 0, false};
  if (PH == 0) {
    if (pf) pf[0] = gtimer();
    if (active == 0) {  // quiescent round: converged (fastk.cpp:109-110)
      if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = r + 1;
        p.status[1] = 1;
        p.status[3] = 0;
      }
      if (pf) pf[1] = pf[2] = pf[3] = pf[4] = pf[5] = pf[6] = pf[7] = gtimer();
      return;
    }
    if (active < split_min) {  // small round: the persistent kernel takes over
      if (blockIdx.x == 0 && tid == 0) p.status[ST_HANDOFF] = 1;
      return;
    }
    round_start_ctl(p, nxt, sr, s_qcnt);
    if (skip_eval) return;  // round 1 after PULL: evaluated already
    vl.snap = p.E;
    vl.grab = p.ctl[cur].grab;
    if (cache_n) fill_cache_bulk(smem, s_cache, (const EstT*)p.E, cache_n, &s_mbar, fill_phase);
    if (tid == 0) s_view = vl;
    __syncthreads();
    if (pf) pf[1] = gtimer();
    eval_phase<false>(p, v, sh, ctl, 0, s_cache, s_hist, w_bins, fw, (const uint32_t*)nullptr, pf,
                      acc);
    flush_acc(p, sr, acc, sh.acc);
    if (pf) pf[5] = gtimer();
  } else {
    Enq q;
    q.wbuf = s_wq + (size_t)warp_id() * NCLS * WQ;
    q.wn = wn;
    q.qn = vl.qn;
    q.qnext = vl.qnext;
    if (blockIdx.x == 0 && tid == 0) {  // rounds completed once this kernel has
      p.status[0] = r + 1;
      p.status[3] = 0;
    }
    vl.snap = p.N;
    vl.grab = p.ctl[cur].grab2;
    if (cache_n) fill_cache_bulk(smem, s_cache, (const EstT*)p.N, cache_n, &s_mbar, fill_phase);
    if (tid == 0) s_view = vl;
    __syncthreads();
    if (pf) pf[6] = gtimer();
    notify_phase(p, v, q, sh, ctl, s_cache, s_hist, w_bins, fw, wn, acc);
    flush_acc(p, sr, acc, sh.acc);
    if (pf) pf[7] = gtimer();
  }
}
#endif  // KC_TU_SPLIT


// Round-0 state: E = N = min(deg, H), no lists, the round-0
// "queue" is every vertex (class sizes), everything else cleared.
template <typename OffT, typename EstT>
__global__ void count_init_kernel(CP<OffT, EstT> p, uint32_t h_graph, uint32_t n_pad) {
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
    p.rthr[u] = 0;
    p.spec_r[u] = 0;
  }
  for (uint32_t k = gtid; k < STAT_SLOTS * (uint32_t)(sizeof(RoundStat) / 8); k += gsize)
    reinterpret_cast<unsigned long long*>(p.stats)[k] = 0;
  if (gtid < NCLS) {
    p.ctl[0].grab[gtid] = p.ctl[0].grab2[gtid] = 0;
    p.ctl[0].qcnt[gtid] = p.cb[gtid + 1] - p.cb[gtid];
    p.ctl[1].grab[gtid] = p.ctl[1].grab2[gtid] = p.ctl[1].qcnt[gtid] = 0;
  }
  if (gtid < 2)
    for (int q = 0; q < 2; ++q) p.ctl[q].lqn[gtid] = p.ctl[q].lqc[gtid] = p.ctl[q].lqd[gtid] = 0;
  if (gtid < 3) p.anydrop[gtid] = 0;
  if (gtid < ST_SLOTS) p.status[gtid] = 0;
}

template <typename OffT, typename EstT>
CP<OffT, EstT> make_params(const SolveBuffers& b) {
  CP<OffT, EstT> p{};
  p.off = static_cast<const OffT*>(b.off);
  p.adj = b.adj;
  p.dc.t = KC_DCUT ? b.dcut : nullptr;
  p.dc.n = b.dcut_n;
  p.dc.sorted = p.dc.t && b.rows_sorted;
  p.radj = b.radj;
  p.rlen = b.rlen;
  p.rthr = static_cast<EstT*>(b.rthr);
  const size_t n_pad = ((size_t)b.n_nz + 15) & ~(size_t)15;
  p.spec_r = b.spec;
  p.spec_t = b.spec + n_pad;
  p.spec_c = b.spec + 2 * n_pad;
  p.pflag = b.pflag;
  p.n_nz = b.n_nz;
  for (int c = 0; c <= NCLS; ++c) p.cb[c] = b.cls_begin[c];
  p.E = static_cast<EstT*>(b.est[0]);
  p.N = static_cast<EstT*>(b.est[1]);
  p.cnt = b.cnt;
  p.queue[0] = b.queue;
  p.queue[1] = b.queue2;
  p.lq[0] = b.lq[0];
  p.lq[1] = b.lq[1];
  p.ctl = b.ctl;
  p.anydrop = b.anydrop;
  p.stats = b.stats;
  p.status = b.status;
  p.prof = b.prof;
  p.prof_ctas = b.prof_ctas;
  return p;
}

#if !KC_TU_SPLIT
template <typename OffT, typename EstT>
cudaError_t launch_t(const SolveBuffers& b, const SolveConfig& c, uint32_t r_begin, uint32_t r_end,
                     bool pull_alone, cudaStream_t stream) {
  CP<OffT, EstT> p = make_params<OffT, EstT>(b);
  p.r_begin = r_begin;
  p.r_end = r_end;
  p.cache_n = c.cache_n;
  p.clamp_drop = c.clamp_drop;
  // PULL covers round 0's notify and round 1's evaluate: launches that run
  // both, or (pull_alone) round 0 alone when the per-phase kernels follow
  p.pull = c.pull && (r_begin == R_RESUME || (r_begin == 0 && (r_end >= 2 || pull_alone)));
  const size_t smem = (((size_t)c.cache_n * sizeof(EstT) + 15) & ~(size_t)15) +
                      ((size_t)HREG + (size_t)NWARPS * NCLS * WQ) * sizeof(uint32_t);
  auto kern = count_rounds_kernel<OffT, EstT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SOLVE_THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  dim3 grid(c.num_sms), block(SOLVE_THREADS);
  void* args[] = {&p};
  // c_params is one copy per device: order this solve's copy after the
  // previous solve's kernel (whatever its stream) and publish our own end
  static std::mutex mu;
  static cudaEvent_t done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  cudaEvent_t& ev = done[dev & 63];
  if (!ev && (e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(stream, ev, 0)) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbolAsync(c_params<OffT, EstT>, &p, sizeof(p), 0, cudaMemcpyHostToDevice,
                                   stream)) != cudaSuccess)
    return e;
  e = cudaLaunchCooperativeKernel((const void*)kern, grid, block, args, smem, stream);
  if (e != cudaSuccess) return e;
  return cudaEventRecord(ev, stream);
}

#endif  // !KC_TU_SPLIT

#if !KC_TU_SPLIT
template <typename OffT, typename EstT>
cudaError_t init_t(const SolveBuffers& b, uint32_t h_graph, cudaStream_t stream) {
  CP<OffT, EstT> p = make_params<OffT, EstT>(b);
  const uint32_t n_pad = (b.n_nz + 15) & ~15u;
  count_init_kernel<OffT, EstT><<<148 * 4, 256, 0, stream>>>(p, h_graph, n_pad);
  return cudaGetLastError();
}

#endif  // !KC_TU_SPLIT

#if KC_TU_SPLIT
template <typename OffT, typename EstT>
cudaError_t phases_t(const SolveBuffers& b, const SolveConfig& c, uint32_t r_lo, uint32_t r_hi,
                     bool skip_first_eval, cudaStream_t stream) {
  CP<OffT, EstT> p = make_params<OffT, EstT>(b);
  p.r_begin = r_lo;
  p.r_end = r_hi + 1;
  p.cache_n = c.split_cache ? c.cache_n : 0u;
  p.clamp_drop = c.clamp_drop;
  p.pull = false;
  const size_t smem = (((size_t)p.cache_n * sizeof(EstT) + 15) & ~(size_t)15) +
                      ((size_t)HREG + (size_t)NWARPS * NCLS * WQ) * sizeof(uint32_t);
  const void* kern[2] = {(const void*)count_phase_kernel<0, OffT, EstT>,
                         (const void*)count_phase_kernel<1, OffT, EstT>};
  int per_sm = KC_SPLIT_CTAS;
  for (int ph = 0; ph < 2; ++ph) {
    cudaError_t e = cudaFuncSetAttribute(kern[ph], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int k = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k, kern[ph], SOLVE_THREADS, smem);
    if (e != cudaSuccess) return e;
    if (k < 1) return cudaErrorInvalidConfiguration;
    if (k < per_sm) per_sm = k;
  }
  // every CTA resident (cooperative launch): the long-scan queue's final
  // drain waits for all CTAs of the kernel (consume_long)
  dim3 grid(c.num_sms * per_sm), block(SOLVE_THREADS);
  static std::mutex mu;
  static cudaEvent_t done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  cudaEvent_t& ev = done[dev & 63];
  cudaError_t e;
  if (!ev && (e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(stream, ev, 0)) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbolAsync(c_params<OffT, EstT>, &p, sizeof(p), 0, cudaMemcpyHostToDevice,
                                   stream)) != cudaSuccess)
    return e;
  for (uint32_t r = r_lo; r <= r_hi; ++r) {
    uint32_t rr = r, skip = (r == r_lo && skip_first_eval) ? 1u : 0u, smin = c.split_min;
    void* args[] = {&p, &rr, &skip, &smin};
    for (int ph = 0; ph < 2; ++ph)
      if ((e = cudaLaunchCooperativeKernel(kern[ph], grid, block, args, smem, stream)) != cudaSuccess)
        return e;
  }
  return cudaEventRecord(ev, stream);
}
#endif  // KC_TU_SPLIT

}  // namespace

#if KC_TU_SPLIT
cudaError_t launch_count_phases(const SolveBuffers& b, const SolveConfig& c, bool est16, bool off64,
                                uint32_t r_lo, uint32_t r_hi, bool skip_first_eval,
                                cudaStream_t stream) {
  if (est16)
    return off64 ? phases_t<uint64_t, uint16_t>(b, c, r_lo, r_hi, skip_first_eval, stream)
                 : phases_t<uint32_t, uint16_t>(b, c, r_lo, r_hi, skip_first_eval, stream);
  return off64 ? phases_t<uint64_t, uint32_t>(b, c, r_lo, r_hi, skip_first_eval, stream)
               : phases_t<uint32_t, uint32_t>(b, c, r_lo, r_hi, skip_first_eval, stream);
}
#endif  // KC_TU_SPLIT

#if !KC_TU_SPLIT
cudaError_t launch_count_rounds(const SolveBuffers& b, const SolveConfig& c, bool est16, bool off64,
                                uint32_t r_begin, uint32_t r_end, cudaStream_t stream) {
  auto persistent = [&](uint32_t r0, uint32_t r1, bool pull_alone) {
    if (est16)
      return off64 ? launch_t<uint64_t, uint16_t>(b, c, r0, r1, pull_alone, stream)
                   : launch_t<uint32_t, uint16_t>(b, c, r0, r1, pull_alone, stream);
    return off64 ? launch_t<uint64_t, uint32_t>(b, c, r0, r1, pull_alone, stream)
                 : launch_t<uint32_t, uint32_t>(b, c, r0, r1, pull_alone, stream);
  };
  // A whole solve with the large rounds on the per-phase kernels
  // (kc_count_split.cu): round 0 (+ PULL) here, rounds 1 .. split_rounds one
  // kernel per phase until a round starts small, the rest here again.
  if (c.split_rounds && r_begin == 0 && r_end > 2) {
    cudaError_t e = persistent(0, 1, true);
    if (e != cudaSuccess) return e;
    const uint32_t r_hi = c.split_rounds < r_end - 1 ? c.split_rounds : r_end - 1;
    e = launch_count_phases(b, c, est16, off64, 1, r_hi, c.pull != 0, stream);
    if (e != cudaSuccess) return e;
    return persistent(R_RESUME, r_end, false);
  }
  return persistent(r_begin, r_end, false);
}

cudaError_t launch_count_init(const SolveBuffers& b, bool est16, bool off64, uint32_t h_graph,
                              cudaStream_t stream) {
  if (est16)
    return off64 ? init_t<uint64_t, uint16_t>(b, h_graph, stream)
                 : init_t<uint32_t, uint16_t>(b, h_graph, stream);
  return off64 ? init_t<uint64_t, uint32_t>(b, h_graph, stream)
               : init_t<uint32_t, uint32_t>(b, h_graph, stream);
}

#endif  // !KC_TU_SPLIT

}  // namespace kcb
