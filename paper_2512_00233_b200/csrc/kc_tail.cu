// kc_tail.cu — FastK's hybrid sequential tail on the device.
//
// Reference: sequential_tail, /root/reference/proj/src/fastk.cpp:28-55, and
// the switch in the barrier completion, fastk.cpp:102-118 / fastk.hpp:29-31:
// once a round changed something but fewer than `batch` vertices are active,
// the reference stops the parallel rounds and finishes on one thread with a
// min-priority queue of (estimate at push, vertex), lazy deletion of stale
// entries, immediate apply and immediate notification.
//
// The queue discipline reduces to a rule that needs no heap:
//   - an active v always has an entry (est[v], v) (it is pushed with its
//     current estimate, and est[v] only changes when v itself is popped);
//   - entries never carry a key below the vertex's current estimate;
//   so the next non-stale pop is the ACTIVE vertex with the smallest
//   (est[v], v) — v in the caller's (reference) ids, hence `perm` — and
//   every pushed entry is popped exactly once:
//       tail_pops = (active vertices at the switch) + (notifications fired
//                   in the tail).
// The device tail keeps the active set as an unordered list plus byte flags
// and takes a CTA-wide argmin per step.  Same pops, same order, same
// estimates, same counters as the reference.
//
// Two launches on the solver's stream:
//   tail_list_kernel  (grid)    active flags -> list
//   tail_kernel       (1 CTA)   the sequential loop
// Both are no-ops unless the rounds kernel stopped for the tail
// (status[2] == 1) or the caller forces the tail (observed mode).
#include <cstdint>

#include "kc_internal.h"

namespace kcb {
namespace {

constexpr int TB = 1024;                    // tail CTA
constexpr int TW = TB / 32;
constexpr uint32_t TAIL_BINS = 16384;       // h-index histogram (64 KB shared)
constexpr uint32_t KEYCAP = 4096;           // active list mirrored in shared memory up to this size
constexpr unsigned FULLM = 0xffffffffu;

struct TailState {     // device scalars
  uint32_t m;          // list length
  uint32_t pad;
};

template <typename OffT, typename EstT>
struct TP {
  const OffT* off;
  const uint32_t* adj;
  EstT* E;
  EstT* N;
  const uint32_t* perm;  // new id -> caller id (the reference's NodeId)
  uint8_t* flag[2];
  uint32_t* list;        // [n_nz]
  TailState* ts;
  unsigned long long* tc;  // tail counters (kc_internal.h TAIL_*)
  uint32_t* status;
  uint32_t n_nz;
  int ext;
  int force_flags;       // >= 0: take the active set from flag[force_flags]
};

template <typename OffT, typename EstT>
__device__ __forceinline__ bool tail_on(const TP<OffT, EstT>& p) {
  return p.force_flags >= 0 || p.status[2] == 1;
}
template <typename OffT, typename EstT>
__device__ __forceinline__ uint8_t* tail_flags(const TP<OffT, EstT>& p) {
  // the rounds kernel stopped at the start of round status[0], whose active
  // set it left in flag[status[0] & 1]
  return p.flag[p.force_flags >= 0 ? p.force_flags : (p.status[0] & 1)];
}

template <typename OffT, typename EstT>
__global__ void tail_list_kernel(TP<OffT, EstT> p) {
  if (!tail_on(p)) return;
  const uint8_t* fl = tail_flags(p);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x; base < p.n_nz; base += stride) {
    const uint32_t u = base + threadIdx.x;
    const bool a = u < p.n_nz && fl[u] != 0;
    const uint32_t m = __ballot_sync(FULLM, a);
    if (!m) continue;
    uint32_t pos = 0;
    if (lane == 0) pos = atomicAdd(&p.ts->m, (uint32_t)__popc(m));
    pos = __shfl_sync(FULLM, pos, 0);
    if (a) p.list[pos + __popc(m & ((1u << lane) - 1u))] = u;
  }
}

__device__ __forceinline__ unsigned long long blk_min64(unsigned long long v,
                                                        unsigned long long* red) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long o = __shfl_xor_sync(FULLM, v, d);
    v = o < v ? o : v;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long w = red[threadIdx.x];  // TW == 32
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned long long o = __shfl_xor_sync(FULLM, w, d);
      w = o < w ? o : w;
    }
    if (threadIdx.x == 0) red[32] = w;
  }
  __syncthreads();
  const unsigned long long r = red[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ uint32_t blk_sum(uint32_t v, uint32_t* red) {
  v = __reduce_add_sync(FULLM, v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    const uint32_t w = __reduce_add_sync(FULLM, red[threadIdx.x]);
    if (threadIdx.x == 0) red[32] = w;
  }
  __syncthreads();
  const uint32_t r = red[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ uint32_t blk_max(uint32_t v, uint32_t* red) {
  v = __reduce_max_sync(FULLM, v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    const uint32_t w = __reduce_max_sync(FULLM, red[threadIdx.x]);
    if (threadIdx.x == 0) red[32] = w;
  }
  __syncthreads();
  const uint32_t r = red[32];
  __syncthreads();
  return r;
}

// Suffix sum over the CTA in thread order: sum of v over threads > tid.
__device__ __forceinline__ uint32_t blk_suffix_excl(uint32_t v, uint32_t* red) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = v;  // inclusive suffix within the warp (lanes >= lane)
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_down_sync(FULLM, incl, d);
    if (lane + d < 32) incl += y;
  }
  if (lane == 0) red[w] = incl;  // warp total
  __syncthreads();
  uint32_t above = 0;
  for (uint32_t k = w + 1; k < (uint32_t)TW; ++k) above += red[k];
  __syncthreads();
  return above + incl - v;
}

// compute_index_over (include/kcore/kernel.hpp:27-42) of u at cap, CTA-wide:
// the largest t <= cap with #{neighbours: min(est, cap) >= t} >= t; 0 when
// cap == 0.
// e0: the estimate of entry tid (tid < deg), gathered by the caller.
template <typename OffT, typename EstT>
__device__ uint32_t tail_index(const TP<OffT, EstT>& p, uint64_t ob, uint32_t deg, uint32_t cap,
                               uint32_t e0, uint32_t* hist, uint32_t* red) {
  if (cap == 0) return 0;  // kernel.hpp:30
  const uint32_t tid = threadIdx.x;
  if (cap < TAIL_BINS) {
    // histogram counts[min(e, cap)] (kernel.hpp:31-35), bins [0, cap]
    for (uint32_t i = tid; i <= cap; i += TB) hist[i] = 0;
    __syncthreads();
    for (uint32_t j = tid; j < deg; j += TB) {
      const uint32_t e = j == tid ? e0 : p.E[p.adj[ob + j]];
      atomicAdd(&hist[e < cap ? e : cap], 1u);
    }
    __syncthreads();
    // suffix scan t = cap..1 (kernel.hpp:36-41): thread k owns the bins
    // [lo_k, hi_k) of a contiguous split of [1, cap]
    const uint32_t per = (cap + TB - 1) / TB;
    const uint32_t lo = 1 + tid * per, hi = lo + per < cap + 1 ? lo + per : cap + 1;
    uint32_t s = 0;
    for (uint32_t b = lo; b < hi; ++b) s += hist[b];
    uint32_t run = blk_suffix_excl(s, red);  // count(>= hi)
    uint32_t best = 0;
    for (uint32_t b = hi; b > lo;) {
      --b;
      run += hist[b];
      if (run >= b) {
        best = b;
        break;
      }
    }
    const uint32_t t = blk_max(best, red);
    return t;
  }
  // wide estimates (32-bit graphs with H >= TAIL_BINS): bisection on
  // count(>= x) >= x over [0, cap], one pass over the row per probe
  uint32_t lo = 0, hi = cap;  // invariant: lo qualifies
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo + 1) / 2;
    uint32_t c = 0;
    for (uint32_t j = tid; j < deg; j += TB) c += p.E[p.adj[ob + j]] >= mid;
    if (blk_sum(c, red) >= mid) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <typename OffT, typename EstT>
__global__ void __launch_bounds__(TB, 1) tail_kernel(TP<OffT, EstT> p) {
  if (!tail_on(p)) return;
  extern __shared__ uint32_t hist[];
  // The active list's pop keys (est, caller id) never change while an entry
  // waits (only the popped vertex's estimate moves), so while the list holds
  // at most KEYCAP entries it is mirrored in shared memory: the argmin of a
  // pop reads no global memory.  Past KEYCAP the global list alone is used.
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(hist + TAIL_BINS);
  uint32_t* s_id = reinterpret_cast<uint32_t*>(s_key + KEYCAP);
  __shared__ unsigned long long red64[33];
  __shared__ uint32_t red[33];
  __shared__ uint32_t s_m, s_idx, s_u, s_fires;
  uint8_t* act = tail_flags(p);
  const uint32_t tid = threadIdx.x;
  if (tid == 0) s_m = p.ts->m;
  __syncthreads();
  const uint32_t m0 = s_m;
  bool mir = m0 <= KEYCAP;
  if (mir)
    for (uint32_t i = tid; i < m0; i += TB) {
      const uint32_t v = p.list[i];
      s_id[i] = v;
      s_key[i] = (unsigned long long)p.E[v] << 32 | p.perm[v];
    }
  __syncthreads();
  unsigned long long pops_done = 0, escan = 0, drops = 0, fires = 0;
  for (;;) {
    const uint32_t m = s_m;
    if (m == 0) break;
    if (m > KEYCAP) mir = false;  // (uniform: s_m is read after a barrier)
    // the active vertex with the smallest (est, caller id)
    unsigned long long best = ~0ull;
    for (uint32_t i = tid; i < m; i += TB) {
      const unsigned long long key =
          mir ? s_key[i] : (unsigned long long)p.E[p.list[i]] << 32 | p.perm[p.list[i]];
      best = key < best ? key : best;
    }
    const unsigned long long kmin = blk_min64(best, red64);
    for (uint32_t i = tid; i < m; i += TB) {
      const uint32_t v = mir ? s_id[i] : p.list[i];
      if ((mir ? s_key[i] : (unsigned long long)p.E[v] << 32 | p.perm[v]) == kmin) {
        s_idx = i;  // keys are unique (perm is a bijection)
        s_u = v;
      }
    }
    __syncthreads();
    const uint32_t u = s_u;
    if (tid == 0) {
      if (mir) {
        s_key[s_idx] = s_key[m - 1];
        s_id[s_idx] = s_id[m - 1];
      }
      p.list[s_idx] = p.list[m - 1];  // unordered list: swap-remove
      s_m = m - 1;
      act[u] = 0;  // fastk.cpp:41
      s_fires = 0;
    }
    ++pops_done;  // fastk.cpp:42 (messages_drained)
    const uint64_t ob = (uint64_t)p.off[u];
    const uint32_t deg = (uint32_t)((uint64_t)p.off[u + 1] - ob);
    escan += deg;
    const uint32_t cap = p.E[u];
    // the first TB row entries and their estimates stay in registers for
    // both scans of this pop (only u's own estimate changes in between)
    const uint32_t v0 = tid < deg ? p.adj[ob + tid] : 0u;
    const uint32_t e0 = tid < deg ? (uint32_t)p.E[v0] : 0u;
    const uint32_t t = tail_index(p, ob, deg, cap, e0, hist, red);  // fastk.cpp:43-44
    if (t < cap) {  // fastk.cpp:45-46: apply immediately
      ++drops;
      __syncthreads();
      if (tid == 0) {
        p.E[u] = (EstT)t;
        p.N[u] = (EstT)t;
      }
      __syncthreads();
      uint32_t f = 0;
      for (uint32_t j = tid; j < deg; j += TB) {  // fastk.cpp:47-53
        const uint32_t v = j == tid ? v0 : p.adj[ob + j];
        const uint32_t ev = j == tid ? (v0 == u ? t : e0) : (uint32_t)p.E[v];
        const bool fire = p.ext ? (t < ev && cap >= ev) : ev > t;  // fastk.cpp:22-24
        if (!fire) continue;
        ++f;
        if (act[v] == 0) {  // a simple row holds v once: no race
          act[v] = 1;
          const uint32_t pos = atomicAdd(&s_m, 1u);
          p.list[pos] = v;
          if (pos < KEYCAP) {  // mirror (est does not change until v is popped)
            s_id[pos] = v;
            s_key[pos] = (unsigned long long)ev << 32 | p.perm[v];
          }
        }
      }
      f = __reduce_add_sync(FULLM, f);
      if ((tid & 31) == 0 && f) atomicAdd(&s_fires, f);
      __syncthreads();
      fires += s_fires;
    }
    __syncthreads();
  }
  if (tid == 0) {
    p.tc[TAIL_POPS] = m0 + fires;  // every pushed entry is popped once
    p.tc[TAIL_EVALS] = pops_done;
    p.tc[TAIL_FIRES] = fires;
    p.tc[TAIL_DROPS] = drops;
    p.tc[TAIL_ESCAN] = escan;
    p.tc[TAIL_RAN] = 1;
  }
}

template <typename OffT, typename EstT>
cudaError_t launch_tail_t(const SolveBuffers& b, const uint32_t* perm, int ext, int force_flags,
                          int num_sms, cudaStream_t s) {
  TP<OffT, EstT> p{};
  p.off = static_cast<const OffT*>(b.off);
  p.adj = b.adj;
  p.E = static_cast<EstT*>(b.est[0]);
  p.N = static_cast<EstT*>(b.est[1]);
  p.perm = perm;
  p.flag[0] = b.flag[0];
  p.flag[1] = b.flag[1];
  p.list = b.queue2;
  p.ts = reinterpret_cast<TailState*>(b.tailc + TAIL_SCRATCH);
  p.tc = b.tailc;
  p.status = b.status;
  p.n_nz = b.n_nz;
  p.ext = ext;
  p.force_flags = force_flags;
  cudaError_t e = cudaMemsetAsync(p.ts, 0, sizeof(TailState), s);
  if (e != cudaSuccess) return e;
  tail_list_kernel<OffT, EstT><<<num_sms * 4, 256, 0, s>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const size_t smem = TAIL_BINS * sizeof(uint32_t) + KEYCAP * (sizeof(unsigned long long) + sizeof(uint32_t));
  e = cudaFuncSetAttribute(tail_kernel<OffT, EstT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
  if (e != cudaSuccess) return e;
  tail_kernel<OffT, EstT><<<1, TB, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_tail(const SolveBuffers& b, const uint32_t* perm, bool est16, bool off64,
                        int ext, int force_flags, int num_sms, cudaStream_t s) {
  if (est16)
    return off64 ? launch_tail_t<uint64_t, uint16_t>(b, perm, ext, force_flags, num_sms, s)
                 : launch_tail_t<uint32_t, uint16_t>(b, perm, ext, force_flags, num_sms, s);
  return off64 ? launch_tail_t<uint64_t, uint32_t>(b, perm, ext, force_flags, num_sms, s)
               : launch_tail_t<uint32_t, uint32_t>(b, perm, ext, force_flags, num_sms, s);
}

}  // namespace kcb
