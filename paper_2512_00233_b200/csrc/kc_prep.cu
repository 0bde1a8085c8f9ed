// kc_prep.cu — on-device layout of the uploaded CSR for the solver.
//
// Input: the reference Graph's CSR (uint64 offsets, uint32 neighbours,
// include/kcore/graph.hpp:72-73) already in device memory.
// Output (owned by kc_graph):
//   * vertices relabelled by descending degree (stable, so equal-degree runs
//     keep their original order): degree classes become id ranges, the most
//     gathered estimates become a dense prefix that fits shared memory, and
//     isolated vertices (coreness 0, never evaluated) drop off the end;
//   * offsets narrowed to uint32 whenever nnz < 2^32 (uint64 otherwise);
//   * neighbours rewritten to new ids, each row sorted ascending so a warp's
//     gathers walk est[] in increasing address order (5-20% faster solves;
//     skipped for one-shot solves, where the sort costs more than it saves);
//   * perm[new] = old for the permute-back at download.
#include <cub/cub.cuh>
#include <cstdint>

#include "kc_internal.h"

#ifndef KC_PREP_SORT
#define KC_PREP_SORT 1
#endif

namespace kcb {
namespace {

// Degrees, and the CSR's structural checks the reference's Graph guarantees
// by construction (graph.hpp:37-75): offsets[0] == 0, non-decreasing,
// offsets[n] == nnz, every degree < 2^32.  A violation sets *bad (the
// upload then fails with KC_ERR_INVALID_ARGUMENT instead of indexing out of
// bounds in the layout or the solver).
__global__ void degrees_kernel(const uint64_t* __restrict__ off, uint32_t n, uint64_t nnz,
                               uint32_t* __restrict__ deg, uint32_t* __restrict__ iota,
                               uint32_t* bad) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    const uint64_t a = off[u], b = off[u + 1];
    if (b < a || b - a > 0xffffffffull || (u == 0 && a != 0) || (u == n - 1 && b != nnz))
      atomicOr(bad, 1u);
    deg[u] = b >= a ? (uint32_t)(b - a) : 0u;
    iota[u] = u;
  }
}

// dcut[x] = #{new ids of degree >= x} from the degrees sorted descending
// (binary search per x, all x in parallel); dcut[0] = all, dcut[max + 1] = 0.
__global__ void degcut_kernel(const uint32_t* __restrict__ sdeg, uint32_t n_nz, uint32_t max_deg,
                              uint32_t* __restrict__ dcut) {
  const uint32_t gs = gridDim.x * blockDim.x;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x <= max_deg + 1; x += gs) {
    if (x == 0) {
      dcut[0] = 0xffffffffu;
      continue;
    }
    uint32_t lo = 0, hi = n_nz;  // first w with sdeg[w] < x
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (sdeg[mid] >= x) lo = mid + 1; else hi = mid;
    }
    dcut[x] = lo;
  }
}

__global__ void inverse_kernel(const uint32_t* __restrict__ perm, uint32_t n,
                               uint32_t* __restrict__ inv) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    inv[perm[i]] = i;
}

// Boundaries on the descending degree sequence: out[0] = H (h-index of the
// degree sequence), out[1..4] = #vertices with degree > {8192, 1024, 64, 8},
// out[5] = #vertices with degree > 0 (n_nz), out[6] = maximum degree.  Thresholds: kc_internal.h.
__global__ void bounds_kernel(const uint32_t* __restrict__ sdeg, uint32_t n, uint32_t* out) {
  const uint32_t k = threadIdx.x;
  if (k == 6) out[6] = n ? sdeg[0] : 0u;  // maximum degree
  if (k > 5) return;
  if (k == 0) {  // largest h with sdeg[h-1] >= h
    uint32_t lo = 0, hi = n;  // answer in [lo, hi]
    while (lo < hi) {
      uint32_t mid = lo + (hi - lo + 1) / 2;
      if (sdeg[mid - 1] >= mid) lo = mid; else hi = mid - 1;
    }
    out[0] = lo;
    return;
  }
  const uint32_t thr[6] = {0, DEG_BIG_MAX, DEG_WARP_MAX, DEG_SUB_MAX, DEG_THREAD_MAX, 0};
  const uint32_t t = thr[k];
  uint32_t lo = 0, hi = n;  // count of sdeg[i] > t (prefix, sdeg descending)
  while (lo < hi) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (sdeg[mid] > t) lo = mid + 1; else hi = mid;
  }
  out[k] = lo;
}

template <typename OffT>
__global__ void narrow_offsets_kernel(const uint64_t* __restrict__ src, uint32_t m,
                                      OffT* __restrict__ dst) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    dst[i] = (OffT)src[i];
}

// Rewrite row i (old row perm[i]) into new ids.  Rows are split into
// 1024-entry chunks so hub rows spread over many warps.
template <typename OffT>
__global__ void relabel_rows_kernel(const uint64_t* __restrict__ old_off,
                                    const uint32_t* __restrict__ old_adj,
                                    const uint32_t* __restrict__ perm,
                                    const uint32_t* __restrict__ inv,
                                    const uint64_t* __restrict__ chunk_base,  // per row, scan of chunks
                                    uint32_t n_nz, const OffT* __restrict__ new_off,
                                    uint32_t* __restrict__ new_adj, uint64_t total_chunks,
                                    uint32_t o_lo, uint32_t o_hi, uint32_t n, uint32_t* bad) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  for (uint64_t c = w0; c < total_chunks; c += nw) {
    // row containing chunk c: largest i with chunk_base[i] <= c
    uint32_t lo = 0, hi = n_nz;
    while (hi - lo > 1) {
      uint32_t mid = lo + (hi - lo) / 2;
      if (chunk_base[mid] <= c) lo = mid; else hi = mid;
    }
    const uint32_t i = lo;
    const uint32_t o = perm[i];
    if (o < o_lo || o >= o_hi) continue;  // pipelined upload: its bytes are not here yet
    const uint64_t k0 = (c - chunk_base[i]) * 1024;
    const uint64_t deg = (uint64_t)(new_off[i + 1] - new_off[i]);
    const uint64_t k1 = k0 + 1024 < deg ? k0 + 1024 : deg;
    const uint32_t* src = old_adj + old_off[o];
    uint32_t* dst = new_adj + new_off[i];
    for (uint64_t k = k0 + lane; k < k1; k += 32) {
      const uint32_t x = src[k];
      if (x >= n) atomicOr(bad, 2u);  // neighbour id out of range
      dst[k] = x < n ? inv[x] : 0u;
    }
  }
}

// Rows of degree <= 64 (new ids [first, n_nz), the tail of the degree-sorted
// order): 8-lane tile per row, up to 8 entries per lane — no per-row search.
template <typename OffT>
__global__ void relabel_small_rows_kernel(const uint64_t* __restrict__ old_off,
                                          const uint32_t* __restrict__ old_adj,
                                          const uint32_t* __restrict__ perm,
                                          const uint32_t* __restrict__ inv, uint32_t first,
                                          uint32_t n_nz, const OffT* __restrict__ new_off,
                                          uint32_t* __restrict__ new_adj, uint32_t o_lo,
                                          uint32_t o_hi, uint32_t n, uint32_t* bad) {
  const uint32_t k = threadIdx.x & 7;
  const uint64_t t0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 3;
  const uint64_t nt = (gridDim.x * (uint64_t)blockDim.x) >> 3;
  for (uint64_t i = first + t0; i < n_nz; i += nt) {
    const uint32_t o = perm[i];
    if (o < o_lo || o >= o_hi) continue;  // pipelined upload: not here yet
    const uint64_t b = (uint64_t)new_off[i];
    const uint32_t deg = (uint32_t)((uint64_t)new_off[i + 1] - b);
    const uint32_t* src = old_adj + old_off[o];
    uint32_t v[DEG_SUB_MAX / 8];
#pragma unroll
    for (int j = 0; j < (int)(DEG_SUB_MAX / 8); ++j) {
      const uint32_t e = k + 8u * j;
      v[j] = e < deg ? src[e] : 0u;
    }
#pragma unroll
    for (int j = 0; j < (int)(DEG_SUB_MAX / 8); ++j) {
      const uint32_t e = k + 8u * j;
      if (e < deg) {
        if (v[j] >= n) atomicOr(bad, 2u);  // neighbour id out of range
        new_adj[b + e] = v[j] < n ? inv[v[j]] : 0u;
      }
    }
  }
}

template <typename OffT>
__global__ void chunk_count_kernel(const OffT* __restrict__ new_off, uint32_t n_nz,
                                   uint64_t* __restrict__ chunks) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_nz; i += gridDim.x * blockDim.x)
    chunks[i] = ((uint64_t)(new_off[i + 1] - new_off[i]) + 1023) / 1024;
}


// ---------------------------------------------------------------------------
// Relabel + sort fused (sorted layouts).  The solver's degree cuts need every
// row ascending in the new ids (= non-increasing neighbour degree).  A row is
// sorted on chip while it is being rewritten, so the sorted layout costs one
// pass over the adjacency — per upload chunk, i.e. under the host-to-device
// copy of the next chunk — instead of a segmented sort of the finished array:
//   rows <= 64        8-lane tile, 8 keys per lane, bitonic network (shuffles)
//   rows <= 8,192     one CTA per row, cub::BlockRadixSort in shared memory,
//                     seven capacities (128 .. 8,192 keys)
//   rows  > 8,192     (HUGE class) relabelled into a side buffer, then one
//                     cub::DeviceSegmentedRadixSort per chunk over its hubs
// Ids are assigned by descending degree, so each tier is an id range.
// ---------------------------------------------------------------------------

// out[k] = #{i : sdeg[i] > thr[k]} on the descending degree sequence.
constexpr int N_TIERS = 8;
struct TierThr { uint32_t t[N_TIERS]; };
__global__ void tier_bounds_kernel(const uint32_t* __restrict__ sdeg, uint32_t n, TierThr thr,
                                   uint32_t* __restrict__ out) {
  const uint32_t k = threadIdx.x;
  if (k >= N_TIERS) return;
  const uint32_t t = thr.t[k];
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (sdeg[mid] > t) lo = mid + 1; else hi = mid;
  }
  out[k] = lo;
}

// One step of the bitonic network over the 64 keys of an 8-lane tile, key
// index e = 8 * r + lane8 (register r of lane lane8: the coalesced order the
// row is read and written in).  K: size of the runs being merged, J: stride.
template <int K, int J>
__device__ __forceinline__ void bitonic_step(uint32_t (&v)[8], uint32_t lane8, unsigned mask,
                                             int nreg) {
  if constexpr (J < 8) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r >= nreg) break;
      const uint32_t other = __shfl_xor_sync(mask, v[r], J);
      const bool lower = (lane8 & J) == 0;
      const bool asc = ((8u * r + lane8) & K) == 0;
      const uint32_t mn = v[r] < other ? v[r] : other, mx = v[r] < other ? other : v[r];
      v[r] = lower == asc ? mn : mx;
    }
  } else {
    constexpr int RJ = J / 8;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if ((r & RJ) != 0 || (r | RJ) >= nreg) continue;
      const bool asc = ((8 * r) & K) == 0;
      const uint32_t a = v[r], b = v[r | RJ];
      const uint32_t mn = a < b ? a : b, mx = a < b ? b : a;
      v[r] = asc ? mn : mx;
      v[r | RJ] = asc ? mx : mn;
    }
  }
}

// Sorts the first 8 * nreg keys of the tile ascending (nreg = 1, 2, 4 or 8,
// tile-uniform; the keys beyond are padding).
__device__ __forceinline__ void tile_sort64(uint32_t (&v)[8], uint32_t lane8, unsigned mask,
                                            int nreg) {
  bitonic_step<2, 1>(v, lane8, mask, nreg);
  bitonic_step<4, 2>(v, lane8, mask, nreg);
  bitonic_step<4, 1>(v, lane8, mask, nreg);
  // runs of 8: the last merge of an 8-key sort must ascend everywhere, which
  // (e & 8) == 0 gives for r = 0; wider sorts alternate by register
  bitonic_step<8, 4>(v, lane8, mask, nreg);
  bitonic_step<8, 2>(v, lane8, mask, nreg);
  bitonic_step<8, 1>(v, lane8, mask, nreg);
  if (nreg >= 2) {
    bitonic_step<16, 8>(v, lane8, mask, nreg);
    bitonic_step<16, 4>(v, lane8, mask, nreg);
    bitonic_step<16, 2>(v, lane8, mask, nreg);
    bitonic_step<16, 1>(v, lane8, mask, nreg);
  }
  if (nreg >= 4) {
    bitonic_step<32, 16>(v, lane8, mask, nreg);
    bitonic_step<32, 8>(v, lane8, mask, nreg);
    bitonic_step<32, 4>(v, lane8, mask, nreg);
    bitonic_step<32, 2>(v, lane8, mask, nreg);
    bitonic_step<32, 1>(v, lane8, mask, nreg);
  }
  if (nreg >= 8) {
    bitonic_step<64, 32>(v, lane8, mask, nreg);
    bitonic_step<64, 16>(v, lane8, mask, nreg);
    bitonic_step<64, 8>(v, lane8, mask, nreg);
    bitonic_step<64, 4>(v, lane8, mask, nreg);
    bitonic_step<64, 2>(v, lane8, mask, nreg);
    bitonic_step<64, 1>(v, lane8, mask, nreg);
  }
}

// The rows [first, last) whose caller id lies in [o_lo, o_hi), 32 at a time:
// a warp checks 32 candidates per step (one coalesced perm[] load) and queues
// the hits in shared memory (wq: 2 x 64 words per warp — row, caller id);
// drain(count) is called with wq[0 .. count) filled, count = 32 except for
// the last call.  Rows of other chunks cost 1/32 of a warp step each.
template <typename F>
__device__ __forceinline__ void for_chunk_rows(const uint32_t* __restrict__ perm, uint32_t first,
                                               uint32_t last, uint32_t o_lo, uint32_t o_hi,
                                               uint32_t* wq, F&& drain) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  uint32_t qn = 0;  // warp-uniform
  for (uint64_t base = first + w0 * 32; base < last; base += nw * 32) {
    const uint64_t cand = base + lane;
    uint32_t o = 0;
    bool in = false;
    if (cand < last) {
      o = perm[cand];
      in = o >= o_lo && o < o_hi;
    }
    const unsigned m = __ballot_sync(0xffffffffu, in);
    if (in) {
      const uint32_t at = qn + __popc(m & ((1u << lane) - 1u));
      wq[at] = (uint32_t)cand;
      wq[64 + at] = o;
    }
    qn += __popc(m);
    __syncwarp();
    if (qn >= 32) {
      drain(32u);
      __syncwarp();
      const uint32_t r = wq[32 + lane], ro = wq[96 + lane];
      __syncwarp();
      wq[lane] = r;
      wq[64 + lane] = ro;
      qn -= 32;
      __syncwarp();
    }
  }
  if (qn) drain(qn);
}

// Rows of degree 9 .. 64 of one upload chunk, relabelled and sorted: 8-lane
// tile per row, four rows per warp step.
template <typename OffT>
__global__ void __launch_bounds__(256)
    relabel_sort_sub_rows_kernel(const uint64_t* __restrict__ old_off, const uint32_t* __restrict__ old_adj,
                                 const uint32_t* __restrict__ perm, const uint32_t* __restrict__ inv,
                                 uint32_t first, uint32_t last, const OffT* __restrict__ new_off,
                                 uint32_t* __restrict__ new_adj, uint32_t o_lo, uint32_t o_hi,
                                 uint32_t n, uint32_t* bad) {
  __shared__ uint32_t s_wq[8][128];
  uint32_t* wq = s_wq[threadIdx.x >> 5];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t k = lane & 7, tile = lane >> 3;
  const unsigned tmask = 0xffu << (lane & 24);
  for_chunk_rows(perm, first, last, o_lo, o_hi, wq, [&](uint32_t count) {
    for (uint32_t q = tile; q < count; q += 4) {
      const uint32_t i = wq[q];
      const uint64_t b = (uint64_t)new_off[i];
      const uint32_t deg = (uint32_t)((uint64_t)new_off[i + 1] - b);
      const uint32_t* src = old_adj + old_off[wq[64 + q]];
      const int nreg = deg <= 8 ? 1 : deg <= 16 ? 2 : deg <= 32 ? 4 : 8;
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t e = k + 8u * j;
        v[j] = e < deg ? src[e] : 0xffffffffu;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t e = k + 8u * j;
        if (e < deg) {
          if (v[j] >= n) atomicOr(bad, 2u);  // neighbour id out of range
          v[j] = v[j] < n ? inv[v[j]] : 0u;
        }
      }
      tile_sort64(v, k, tmask, nreg);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t e = k + 8u * j;
        if (e < deg) new_adj[b + e] = v[j];
      }
    }
  });
}

// Rows of degree <= 8 of one upload chunk, relabelled and sorted: a lane per
// row, the row in registers, a 19-exchange sorting network.
__device__ __forceinline__ void cex(uint32_t& a, uint32_t& b) {
  const uint32_t mn = a < b ? a : b, mx = a < b ? b : a;
  a = mn;
  b = mx;
}
template <typename OffT>
__global__ void __launch_bounds__(256)
    relabel_sort_thread_rows_kernel(const uint64_t* __restrict__ old_off, const uint32_t* __restrict__ old_adj,
                                    const uint32_t* __restrict__ perm, const uint32_t* __restrict__ inv,
                                    uint32_t first, uint32_t last, const OffT* __restrict__ new_off,
                                    uint32_t* __restrict__ new_adj, uint32_t o_lo, uint32_t o_hi,
                                    uint32_t n, uint32_t* bad) {
  __shared__ uint32_t s_wq[8][128];
  uint32_t* wq = s_wq[threadIdx.x >> 5];
  const uint32_t lane = threadIdx.x & 31;
  for_chunk_rows(perm, first, last, o_lo, o_hi, wq, [&](uint32_t count) {
    if (lane >= count) return;
    const uint32_t i = wq[lane];
    const uint64_t b = (uint64_t)new_off[i];
    const uint32_t deg = (uint32_t)((uint64_t)new_off[i + 1] - b);
    const uint32_t* src = old_adj + old_off[wq[64 + lane]];
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (uint32_t)j < deg ? src[j] : 0xffffffffu;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if ((uint32_t)j < deg) {
        if (v[j] >= n) atomicOr(bad, 2u);  // neighbour id out of range
        v[j] = v[j] < n ? inv[v[j]] : 0u;
      }
    // optimal 8-input network (19 exchanges, depth 6)
    cex(v[0], v[2]); cex(v[1], v[3]); cex(v[4], v[6]); cex(v[5], v[7]);
    cex(v[0], v[4]); cex(v[1], v[5]); cex(v[2], v[6]); cex(v[3], v[7]);
    cex(v[0], v[1]); cex(v[2], v[3]); cex(v[4], v[5]); cex(v[6], v[7]);
    cex(v[2], v[4]); cex(v[3], v[5]);
    cex(v[1], v[4]); cex(v[3], v[6]);
    cex(v[1], v[2]); cex(v[3], v[4]); cex(v[5], v[6]);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if ((uint32_t)j < deg) new_adj[b + j] = v[j];
  });
}

// The rows of one upload chunk, per block-sort tier: list[tb[k] - tb[0] + j] =
// the j-th row of tier k (rows [tb[k], tb[k + 1])) whose caller id lies in
// [o_lo, o_hi), cnt[k] their number.  The sort kernels walk these lists, so
// every CTA has work however few rows a tier has and skipped rows cost
// nothing.  One warp-aggregated atomic per tier present in a warp.
struct TierTab { uint32_t b[N_TIERS]; };
__global__ void chunk_rows_kernel(const uint32_t* __restrict__ perm, TierTab tb, uint32_t o_lo,
                                  uint32_t o_hi, uint32_t* __restrict__ list,
                                  uint32_t* __restrict__ cnt) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lo = tb.b[0], hi = tb.b[N_TIERS - 1];
  const uint32_t span = (hi - lo + 31) & ~31u;  // whole warps stay in the loop
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < span; k += gridDim.x * blockDim.x) {
    const uint32_t i = lo + k;
    bool in = false;
    int tier = -1;
    if (i < hi) {
      const uint32_t o = perm[i];
      in = o >= o_lo && o < o_hi;
#pragma unroll
      for (int t = 0; t < N_TIERS - 1; ++t)
        if (i >= tb.b[t] && i < tb.b[t + 1]) tier = t;
    }
    if (!in) tier = -1;
    for (int t = 0; t < N_TIERS - 1; ++t) {
      const unsigned m = __ballot_sync(0xffffffffu, tier == t);
      if (!m) continue;
      uint32_t base = 0;
      if (lane == (uint32_t)(__ffs(m) - 1)) base = atomicAdd(&cnt[t], (uint32_t)__popc(m));
      base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
      if (tier == t) list[tb.b[t] - lo + base + __popc(m & ((1u << lane) - 1u))] = i;
    }
  }
}

// Bitonic network over the keys of a CTA of NW warps, NREG keys per lane,
// key index e = w * 1024 + r * 32 + lane (register r of lane `lane` of warp
// w: the coalesced order the row is read and written in; NW > 1 only with
// NREG = 32).  Merge stage K, stride J: strides below 32 are warp shuffles
// (one loop body per K, J at run time), strides 32 .. 512 compare registers
// of one lane (static indices), strides >= 1024 go through shared memory.
template <int NREG, int K, int J>
__device__ __forceinline__ void reg_stages(uint32_t (&v)[NREG], uint32_t w) {
  if constexpr (J >= 32) {
    constexpr int RJ = J / 32;
#pragma unroll
    for (int r = 0; r < NREG; ++r) {
      if ((r & RJ) != 0) continue;
      const bool asc = (((w << 10) | (uint32_t)(r << 5)) & (uint32_t)K) == 0;
      const uint32_t a = v[r], b = v[r | RJ];
      const uint32_t mn = a < b ? a : b, mx = a < b ? b : a;
      v[r] = asc ? mn : mx;
      v[r | RJ] = asc ? mx : mn;
    }
    reg_stages<NREG, K, J / 2>(v, w);
  }
}

template <int NREG, int K>
__device__ __forceinline__ void warp_merge(uint32_t (&v)[NREG], uint32_t lane, uint32_t w) {
  constexpr int JTOP = (K / 2 < 16 * NREG) ? K / 2 : 16 * NREG;
  reg_stages<NREG, K, JTOP>(v, w);
#pragma unroll 1
  for (int J = JTOP < 16 ? JTOP : 16; J >= 1; J >>= 1) {
    const bool lower = (lane & (uint32_t)J) == 0;
#pragma unroll
    for (int r = 0; r < NREG; ++r) {
      const uint32_t other = __shfl_xor_sync(0xffffffffu, v[r], J);
      const bool asc = (((w << 10) | (uint32_t)(r << 5) | lane) & (uint32_t)K) == 0;
      const uint32_t mn = v[r] < other ? v[r] : other, mx = v[r] < other ? other : v[r];
      v[r] = lower == asc ? mn : mx;
    }
  }
}

template <int NREG, int K>
__device__ __forceinline__ void warp_sort_upto(uint32_t (&v)[NREG], uint32_t lane, uint32_t w) {
  if constexpr (K > 2) warp_sort_upto<NREG, K / 2>(v, lane, w);
  warp_merge<NREG, K>(v, lane, w);
}

// Cross-warp strides of merge stage K (J = K / 2 .. 1024) through `xch`
// (NW * 1024 keys), then the in-warp part.
template <int NW, int K>
__device__ __forceinline__ void cta_merge(uint32_t (&v)[32], uint32_t lane, uint32_t w,
                                          uint32_t* xch) {
  const bool asc = ((w << 10) & (uint32_t)K) == 0;
#pragma unroll 1
  for (int J = K / 2; J >= 1024; J >>= 1) {
#pragma unroll
    for (int r = 0; r < 32; ++r) xch[(w << 10) | (r << 5) | lane] = v[r];
    __syncthreads();
    const uint32_t pw = w ^ (uint32_t)(J >> 10);
    const bool lower = (w & (uint32_t)(J >> 10)) == 0;
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const uint32_t other = xch[(pw << 10) | (r << 5) | lane];
      const uint32_t mn = v[r] < other ? v[r] : other, mx = v[r] < other ? other : v[r];
      v[r] = lower == asc ? mn : mx;
    }
    __syncthreads();
  }
  warp_merge<32, K>(v, lane, w);
}

template <int NW, int K>
__device__ __forceinline__ void cta_sort_upto(uint32_t (&v)[32], uint32_t lane, uint32_t w,
                                              uint32_t* xch) {
  if constexpr (K > 2048) cta_sort_upto<NW, K / 2>(v, lane, w, xch);
  cta_merge<NW, K>(v, lane, w, xch);
}

// Rows of one tier (capacity NW * NREG * 32 keys) of one upload chunk,
// relabelled and sorted ascending.  NW == 1: a warp per row, four rows per
// CTA, no barriers.  NW > 1: a CTA per row.  The 0xffffffff padding sorts
// last (ids are < n <= 2^32 - 1).
template <typename OffT, int NW, int NREG>
__global__ void __launch_bounds__(NW == 1 ? 128 : NW * 32)
    relabel_sort_rows_kernel(const uint64_t* __restrict__ old_off, const uint32_t* __restrict__ old_adj,
                             const uint32_t* __restrict__ perm, const uint32_t* __restrict__ inv,
                             const OffT* __restrict__ new_off, uint32_t* __restrict__ new_adj,
                             const uint32_t* __restrict__ list, const uint32_t* __restrict__ cnt_ptr,
                             uint32_t n, uint32_t* bad) {
  static_assert(NW == 1 || NREG == 32, "multi-warp tiers hold 1,024 keys per warp");
  __shared__ uint32_t xch[NW > 1 ? NW * 1024 : 1];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w = NW == 1 ? 0u : threadIdx.x >> 5;
  const uint32_t cnt = *cnt_ptr;
  const uint32_t unit = NW == 1 ? (blockIdx.x * blockDim.x + threadIdx.x) >> 5 : blockIdx.x;
  const uint32_t units = NW == 1 ? (gridDim.x * blockDim.x) >> 5 : gridDim.x;
  for (uint32_t q = unit; q < cnt; q += units) {
    const uint32_t i = list[q];
    const uint64_t b = (uint64_t)new_off[i];
    const uint32_t deg = (uint32_t)((uint64_t)new_off[i + 1] - b);
    const uint32_t* src = old_adj + old_off[perm[i]];
    uint32_t v[NREG];
#pragma unroll
    for (int r = 0; r < NREG; ++r) {
      const uint32_t e = (w << 10) | (uint32_t)(r << 5) | lane;
      v[r] = e < deg ? src[e] : 0xffffffffu;
    }
#pragma unroll
    for (int r = 0; r < NREG; ++r) {
      const uint32_t e = (w << 10) | (uint32_t)(r << 5) | lane;
      if (e < deg) {
        if (v[r] >= n) atomicOr(bad, 2u);  // neighbour id out of range
        v[r] = v[r] < n ? inv[v[r]] : 0u;
      }
    }
    warp_sort_upto<NREG, 32 * NREG>(v, lane, w);
    if constexpr (NW > 1) cta_sort_upto<NW, NW * 1024>(v, lane, w, xch);
#pragma unroll
    for (int r = 0; r < NREG; ++r) {
      const uint32_t e = (w << 10) | (uint32_t)(r << 5) | lane;
      if (e < deg) new_adj[b + e] = v[r];
    }
  }
}

// Segment bounds of the HUGE rows for the segmented radix sort of one upload
// chunk: a hub outside the chunk is an empty segment.
template <typename OffT>
struct SegBegin {
  const OffT* off;
  __host__ __device__ int operator()(int i) const { return (int)off[i]; }
};
template <typename OffT>
struct SegEnd {
  const OffT* off;
  const uint32_t* perm;
  uint32_t o_lo, o_hi;
  __host__ __device__ int operator()(int i) const {
    const uint32_t o = perm[i];
    return (int)((o >= o_lo && o < o_hi) ? off[i + 1] : off[i]);
  }
};

}  // namespace

#define PREP_CK(x)                         \
  do {                                     \
    cudaError_t e_ = (x);                  \
    if (e_ != cudaSuccess) {               \
      err = e_;                            \
      goto done;                           \
    }                                      \
  } while (0)

// The sort tiers and the small rows of one upload chunk.  tb[k] = #rows of
// degree > {8192, 4096, 2048, 1024, 512, 256, 128, 64}[k]: tier k sorts the
// rows [tb[k], tb[k + 1]) listed for this chunk (chunk_rows_kernel).
template <typename OffT, int NW, int NREG>
static cudaError_t sort_tier(const uint64_t* off, const uint32_t* adj, const uint32_t* perm,
                             const uint32_t* inv, const OffT* new_off, uint32_t* new_adj,
                             const uint32_t* tb, int k, const uint32_t* list, const uint32_t* cnt,
                             uint32_t n, uint32_t* bad, cudaStream_t s) {
  if (tb[k + 1] <= tb[k]) return cudaSuccess;
  const uint32_t rows = tb[k + 1] - tb[k];
  uint32_t grid;
  if (NW == 1) {
    const uint32_t want = (rows + 3) / 4, cap = 148u * 12u;
    grid = want < cap ? want : cap;
  } else {
    const uint32_t cap = 148u * (16u / NW);
    grid = rows < cap ? rows : cap;
  }
  relabel_sort_rows_kernel<OffT, NW, NREG><<<grid, NW == 1 ? 128 : NW * 32, 0, s>>>(
      off, adj, perm, inv, new_off, new_adj, list + (tb[k] - tb[0]), cnt + k, n, bad);
  return cudaGetLastError();
}

template <typename OffT>
static cudaError_t sort_tiers(const uint64_t* off, const uint32_t* adj, const uint32_t* perm,
                              const uint32_t* inv, const OffT* new_off, uint32_t* new_adj,
                              const uint32_t* tb, uint32_t n_sub, uint32_t n_nz, uint32_t o_lo,
                              uint32_t o_hi, uint32_t n, uint32_t* list, uint32_t* cnt,
                              uint32_t* bad, cudaStream_t s) {
  cudaError_t e;
  if (tb[N_TIERS - 1] > tb[0]) {
    TierTab t;
    for (int k = 0; k < N_TIERS; ++k) t.b[k] = tb[k];
    const uint32_t rows = tb[N_TIERS - 1] - tb[0];
    const uint32_t want = (rows + 255) / 256;
    chunk_rows_kernel<<<want < 148u * 8u ? want : 148u * 8u, 256, 0, s>>>(perm, t, o_lo, o_hi, list,
                                                                          cnt);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
#define KC_TIER(K, W, R)                                                                          \
  if ((e = sort_tier<OffT, W, R>(off, adj, perm, inv, new_off, new_adj, tb, K, list, cnt, n, bad, \
                                 s)) != cudaSuccess)                                              \
    return e;
  KC_TIER(0, 8, 32)  // 4,097 .. 8,192: longest rows first (they finish last)
  KC_TIER(1, 4, 32)  // 2,049 .. 4,096
  KC_TIER(2, 2, 32)  // 1,025 .. 2,048
  KC_TIER(3, 1, 32)  //   513 .. 1,024
  KC_TIER(4, 1, 16)  //   257 .. 512
  KC_TIER(5, 1, 8)   //   129 .. 256
  KC_TIER(6, 1, 4)   //    65 .. 128
#undef KC_TIER
  // SUB rows [tb[7], n_sub), THREAD rows [n_sub, n_nz)
  if (n_sub > tb[7]) {
    relabel_sort_sub_rows_kernel<OffT><<<148 * 8, 256, 0, s>>>(off, adj, perm, inv, tb[7], n_sub,
                                                               new_off, new_adj, o_lo, o_hi, n, bad);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (n_nz > n_sub) {
    relabel_sort_thread_rows_kernel<OffT><<<148 * 8, 256, 0, s>>>(off, adj, perm, inv, n_sub, n_nz,
                                                                  new_off, new_adj, o_lo, o_hi, n, bad);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <typename T>
static cudaError_t dalloc(T** p, size_t count, cudaStream_t s) {
  return dmalloc_n(p, count, s);
}

// Relabel + narrow + sort rows.  `off`/`adj` are device pointers to the
// uploaded reference CSR (not modified).
cudaError_t prep_layout(const uint64_t* off, const uint32_t* adj, uint32_t n, uint64_t nnz,
                        bool force_off64, bool sort_rows, cudaStream_t s, PrepOut* out,
                        const AdjFeed* feed) {
  cudaError_t err = cudaSuccess;
  uint32_t *deg = nullptr, *iota = nullptr, *sdeg = nullptr, *perm = nullptr, *inv = nullptr;
  uint32_t* bounds = nullptr;
  uint64_t* off64_tmp = nullptr;
  uint64_t* chunks = nullptr;
  void* new_off = nullptr;
  uint32_t* new_adj = nullptr;
  uint32_t* sort_tmp = nullptr;
  uint32_t* tiers = nullptr;
  uint32_t *tier_list = nullptr, *tier_cnt = nullptr;
  void* hub_tmp_store = nullptr;
  cudaStream_t hs = nullptr;  // sorted layouts: the hubs' relabel + sort, beside the tiers
  cudaEvent_t hev = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0, need = 0;
  uint32_t hb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  out->invalid = false;
  const bool off64 = force_off64 || nnz >= (1ull << 32);
  const int G = 148 * 8, B = 256;
  out->off = nullptr;
  out->adj = nullptr;
  out->perm = nullptr;
  out->dcut = nullptr;
  out->rows_sorted = false;
  uint32_t* dcut = nullptr;

  PREP_CK(dalloc(&deg, n, s));
  PREP_CK(dalloc(&iota, n, s));
  PREP_CK(dalloc(&sdeg, n, s));
  PREP_CK(dalloc(&perm, n, s));
  PREP_CK(dalloc(&inv, n, s));
  PREP_CK(dalloc(&bounds, 8, s));
  PREP_CK(cudaMemsetAsync(bounds, 0, 8 * sizeof(uint32_t), s));
  degrees_kernel<<<G, B, 0, s>>>(off, n, nnz, deg, iota, bounds + 7);
  PREP_CK(cudaGetLastError());
  // stable descending radix sort of (degree, id)
  PREP_CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, need, deg, sdeg, iota, perm, n, 0, 32, s));
  tmp_bytes = need;
  PREP_CK(dmalloc(&tmp, tmp_bytes, s));
  PREP_CK(cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, deg, sdeg, iota, perm, n, 0, 32, s));
  inverse_kernel<<<G, B, 0, s>>>(perm, n, inv);
  PREP_CK(cudaGetLastError());
  bounds_kernel<<<1, 32, 0, s>>>(sdeg, n, bounds);
  PREP_CK(cudaGetLastError());
  PREP_CK(cudaMemcpyAsync(hb, bounds, sizeof(hb), cudaMemcpyDeviceToHost, s));
  PREP_CK(cudaStreamSynchronize(s));
  if (hb[7]) {  // malformed offsets: nothing below may trust them
    out->invalid = true;
    goto done;
  }
  out->h_graph = hb[0];
  out->max_degree = hb[6];
  out->n_nz = hb[5];
  out->cls_begin[0] = 0;
  for (int c = 1; c <= 4; ++c) out->cls_begin[c] = hb[c];
  out->cls_begin[5] = hb[5];
  out->off64 = off64;
  {
    const uint32_t n_nz = out->n_nz;
    // new offsets: exclusive scan of sorted degrees (n_nz + 1 entries)
    PREP_CK(dalloc(&off64_tmp, (size_t)n_nz + 1, s));
    PREP_CK(cudaMemsetAsync(off64_tmp, 0, sizeof(uint64_t), s));
    {
      auto in = cub::TransformInputIterator<uint64_t, cub::CastOp<uint64_t>, const uint32_t*>(
          sdeg, cub::CastOp<uint64_t>());
      size_t nb = 0;
      PREP_CK(cub::DeviceScan::InclusiveSum(nullptr, nb, in, off64_tmp + 1, n_nz, s));
      if (nb > tmp_bytes) {
        dfree(tmp, s);
        tmp = nullptr;
        tmp_bytes = nb;
        PREP_CK(dmalloc(&tmp, tmp_bytes, s));
      }
      PREP_CK(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, in, off64_tmp + 1, n_nz, s));
    }
    if (off64) {
      new_off = off64_tmp;
      off64_tmp = nullptr;
    } else {
      PREP_CK(dmalloc(&new_off, ((size_t)n_nz + 1) * sizeof(uint32_t), s));
      narrow_offsets_kernel<uint32_t><<<G, B, 0, s>>>(off64_tmp, n_nz + 1, (uint32_t*)new_off);
      PREP_CK(cudaGetLastError());
    }
    PREP_CK(dalloc(&new_adj, nnz + ADJ_PAD, s));
    PREP_CK(cudaMemsetAsync(new_adj + nnz, 0, ADJ_PAD * sizeof(uint32_t), s));
    // Sorted layouts: every row is sorted while it is relabelled (see the
    // kernels above); the HUGE rows go through a side buffer and a segmented
    // radix sort.  Needs the hubs' entries to fit CUB's int item count.
    uint32_t tb[N_TIERS] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool fused_sort = KC_PREP_SORT && sort_rows && nnz > 0;
    const uint32_t n_huge = out->cls_begin[C_BIG];
    uint64_t hub_entries = 0;
    if (fused_sort) {
      // tb[k] = #rows of degree > {8192, 4096, 2048, 1024, 512, 256, 128, 64}
      TierThr thr{{8192u, 4096u, 2048u, 1024u, 512u, 256u, 128u, 64u}};
      static_assert(DEG_BIG_MAX == 8192 && DEG_SUB_MAX == 64, "tier table");
      PREP_CK(dalloc(&tiers, N_TIERS, s));
      tier_bounds_kernel<<<1, 32, 0, s>>>(sdeg, n_nz, thr, tiers);
      PREP_CK(cudaGetLastError());
      PREP_CK(cudaMemcpyAsync(tb, tiers, sizeof(tb), cudaMemcpyDeviceToHost, s));
      if (n_huge) {
        if (off64)
          PREP_CK(cudaMemcpyAsync(&hub_entries, (const uint64_t*)new_off + n_huge, sizeof(uint64_t),
                                  cudaMemcpyDeviceToHost, s));
        else
          PREP_CK(cudaMemcpyAsync(&hub_entries, (const uint32_t*)new_off + n_huge, sizeof(uint32_t),
                                  cudaMemcpyDeviceToHost, s));
      }
      PREP_CK(cudaStreamSynchronize(s));
      if (hub_entries >= (1ull << 31)) fused_sort = false;  // (not on one GPU's memory in practice)
    }
    // rows cut into 1024-entry chunks for warps (plain relabel): the rows of
    // degree > 64 (ids [0, n_big)) of an unsorted layout, the HUGE rows of a
    // sorted one; the other rows of an unsorted layout take the 8-lane kernel
    const uint32_t n_big = fused_sort ? n_huge : out->cls_begin[C_SUB];
    uint64_t total = 0;  // 1024-entry chunks of those rows
    PREP_CK(dalloc(&chunks, (size_t)n_big + 1, s));
    if (n_big) {
      if (off64)
        chunk_count_kernel<uint64_t><<<G, B, 0, s>>>((const uint64_t*)new_off, n_big, chunks);
      else
        chunk_count_kernel<uint32_t><<<G, B, 0, s>>>((const uint32_t*)new_off, n_big, chunks);
      PREP_CK(cudaGetLastError());
      size_t nb = 0;
      PREP_CK(cub::DeviceScan::ExclusiveSum(nullptr, nb, chunks, chunks, n_big + 1, s));
      if (nb > tmp_bytes) {
        dfree(tmp, s);
        tmp = nullptr;
        tmp_bytes = nb;
        PREP_CK(dmalloc(&tmp, tmp_bytes, s));
      }
      // chunks[n_big] must be 0 before the exclusive scan so the total lands there
      PREP_CK(cudaMemsetAsync(chunks + n_big, 0, sizeof(uint64_t), s));
      PREP_CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, chunks, chunks, n_big + 1, s));
      PREP_CK(cudaMemcpyAsync(&total, chunks + n_big, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      PREP_CK(cudaStreamSynchronize(s));
    }
    int end_bit = 1;  // ids < n <= 2^end_bit (the hubs' radix sort looks at these bits only)
    while (end_bit < 32 && (1ull << end_bit) < (uint64_t)n) ++end_bit;
    const int nparts = feed ? feed->k : 1;
    if (fused_sort && tb[N_TIERS - 1] > tb[0]) {
      // per-chunk row lists of the sort tiers (chunk_rows_kernel)
      PREP_CK(dalloc(&tier_list, (size_t)(tb[N_TIERS - 1] - tb[0]), s));
      PREP_CK(dalloc(&tier_cnt, (size_t)nparts * N_TIERS, s));
      PREP_CK(cudaMemsetAsync(tier_cnt, 0, (size_t)nparts * N_TIERS * sizeof(uint32_t), s));
    }
    // hubs: hub_buf[0] receives the relabelled rows, the segmented sort
    // ping-pongs between the two buffers; the first chunk shows where its
    // result lands, and the roles are swapped if that is not new_adj
    uint32_t* hub_buf[2] = {nullptr, new_adj};
    size_t hub_tmp_bytes = 0;
    bool hub_roles_known = false;
    if (fused_sort && n_huge) {
      PREP_CK(dalloc(&sort_tmp, (size_t)hub_entries + ADJ_PAD, s));
      hub_buf[0] = sort_tmp;
      cub::DoubleBuffer<uint32_t> db(hub_buf[0], hub_buf[1]);
      if (off64) {
        const uint64_t* o = (const uint64_t*)new_off;
        cub::TransformInputIterator<int, SegBegin<uint64_t>, cub::CountingInputIterator<int>> sb(
            cub::CountingInputIterator<int>(0), SegBegin<uint64_t>{o});
        cub::TransformInputIterator<int, SegEnd<uint64_t>, cub::CountingInputIterator<int>> se(
            cub::CountingInputIterator<int>(0), SegEnd<uint64_t>{o, perm, 0u, n});
        PREP_CK(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, hub_tmp_bytes, db, (int)hub_entries,
                                                        (int)n_huge, sb, se, 0, end_bit, s));
      } else {
        const uint32_t* o = (const uint32_t*)new_off;
        cub::TransformInputIterator<int, SegBegin<uint32_t>, cub::CountingInputIterator<int>> sb(
            cub::CountingInputIterator<int>(0), SegBegin<uint32_t>{o});
        cub::TransformInputIterator<int, SegEnd<uint32_t>, cub::CountingInputIterator<int>> se(
            cub::CountingInputIterator<int>(0), SegEnd<uint32_t>{o, perm, 0u, n});
        PREP_CK(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, hub_tmp_bytes, db, (int)hub_entries,
                                                        (int)n_huge, sb, se, 0, end_bit, s));
      }
      PREP_CK(dmalloc(&hub_tmp_store, hub_tmp_bytes ? hub_tmp_bytes : 1, s));
      // the hubs of a chunk are sorted one CTA each (a 500 K-entry hub takes
      // ~1 ms alone): on their own stream they run beside the tier kernels
      PREP_CK(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
      PREP_CK(cudaEventCreateWithFlags(&hev, cudaEventDisableTiming));
      PREP_CK(cudaEventRecord(hev, s));  // allocations and tables above are stream-ordered on s
      PREP_CK(cudaStreamWaitEvent(hs, hev, 0));
    }
    // relabel: all rows at once, or — pipelined upload — the rows of each
    // chunk of old ids as soon as its bytes have landed (event), so the
    // layout overlaps the host-to-device copy
    for (int c = 0; c < nparts; ++c) {
      const uint32_t o_lo = feed ? feed->old_lo[c] : 0u;
      const uint32_t o_hi = feed ? feed->old_lo[c + 1] : n;
      if (feed && feed->host_wait) feed->host_wait(feed->ctx, c);  // recorded by the stager
      if (feed) PREP_CK(cudaStreamWaitEvent(s, feed->ready[c], 0));
      if (!fused_sort) {
        if (n_nz > n_big) {
          if (off64)
            relabel_small_rows_kernel<uint64_t><<<G, B, 0, s>>>(off, adj, perm, inv, n_big, n_nz,
                                                                (const uint64_t*)new_off, new_adj,
                                                                o_lo, o_hi, n, bounds + 7);
          else
            relabel_small_rows_kernel<uint32_t><<<G, B, 0, s>>>(off, adj, perm, inv, n_big, n_nz,
                                                                (const uint32_t*)new_off, new_adj,
                                                                o_lo, o_hi, n, bounds + 7);
          PREP_CK(cudaGetLastError());
        }
      } else {
        // tiers of the block sort, longest rows first (they finish last)
        PREP_CK(off64 ? sort_tiers<uint64_t>(off, adj, perm, inv, (const uint64_t*)new_off, new_adj,
                                             tb, out->cls_begin[C_THREAD], n_nz, o_lo, o_hi, n, tier_list,
                                             tier_cnt + c * N_TIERS,
                                             bounds + 7, s)
                      : sort_tiers<uint32_t>(off, adj, perm, inv, (const uint32_t*)new_off, new_adj,
                                             tb, out->cls_begin[C_THREAD], n_nz, o_lo, o_hi, n, tier_list,
                                             tier_cnt + c * N_TIERS,
                                             bounds + 7, s));
      }
      if (n_big) {
        uint32_t* dst = fused_sort ? hub_buf[0] : new_adj;
        cudaStream_t rs = fused_sort ? hs : s;
        if (fused_sort && feed) PREP_CK(cudaStreamWaitEvent(hs, feed->ready[c], 0));
        if (off64)
          relabel_rows_kernel<uint64_t><<<G, B, 0, rs>>>(off, adj, perm, inv, chunks, n_big,
                                                        (const uint64_t*)new_off, dst, total,
                                                        o_lo, o_hi, n, bounds + 7);
        else
          relabel_rows_kernel<uint32_t><<<G, B, 0, rs>>>(off, adj, perm, inv, chunks, n_big,
                                                        (const uint32_t*)new_off, dst, total,
                                                        o_lo, o_hi, n, bounds + 7);
        PREP_CK(cudaGetLastError());
        if (fused_sort) {
          cub::DoubleBuffer<uint32_t> db(hub_buf[0], hub_buf[1]);
          size_t nb = hub_tmp_bytes;
          if (off64) {
            const uint64_t* o = (const uint64_t*)new_off;
            cub::TransformInputIterator<int, SegBegin<uint64_t>, cub::CountingInputIterator<int>> sb(
                cub::CountingInputIterator<int>(0), SegBegin<uint64_t>{o});
            cub::TransformInputIterator<int, SegEnd<uint64_t>, cub::CountingInputIterator<int>> se(
                cub::CountingInputIterator<int>(0), SegEnd<uint64_t>{o, perm, o_lo, o_hi});
            PREP_CK(cub::DeviceSegmentedRadixSort::SortKeys(hub_tmp_store, nb, db, (int)hub_entries,
                                                            (int)n_huge, sb, se, 0, end_bit, hs));
          } else {
            const uint32_t* o = (const uint32_t*)new_off;
            cub::TransformInputIterator<int, SegBegin<uint32_t>, cub::CountingInputIterator<int>> sb(
                cub::CountingInputIterator<int>(0), SegBegin<uint32_t>{o});
            cub::TransformInputIterator<int, SegEnd<uint32_t>, cub::CountingInputIterator<int>> se(
                cub::CountingInputIterator<int>(0), SegEnd<uint32_t>{o, perm, o_lo, o_hi});
            PREP_CK(cub::DeviceSegmentedRadixSort::SortKeys(hub_tmp_store, nb, db, (int)hub_entries,
                                                            (int)n_huge, sb, se, 0, end_bit, hs));
          }
          if (!hub_roles_known) {
            hub_roles_known = true;
            if (db.Current() != new_adj) {
              // the sorted rows landed in the side buffer: move this chunk's
              // (the other rows are rewritten by their own chunks) and let the
              // later chunks start from new_adj, so they end in new_adj
              PREP_CK(cudaMemcpyAsync(new_adj, db.Current(), (size_t)hub_entries * sizeof(uint32_t),
                                      cudaMemcpyDeviceToDevice, hs));
              hub_buf[0] = new_adj;
              hub_buf[1] = sort_tmp;
            }
          }
        }
      }
    }
    if (hs) {  // the layout is complete when both streams are
      PREP_CK(cudaEventRecord(hev, hs));
      PREP_CK(cudaStreamWaitEvent(s, hev, 0));
    }
    {
      if (fused_sort) out->rows_sorted = true;
      // the degree cut table (kc_count.cu DegCut)
      PREP_CK(dalloc(&dcut, (size_t)out->max_degree + 2, s));
      degcut_kernel<<<G, B, 0, s>>>(sdeg, n_nz, out->max_degree, dcut);
      PREP_CK(cudaGetLastError());
    }
    PREP_CK(cudaStreamSynchronize(s));
    PREP_CK(cudaMemcpy(hb + 7, bounds + 7, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    if (hb[7]) {  // a neighbour id >= n
      out->invalid = true;
      goto done;
    }
  }
  out->off = new_off;
  out->adj = new_adj;
  out->perm = perm;
  out->dcut = dcut;
  dcut = nullptr;
  new_off = nullptr;
  new_adj = nullptr;
  perm = nullptr;
done:
  if (hs) {
    cudaStreamSynchronize(hs);
    cudaStreamDestroy(hs);
  }
  if (hev) cudaEventDestroy(hev);
  dfree(deg, s);
  dfree(iota, s);
  dfree(sdeg, s);
  dfree(perm, s);
  dfree(inv, s);
  dfree(bounds, s);
  dfree(off64_tmp, s);
  dfree(chunks, s);
  dfree(new_off, s);
  dfree(new_adj, s);
  dfree(sort_tmp, s);
  dfree(tiers, s);
  dfree(hub_tmp_store, s);
  dfree(tier_list, s);
  dfree(tier_cnt, s);
  dfree(dcut, s);
  dfree(tmp, s);
  return err;
}

}  // namespace kcb
