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

}  // namespace

#define PREP_CK(x)                         \
  do {                                     \
    cudaError_t e_ = (x);                  \
    if (e_ != cudaSuccess) {               \
      err = e_;                            \
      goto done;                           \
    }                                      \
  } while (0)

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
    // rows of degree > 64 (ids [0, n_big)) are cut into 1024-entry chunks
    // for warps; the rest take the 8-lane-per-row kernel
    const uint32_t n_big = out->cls_begin[C_SUB];
    uint64_t total = 0;  // 1024-entry chunks of the big rows
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
    // relabel: all rows at once, or — pipelined upload — the rows of each
    // chunk of old ids as soon as its bytes have landed (event), so the
    // layout overlaps the host-to-device copy
    const int nparts = feed ? feed->k : 1;
    for (int c = 0; c < nparts; ++c) {
      const uint32_t o_lo = feed ? feed->old_lo[c] : 0u;
      const uint32_t o_hi = feed ? feed->old_lo[c + 1] : n;
      if (feed && feed->host_wait) feed->host_wait(feed->ctx, c);  // recorded by the stager
      if (feed) PREP_CK(cudaStreamWaitEvent(s, feed->ready[c], 0));
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
      if (n_big) {
        if (off64)
          relabel_rows_kernel<uint64_t><<<G, B, 0, s>>>(off, adj, perm, inv, chunks, n_big,
                                                        (const uint64_t*)new_off, new_adj, total,
                                                        o_lo, o_hi, n, bounds + 7);
        else
          relabel_rows_kernel<uint32_t><<<G, B, 0, s>>>(off, adj, perm, inv, chunks, n_big,
                                                        (const uint32_t*)new_off, new_adj, total,
                                                        o_lo, o_hi, n, bounds + 7);
        PREP_CK(cudaGetLastError());
      }
    }
    {
      // sort each row ascending (segmented sort over the new offsets)
      if (KC_PREP_SORT && sort_rows && nnz > 0 && nnz < (1ull << 31)) {
        PREP_CK(dalloc(&sort_tmp, nnz + ADJ_PAD, s));
        PREP_CK(cudaMemsetAsync(sort_tmp + nnz, 0, ADJ_PAD * sizeof(uint32_t), s));
        size_t nb2 = 0;
        if (off64) {
          const uint64_t* o = (const uint64_t*)new_off;
          PREP_CK(cub::DeviceSegmentedSort::SortKeys(nullptr, nb2, new_adj, sort_tmp, (int64_t)nnz,
                                                     (int64_t)n_nz, o, o + 1, s));
        } else {
          const uint32_t* o = (const uint32_t*)new_off;
          PREP_CK(cub::DeviceSegmentedSort::SortKeys(nullptr, nb2, new_adj, sort_tmp, (int64_t)nnz,
                                                     (int64_t)n_nz, o, o + 1, s));
        }
        if (nb2 > tmp_bytes) {
          dfree(tmp, s);
          tmp = nullptr;
          tmp_bytes = nb2;
          PREP_CK(dmalloc(&tmp, tmp_bytes, s));
        }
        if (off64) {
          const uint64_t* o = (const uint64_t*)new_off;
          PREP_CK(cub::DeviceSegmentedSort::SortKeys(tmp, tmp_bytes, new_adj, sort_tmp, (int64_t)nnz,
                                                     (int64_t)n_nz, o, o + 1, s));
        } else {
          const uint32_t* o = (const uint32_t*)new_off;
          PREP_CK(cub::DeviceSegmentedSort::SortKeys(tmp, tmp_bytes, new_adj, sort_tmp, (int64_t)nnz,
                                                     (int64_t)n_nz, o, o + 1, s));
        }
        std::swap(new_adj, sort_tmp);
        out->rows_sorted = true;
      }
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
  dfree(dcut, s);
  dfree(tmp, s);
  return err;
}

}  // namespace kcb
