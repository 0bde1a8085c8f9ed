// kc_peel.cu — an independent on-device coreness algorithm and a device
// verify: the checker side of the path at sizes where the host oracle would
// need the 8-9 GB CSR round trip.
//
// Reference: kcore::peel_coreness, /root/reference/proj/src/oracle.cpp:21-66
// (bucket peeling: repeatedly remove a minimum-degree vertex; its coreness
// is its degree at removal, made monotone), and kcore::verify,
// oracle.cpp:68-75 (pointwise comparison, ascending node id).
//
// Device form: level-synchronous peeling.  Level k removes, until none is
// left, every remaining vertex whose remaining degree is <= k, and assigns it
// coreness k — the same removal order up to ties inside a level, hence the
// same coreness (the peel value of a vertex does not depend on how ties are
// broken).  It shares nothing with the FastK solvers but the CSR layout.
//
// One cooperative launch (148 CTAs x 1024 threads), per level:
//   A  scan the remaining list: peeled -> dropped, degree <= k -> frontier
//      (core = k), else -> next remaining list
//   B  repeat: every frontier vertex decrements its live neighbours; the
//      decrement that takes a degree from k+1 to k puts that neighbour in the
//      next frontier (exactly once).  Rows longer than BIG_ROW are spread
//      over the whole grid, the rest take a warp each.
// Work: the remaining-list scans sum to sum_v (core(v) + 1) entries, the
// frontier passes to nnz decrements.
#include <cooperative_groups.h>
#include <cstdint>

#include "kc_internal.h"

namespace cg = cooperative_groups;

namespace kcb {
namespace {

constexpr int PT = 1024;                // threads per CTA
constexpr uint32_t NONE = 0xffffffffu;  // not peeled yet
constexpr uint32_t BIG_ROW = 4096;      // rows longer than this: grid-wide

struct PeelCtl {
  uint32_t remc[3];   // remaining-list sizes (3-slot rotation, see below)
  uint32_t fc[3];     // frontier sizes (warp rows)
  uint32_t fcb[3];    // frontier sizes (grid rows)
  uint32_t levels;    // levels run (k_max + 1)
};

template <typename OffT>
struct PP {
  const OffT* off;
  const uint32_t* adj;
  uint32_t n_nz;
  uint32_t* deg;      // remaining degree
  uint32_t* core;     // NONE until peeled
  uint32_t* rem[2];   // remaining lists (ping-pong by level)
  uint32_t* fr[2];    // frontier lists, warp rows
  uint32_t* frb[2];   // frontier lists, grid rows
  PeelCtl* ctl;
};

// Counter slots rotate through 3: a phase reads slot s, appends to s+1 and
// zeroes s+2 — which was last read before the previous grid barrier and is
// next appended to after the coming one.
__device__ __forceinline__ uint32_t slot(uint32_t s) { return s % 3u; }

// Warp-aggregated append of `v` (where `take`) to list/counter.
__device__ __forceinline__ void append(bool take, uint32_t v, uint32_t* list, uint32_t* count) {
  const uint32_t m = __ballot_sync(0xffffffffu, take);
  if (!m) return;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(count, (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (take) list[base + __popc(m & ((1u << lane) - 1u))] = v;
}

template <typename OffT>
__device__ __forceinline__ bool is_big(const PP<OffT>& p, uint32_t v) {
  return (uint64_t)p.off[v + 1] - (uint64_t)p.off[v] > BIG_ROW;
}

// Decrement neighbour w of a vertex peeled at level k; the decrement from
// k+1 to k puts w in the next frontier.
template <typename OffT>
__device__ __forceinline__ void decrement(const PP<OffT>& p, uint32_t w, uint32_t k, bool& add) {
  add = false;
  if (*reinterpret_cast<volatile uint32_t*>(&p.core[w]) != NONE) return;  // peeled already
  const uint32_t old = atomicSub(&p.deg[w], 1u);
  if (old == k + 1) {
    p.core[w] = k;
    add = true;
  }
}

template <typename OffT>
__global__ void __launch_bounds__(PT, 1) peel_kernel(PP<OffT> p) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t gtid = blockIdx.x * PT + threadIdx.x;
  const uint32_t gsize = gridDim.x * PT;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gwarp = gtid >> 5, nwarps = gsize >> 5;
  uint32_t ra = 0, fa = 0;  // rotation steps
  bool first = true;
  for (uint32_t k = 0;; ++k) {
    // ---- A: split the remaining list at level k
    {
      const uint32_t R = first ? p.n_nz : p.ctl->remc[slot(ra)];
      const uint32_t* in = p.rem[ra & 1];
      uint32_t* out = p.rem[(ra + 1) & 1];
      uint32_t* fo = p.fr[(fa + 1) & 1];
      uint32_t* fob = p.frb[(fa + 1) & 1];
      for (uint32_t b = blockIdx.x * PT; b < R; b += gsize) {  // warp-uniform trip count
        const uint32_t i = b + threadIdx.x;
        uint32_t v = 0;
        bool keep = false, now = false;
        if (i < R) {
          v = first ? i : in[i];
          if (p.core[v] == NONE) {
            if (p.deg[v] <= k) {
              p.core[v] = k;
              now = true;
            } else {
              keep = true;
            }
          }
        }
        const bool big = now && is_big(p, v);
        append(keep, v, out, &p.ctl->remc[slot(ra + 1)]);
        append(now && !big, v, fo, &p.ctl->fc[slot(fa + 1)]);
        append(big, v, fob, &p.ctl->fcb[slot(fa + 1)]);
      }
      if (gtid == 0) {
        p.ctl->remc[slot(ra + 2)] = 0;
        p.ctl->fc[slot(fa + 2)] = 0;
        p.ctl->fcb[slot(fa + 2)] = 0;
      }
      grid.sync();
      ++ra;
      ++fa;
      first = false;
    }
    if (p.ctl->remc[slot(ra)] == 0 && p.ctl->fc[slot(fa)] == 0 && p.ctl->fcb[slot(fa)] == 0) {
      if (gtid == 0) p.ctl->levels = k;  // levels 0 .. k-1 peeled something
      return;  // every vertex peeled
    }
    // ---- B: frontier passes at level k
    for (;;) {
      const uint32_t F = p.ctl->fc[slot(fa)], Fb = p.ctl->fcb[slot(fa)];
      if (F == 0 && Fb == 0) break;  // grid-uniform
      const uint32_t* fin = p.fr[fa & 1];
      const uint32_t* finb = p.frb[fa & 1];
      uint32_t* fo = p.fr[(fa + 1) & 1];
      uint32_t* fob = p.frb[(fa + 1) & 1];
      uint32_t* cnt = &p.ctl->fc[slot(fa + 1)];
      uint32_t* cntb = &p.ctl->fcb[slot(fa + 1)];
      // long rows: the whole grid walks each one
      for (uint32_t j = 0; j < Fb; ++j) {
        const uint32_t v = finb[j];
        const uint64_t ob = (uint64_t)p.off[v], oe = (uint64_t)p.off[v + 1];
        for (uint64_t b = ob + (uint64_t)blockIdx.x * PT; b < oe; b += gsize) {
          const uint64_t e = b + threadIdx.x;
          bool add = false;
          uint32_t w = 0;
          if (e < oe) {
            w = p.adj[e];
            decrement(p, w, k, add);
          }
          const bool big = add && is_big(p, w);
          append(add && !big, w, fo, cnt);
          append(big, w, fob, cntb);
        }
      }
      // the rest: a warp per frontier vertex
      for (uint32_t j = gwarp; j < F; j += nwarps) {
        const uint32_t v = fin[j];
        const uint64_t ob = (uint64_t)p.off[v], oe = (uint64_t)p.off[v + 1];
        for (uint64_t b = ob; b < oe; b += 32) {
          const uint64_t e = b + lane;
          bool add = false;
          uint32_t w = 0;
          if (e < oe) {
            w = p.adj[e];
            decrement(p, w, k, add);
          }
          const bool big = add && is_big(p, w);
          append(add && !big, w, fo, cnt);
          append(big, w, fob, cntb);
        }
      }
      if (gtid == 0) {
        p.ctl->fc[slot(fa + 2)] = 0;
        p.ctl->fcb[slot(fa + 2)] = 0;
      }
      grid.sync();
      ++fa;
    }
  }
}

template <typename OffT>
__global__ void peel_init_kernel(PP<OffT> p) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < p.n_nz; u += gridDim.x * blockDim.x) {
    p.deg[u] = (uint32_t)((uint64_t)p.off[u + 1] - (uint64_t)p.off[u]);
    p.core[u] = NONE;
  }
  if (blockIdx.x == 0 && threadIdx.x < 3) {
    p.ctl->remc[threadIdx.x] = p.ctl->fc[threadIdx.x] = p.ctl->fcb[threadIdx.x] = 0;
    if (threadIdx.x == 0) p.ctl->levels = 0;
  }
}

// core (layout ids) -> caller ids; isolated vertices have coreness 0.
__global__ void peel_out_kernel(const uint32_t* core, const uint32_t* perm, uint32_t n,
                                uint32_t n_nz, uint32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[perm[i]] = i < n_nz ? core[i] : 0u;
}

__global__ void mismatch_count_kernel(const uint32_t* a, const uint32_t* b, uint32_t n,
                                      unsigned long long* count) {
  unsigned long long c = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    c += a[i] != b[i];
  c = __reduce_add_sync(0xffffffffu, (uint32_t)c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// The first `cap` mismatching ids in ascending order: block-ordered
// compaction over 1024-id tiles, tiles in order (one CTA, sequential over
// tiles; only runs when mismatches exist).
__global__ void mismatch_list_kernel(const uint32_t* cand, const uint32_t* truth, uint32_t n,
                                     uint32_t* ids, uint32_t cap) {
  __shared__ uint32_t warp_cnt[32];
  __shared__ uint32_t base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t t = 0; t < n && base < cap; t += blockDim.x) {
    const uint32_t i = t + threadIdx.x;
    const bool bad = i < n && cand[i] != truth[i];
    const uint32_t m = __ballot_sync(0xffffffffu, bad);
    if (lane == 0) warp_cnt[w] = __popc(m);
    __syncthreads();
    uint32_t before = base;
    for (uint32_t k = 0; k < w; ++k) before += warp_cnt[k];
    const uint32_t pos = before + __popc(m & ((1u << lane) - 1u));
    if (bad && pos < cap) ids[pos] = i;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t tot = 0;
      for (uint32_t k = 0; k < blockDim.x / 32; ++k) tot += warp_cnt[k];
      base += tot;
    }
    __syncthreads();
  }
}

template <typename OffT>
cudaError_t peel_t(const PeelBuffers& b, int num_sms, cudaStream_t s) {
  PP<OffT> p{};
  p.off = static_cast<const OffT*>(b.off);
  p.adj = b.adj;
  p.n_nz = b.n_nz;
  p.deg = b.deg;
  p.core = b.core;
  p.rem[0] = b.rem[0];
  p.rem[1] = b.rem[1];
  p.fr[0] = b.fr[0];
  p.fr[1] = b.fr[1];
  p.frb[0] = b.frb[0];
  p.frb[1] = b.frb[1];
  p.ctl = reinterpret_cast<PeelCtl*>(b.ctl);
  peel_init_kernel<OffT><<<num_sms * 4, 256, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || b.n_nz == 0) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, peel_kernel<OffT>, PT, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  void* args[] = {&p};
  return cudaLaunchCooperativeKernel((const void*)peel_kernel<OffT>, dim3(num_sms), dim3(PT), args,
                                     0, s);
}

}  // namespace

size_t peel_ctl_bytes() { return sizeof(PeelCtl); }

cudaError_t launch_peel(const PeelBuffers& b, bool off64, int num_sms, cudaStream_t s) {
  return off64 ? peel_t<uint64_t>(b, num_sms, s) : peel_t<uint32_t>(b, num_sms, s);
}

cudaError_t launch_peel_out(const PeelBuffers& b, const uint32_t* perm, uint32_t n, uint32_t* out,
                            int num_sms, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  peel_out_kernel<<<num_sms * 4, 256, 0, s>>>(b.core, perm, n, b.n_nz, out);
  return cudaGetLastError();
}

cudaError_t launch_mismatch_count(const uint32_t* a, const uint32_t* b, uint32_t n,
                                  unsigned long long* count, int num_sms, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  mismatch_count_kernel<<<num_sms * 4, 256, 0, s>>>(a, b, n, count);
  return cudaGetLastError();
}

cudaError_t launch_mismatch_list(const uint32_t* cand, const uint32_t* truth, uint32_t n,
                                 uint32_t* ids, uint32_t cap, cudaStream_t s) {
  if (n == 0 || cap == 0) return cudaSuccess;
  mismatch_list_kernel<<<1, 1024, 0, s>>>(cand, truth, n, ids, cap);
  return cudaGetLastError();
}

}  // namespace kcb
