// kc_gen.cu — synthetic inputs built directly in HBM: the five BASELINE.json
// configs under the "kcgen v1" spec (seeded counter-based PRNG; DESIGN.md
// §Inputs), followed by on-device CSR construction.
//
// CSR construction is the GPU form of the reference's build_csr
// (/root/reference/proj/src/graph.cpp:85-128): drop self-loops, count both
// directions, scatter, sort each row, drop duplicates, compact.  The output
// is byte-identical to the reference's Graph::from_edges on the same edge
// list (tests/test_gen.py pins it against oracle/ and the reference).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/kcore_b200.h"
#include "kc_internal.h"

namespace {

// ---- kcgen v1 PRNG (SplitMix64 finalizer over a counter) -----------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(seed * 0x9E3779B97F4A7C15ULL + mix64(stream + 0x632BE59BD9B4E019ULL));
}
__host__ __device__ __forceinline__ uint64_t rng_at(uint64_t key, uint64_t ctr) {
  return mix64(key + ctr * 0x9E3779B97F4A7C15ULL);
}
__host__ __device__ __forceinline__ uint32_t range32(uint32_t x, uint32_t n) {
  return (uint32_t)(((uint64_t)x * (uint64_t)n) >> 32);
}
// Bijective seeded shuffle of [0, 2^bits) (R-MAT id permutation).
__host__ __device__ __forceinline__ uint32_t perm_bits(uint32_t x, uint32_t bits, uint64_t key) {
  const uint32_t mask = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
  const uint32_t half = bits / 2 ? bits / 2 : 1;
  for (int r = 0; r < 4; ++r) {
    const uint64_t k = rng_at(key, (uint64_t)r);
    x = (uint32_t)((x * ((uint32_t)k | 1u) + (uint32_t)(k >> 32)) & mask);
    x ^= x >> half;
    x &= mask;
  }
  return x;
}

constexpr uint32_t P_KEEP = 3006477107u;  // floor(0.70 * 2^32)
constexpr uint32_t P_DIAG = 214748364u;   // floor(0.05 * 2^32)
constexpr uint32_t T_A = 2448131358u;     // floor(0.57 * 2^32)
constexpr uint32_t T_AB = 3264175144u;    // floor(0.76 * 2^32)
constexpr uint32_t T_ABC = 4080218931u;   // floor(0.95 * 2^32)

__global__ void gen_er_kernel(uint32_t n, uint64_t m, uint64_t key, uint2* pairs) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = rng_at(key, i);
    pairs[i] = make_uint2(range32((uint32_t)r, n), range32((uint32_t)(r >> 32), n));
  }
}

__global__ void gen_grid_kernel(uint32_t side, uint64_t k1, uint64_t k2, uint2* pairs) {
  const uint64_t n = (uint64_t)side * side;
  for (uint64_t id = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; id < n;
       id += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)(id / side), c = (uint32_t)(id % side);
    const uint64_t h = rng_at(k1, id), h2 = rng_at(k2, id);
    const uint32_t u = (uint32_t)id;
    pairs[3 * id + 0] = make_uint2(u, (c + 1 < side && (uint32_t)h < P_KEEP) ? u + 1 : u);
    pairs[3 * id + 1] = make_uint2(u, (r + 1 < side && (uint32_t)(h >> 32) < P_KEEP) ? u + side : u);
    pairs[3 * id + 2] =
        make_uint2(u, (r + 1 < side && c + 1 < side && (uint32_t)h2 < P_DIAG) ? u + side + 1 : u);
  }
}

__global__ void gen_rmat_kernel(uint32_t scale, uint64_t m, uint64_t key, uint64_t pkey,
                                uint2* pairs) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t u = 0, v = 0;
    uint64_t h = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      if ((l & 1) == 0) h = rng_at(key, i * 16 + l / 2);
      const uint32_t x = (l & 1) ? (uint32_t)(h >> 32) : (uint32_t)h;
      const uint32_t bu = x >= T_AB, bv = (x >= T_A && x < T_AB) || x >= T_ABC;
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    pairs[i] = make_uint2(perm_bits(u, scale, pkey), perm_bits(v, scale, pkey));
  }
}

__device__ __forceinline__ uint32_t cdf_search(const uint64_t* pre, uint32_t n, uint64_t target) {
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (pre[mid] <= target) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void gen_chunglu_kernel(uint32_t n, const uint64_t* pre, uint64_t m, uint64_t key,
                                   uint2* pairs) {
  const uint64_t total = pre[n];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = cdf_search(pre, n, __umul64hi(rng_at(key, 2 * i), total));
    const uint32_t b = cdf_search(pre, n, __umul64hi(rng_at(key, 2 * i + 1), total));
    pairs[i] = make_uint2(a, b);
  }
}

__global__ void gen_cliques_kernel(uint32_t n, uint32_t cliques, uint32_t csize, uint64_t ckey,
                                   uint2* pairs) {
  const uint64_t per = (uint64_t)csize * (csize - 1) / 2;
  const uint64_t total = per * cliques;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = (uint32_t)(q / per);
    uint64_t k = q % per;
    // k-th pair (a < b) in row-major order over a
    uint32_t a = 0;
    uint64_t rowlen = csize - 1;
    while (k >= rowlen) {
      k -= rowlen;
      ++a;
      --rowlen;
    }
    const uint32_t b = a + 1 + (uint32_t)k;
    const uint32_t ua = range32((uint32_t)rng_at(ckey, (uint64_t)c * csize + a), n);
    const uint32_t ub = range32((uint32_t)rng_at(ckey, (uint64_t)c * csize + b), n);
    pairs[q] = make_uint2(ua, ub);
  }
}

// ---- CSR construction (graph.cpp:85-128 on the GPU) ----------------------
__global__ void count_kernel(const uint2* pairs, uint64_t m, unsigned long long* cnt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 e = pairs[i];
    if (e.x == e.y) continue;
    atomicAdd(&cnt[e.x], 1ull);
    atomicAdd(&cnt[e.y], 1ull);
  }
}

__global__ void scatter_kernel(const uint2* pairs, uint64_t m, unsigned long long* cur,
                               uint32_t* nbr) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 e = pairs[i];
    if (e.x == e.y) continue;
    nbr[atomicAdd(&cur[e.x], 1ull)] = e.y;
    nbr[atomicAdd(&cur[e.y], 1ull)] = e.x;
  }
}

// keep[i] = 1 iff entry i is the first of its row or differs from its
// predecessor (rows sorted).  Warp per row.
__global__ void keep_kernel(const uint64_t* start, uint32_t n, const uint32_t* nbr,
                            uint32_t* keep) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t u = w0; u < n; u += nw) {
    const uint64_t b = start[u], e = start[u + 1];
    for (uint64_t i = b + lane; i < e; i += 32) keep[i] = (i == b || nbr[i] != nbr[i - 1]) ? 1u : 0u;
  }
}

__global__ void compact_kernel(const uint32_t* nbr, const uint32_t* keep, const uint64_t* pos,
                               uint64_t total, uint32_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (keep[i]) out[pos[i]] = nbr[i];
}

__global__ void new_offsets_kernel(const uint64_t* start, const uint64_t* pos, uint32_t n,
                                   uint64_t* off) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u <= n;
       u += (uint64_t)gridDim.x * blockDim.x)
    off[u] = pos[start[u]];
}

thread_local std::string g_gen_error;

kc_status gfail(cudaError_t e, const char* what) {
  cudaGetLastError();
  g_gen_error = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? KC_ERR_OUT_OF_MEMORY : KC_ERR_CUDA;
}

#define GK(x)                                   \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) return gfail(e_, #x); \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
  template <typename T>
  T* as() { return static_cast<T*>(p); }
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 1); }
  void release() { p = nullptr; }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
  }
};

// Chung–Lu weights on the host: the identical formula and summation order as
// the kcgen v1 spec (double precision, glibc pow, 65536-entry chunks summed in
// order, 100 bisection steps, weights quantised to 1/1024).
void chunglu_prefix(uint32_t n, uint64_t seed, std::vector<uint64_t>& pre, uint64_t* m_out) {
  const double gamma = 2.1, mean_target = 20.0, w_max = 5e5;
  const uint64_t key = stream_key(seed, 5);
  std::vector<double> g(n);
  const double ex = -1.0 / (gamma - 1.0);
  unsigned T = std::thread::hardware_concurrency();
  if (T == 0) T = 4;
  if (T > 32) T = 32;
  auto par = [&](auto fn, uint64_t count) {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        const uint64_t b = count * t / T, e = count * (t + 1) / T;
        for (uint64_t i = b; i < e; ++i) fn(i);
      });
    for (auto& x : th) x.join();
  };
  par([&](uint64_t i) {
    const double U = (double)(rng_at(key, i) >> 11) * 0x1.0p-53;
    g[i] = std::pow(1.0 - U, ex);
  }, n);
  const uint64_t CH = 1 << 16;
  const uint64_t nch = (n + CH - 1) / CH;
  std::vector<double> part(nch ? nch : 1);
  double lo = 0.0, hi = mean_target;
  for (int it = 0; it < 100; ++it) {
    const double x = 0.5 * (lo + hi);
    par([&](uint64_t c) {
      double s = 0.0;
      const uint64_t e = (c + 1) * CH < n ? (c + 1) * CH : n;
      for (uint64_t i = c * CH; i < e; ++i) {
        const double w = x * g[i];
        s += w < w_max ? w : w_max;
      }
      part[c] = s;
    }, nch);
    double s = 0.0;
    for (uint64_t c = 0; c < nch; ++c) s += part[c];
    if (s / (double)n < mean_target) lo = x; else hi = x;
  }
  const double xm = 0.5 * (lo + hi);
  pre.assign((size_t)n + 1, 0);
  std::vector<uint64_t> wq(n);
  par([&](uint64_t i) {
    double w = xm * g[i];
    w = w < w_max ? w : w_max;
    wq[i] = (uint64_t)std::llround(w * 1024.0);
  }, n);
  for (uint32_t i = 0; i < n; ++i) pre[i + 1] = pre[i] + wq[i];
  *m_out = (pre[n] + 1024) / 2048;  // round(sum(w) / 2)
}

// Sort rows [r0, r1) with one segmented sort (CUB's item count is an int).
kc_status sort_rows(uint32_t* keys, uint32_t* alt, const uint64_t* start, uint32_t r0, uint32_t r1,
                    cudaStream_t s) {
  uint64_t b = 0, e = 0;
  GK(cudaMemcpy(&b, start + r0, 8, cudaMemcpyDeviceToHost));
  GK(cudaMemcpy(&e, start + r1, 8, cudaMemcpyDeviceToHost));
  if (e == b) return KC_OK;
  size_t need = 0;
  // offsets relative to b: sort the window keys[b, e) with begin/end offsets start[r0..r1] - b
  DevBuf rel;
  GK(rel.alloc(((size_t)(r1 - r0) + 1) * sizeof(uint64_t)));
  std::vector<uint64_t> h((size_t)(r1 - r0) + 1);
  GK(cudaMemcpy(h.data(), start + r0, h.size() * 8, cudaMemcpyDeviceToHost));
  for (auto& x : h) x -= b;
  GK(cudaMemcpy(rel.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
  const uint64_t* ro = rel.as<uint64_t>();
  const int items = (int)(e - b);
  const int segs = (int)(r1 - r0);
  GK(cub::DeviceSegmentedSort::SortKeys(nullptr, need, keys + b, alt + b, items, segs, ro, ro + 1, s));
  DevBuf tmp;
  GK(tmp.alloc(need));
  GK(cub::DeviceSegmentedSort::SortKeys(tmp.p, need, keys + b, alt + b, items, segs, ro, ro + 1, s));
  GK(cudaMemcpyAsync(keys + b, alt + b, (e - b) * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  GK(cudaStreamSynchronize(s));
  return KC_OK;
}

// Build the CSR of `pairs` (m entries, device) into *out.
kc_status build_csr_dev(uint32_t n, const uint2* pairs, uint64_t m, cudaStream_t s,
                        uint64_t** off_out, uint32_t** nbr_out, uint64_t* nnz_out) {
  const int G = 148 * 8, B = 256;
  DevBuf cnt, start, nbr, alt, keep, pos, off, out;
  GK(cnt.alloc(((size_t)n + 1) * 8));
  GK(cudaMemsetAsync(cnt.p, 0, ((size_t)n + 1) * 8, s));
  count_kernel<<<G, B, 0, s>>>(pairs, m, cnt.as<unsigned long long>());
  GK(cudaGetLastError());
  GK(start.alloc(((size_t)n + 1) * 8));
  size_t need = 0;
  GK(cub::DeviceScan::ExclusiveSum(nullptr, need, cnt.as<uint64_t>(), start.as<uint64_t>(), n + 1, s));
  {
    DevBuf tmp;
    GK(tmp.alloc(need));
    GK(cub::DeviceScan::ExclusiveSum(tmp.p, need, cnt.as<uint64_t>(), start.as<uint64_t>(), n + 1, s));
    GK(cudaStreamSynchronize(s));
  }
  uint64_t total = 0;
  GK(cudaMemcpy(&total, start.as<uint64_t>() + n, 8, cudaMemcpyDeviceToHost));
  GK(cudaMemcpyAsync(cnt.p, start.p, ((size_t)n + 1) * 8, cudaMemcpyDeviceToDevice, s));
  GK(nbr.alloc(total * 4));
  scatter_kernel<<<G, B, 0, s>>>(pairs, m, cnt.as<unsigned long long>(), nbr.as<uint32_t>());
  GK(cudaGetLastError());
  GK(cudaStreamSynchronize(s));
  cnt.reset();
  // segmented sort in row batches of < 2^30 entries
  GK(alt.alloc(total * 4));
  {
    std::vector<uint64_t> hs((size_t)n + 1);
    GK(cudaMemcpy(hs.data(), start.p, hs.size() * 8, cudaMemcpyDeviceToHost));
    uint32_t r0 = 0;
    while (r0 < n) {
      uint32_t r1 = r0;
      // extend while the batch stays under 2^30 entries (a single row may exceed: own batch)
      while (r1 < n && (hs[r1 + 1] - hs[r0] < (1ull << 30) || r1 == r0)) ++r1;
      kc_status st = sort_rows(nbr.as<uint32_t>(), alt.as<uint32_t>(), start.as<uint64_t>(), r0, r1, s);
      if (st != KC_OK) return st;
      r0 = r1;
    }
  }
  alt.reset();
  GK(keep.alloc((total + 1) * 4));
  GK(cudaMemsetAsync(keep.p, 0, (total + 1) * 4, s));
  keep_kernel<<<G, B, 0, s>>>(start.as<uint64_t>(), n, nbr.as<uint32_t>(), keep.as<uint32_t>());
  GK(cudaGetLastError());
  GK(pos.alloc((total + 1) * 8));
  {
    auto in = cub::TransformInputIterator<uint64_t, cub::CastOp<uint64_t>, const uint32_t*>(
        keep.as<uint32_t>(), cub::CastOp<uint64_t>());
    need = 0;
    GK(cub::DeviceScan::ExclusiveSum(nullptr, need, in, pos.as<uint64_t>(), total + 1, s));
    DevBuf tmp;
    GK(tmp.alloc(need));
    GK(cub::DeviceScan::ExclusiveSum(tmp.p, need, in, pos.as<uint64_t>(), total + 1, s));
    GK(cudaStreamSynchronize(s));
  }
  uint64_t nnz = 0;
  GK(cudaMemcpy(&nnz, pos.as<uint64_t>() + total, 8, cudaMemcpyDeviceToHost));
  GK(off.alloc(((size_t)n + 1) * 8));
  new_offsets_kernel<<<G, B, 0, s>>>(start.as<uint64_t>(), pos.as<uint64_t>(), n, off.as<uint64_t>());
  GK(cudaGetLastError());
  GK(out.alloc(nnz * 4));
  compact_kernel<<<G, B, 0, s>>>(nbr.as<uint32_t>(), keep.as<uint32_t>(), pos.as<uint64_t>(), total,
                                 out.as<uint32_t>());
  GK(cudaGetLastError());
  GK(cudaStreamSynchronize(s));
  *off_out = off.as<uint64_t>();
  *nbr_out = out.as<uint32_t>();
  *nnz_out = nnz;
  off.release();
  out.release();
  return KC_OK;
}

}  // namespace

namespace kcb {  // for the edge-list loader (kc_ingest.cu)
kc_status build_csr_dev_public(uint32_t n, const uint2* pairs, uint64_t m, cudaStream_t s,
                               uint64_t** off_out, uint32_t** nbr_out, uint64_t* nnz_out) {
  return build_csr_dev(n, pairs, m, s, off_out, nbr_out, nnz_out);
}
const char* gen_last_error() { return g_gen_error.c_str(); }
}  // namespace kcb

extern "C" {

kc_status kc_gen_config(int cfg, uint64_t p0, uint64_t p1, uint64_t p2, uint64_t seed, int device,
                        kc_csr_dev** out) {
  kcb::DeviceGuard device_guard;  // restore the caller's current device
  if (!out) return KC_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return KC_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= count) return KC_ERR_NO_DEVICE;
  GK(cudaSetDevice(device));
  cudaStream_t s;
  GK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct SG { cudaStream_t s; ~SG() { cudaStreamDestroy(s); } } sg{s};
  const int G = 148 * 8, B = 256;
  uint32_t n = 0;
  uint64_t m = 0;
  DevBuf pairs, pre;
  switch (cfg) {
    case 1: {  // ER G(n, m)
      n = (uint32_t)p0;
      m = p1;
      GK(pairs.alloc(m * 8));
      gen_er_kernel<<<G, B, 0, s>>>(n, m, stream_key(seed, 1), pairs.as<uint2>());
      break;
    }
    case 2: {  // grid side x side
      const uint32_t side = (uint32_t)p0;
      if ((uint64_t)side * side >= (1ull << 32)) return KC_ERR_INVALID_ARGUMENT;
      n = side * side;
      m = 3ull * n;
      GK(pairs.alloc(m * 8));
      gen_grid_kernel<<<G, B, 0, s>>>(side, stream_key(seed, 2), stream_key(seed, 3), pairs.as<uint2>());
      break;
    }
    case 3:
    case 5: {  // R-MAT scale p0, edge factor p1
      const uint32_t scale = (uint32_t)p0;
      if (scale == 0 || scale > 31) return KC_ERR_INVALID_ARGUMENT;
      n = 1u << scale;
      m = p1 << scale;
      GK(pairs.alloc(m * 8));
      gen_rmat_kernel<<<G, B, 0, s>>>(scale, m, stream_key(seed, 4), stream_key(seed, 9), pairs.as<uint2>());
      break;
    }
    case 4: {  // Chung-Lu n = p0, cliques p1 x size p2
      n = (uint32_t)p0;
      std::vector<uint64_t> hpre;
      uint64_t mcl = 0;
      chunglu_prefix(n, seed, hpre, &mcl);
      const uint64_t per = p2 >= 2 ? p2 * (p2 - 1) / 2 : 0;
      m = mcl + p1 * per;
      GK(pre.alloc(hpre.size() * 8));
      GK(cudaMemcpy(pre.p, hpre.data(), hpre.size() * 8, cudaMemcpyHostToDevice));
      GK(pairs.alloc(m * 8));
      gen_chunglu_kernel<<<G, B, 0, s>>>(n, pre.as<uint64_t>(), mcl, stream_key(seed, 6), pairs.as<uint2>());
      if (p1 && per)
        gen_cliques_kernel<<<G, B, 0, s>>>(n, (uint32_t)p1, (uint32_t)p2, stream_key(seed, 7),
                                           pairs.as<uint2>() + mcl);
      break;
    }
    default:
      return KC_ERR_INVALID_ARGUMENT;
  }
  GK(cudaGetLastError());
  GK(cudaStreamSynchronize(s));
  uint64_t* off = nullptr;
  uint32_t* nbr = nullptr;
  uint64_t nnz = 0;
  kc_status st = build_csr_dev(n, pairs.as<uint2>(), m, s, &off, &nbr, &nnz);
  if (st != KC_OK) return st;
  kc_csr_dev* g = new (std::nothrow) kc_csr_dev();
  if (!g) {
    cudaFree(off);
    cudaFree(nbr);
    return KC_ERR_OUT_OF_MEMORY;
  }
  g->view.n = n;
  g->view.nnz = nnz;
  g->view.offsets = off;
  g->view.neighbors = nbr;
  g->device = device;
  *out = g;
  return KC_OK;
}

void kc_csr_dev_free(kc_csr_dev* g) {
  kcb::DeviceGuard device_guard;  // restore the caller's current device
  if (!g) return;
  cudaSetDevice(g->device);
  cudaFree(const_cast<uint64_t*>(g->view.offsets));
  cudaFree(const_cast<uint32_t*>(g->view.neighbors));
  cudaFree(const_cast<uint64_t*>(g->original_ids));
  delete g;
}

kc_status kc_csr_dev_download(const kc_csr_dev* g, uint64_t* offsets, uint32_t* neighbors) {
  kcb::DeviceGuard device_guard;  // restore the caller's current device
  if (!g || !offsets) return KC_ERR_INVALID_ARGUMENT;
  GK(cudaSetDevice(g->device));
  GK(cudaMemcpy(offsets, g->view.offsets, ((size_t)g->view.n + 1) * 8, cudaMemcpyDeviceToHost));
  if (g->view.nnz) {
    if (!neighbors) return KC_ERR_INVALID_ARGUMENT;
    GK(cudaMemcpy(neighbors, g->view.neighbors, g->view.nnz * 4, cudaMemcpyDeviceToHost));
  }
  return KC_OK;
}

}  // extern "C"
