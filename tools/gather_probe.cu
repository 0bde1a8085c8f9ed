// gather_probe.cu — what one B200 sustains for the solver's inner operation:
// a 16-bit estimate gathered at a neighbour id (global: L2-resident or not;
// shared memory), with ids streamed from a CSR-like array.  Informs the
// solver's design: gathers/s per source and per locality.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_probe tools/gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

// ids: nnz u32 (streamed, 128-bit), est: u16 [n]; each thread sums est over its ids
template <int U>
__global__ void gather_global(const uint4* __restrict__ ids, const uint16_t* __restrict__ est,
                              size_t nvec, unsigned long long* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nvec;
       i += (size_t)gridDim.x * blockDim.x * U) {
    uint4 q[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      size_t j = i + (size_t)k * gridDim.x * blockDim.x;
      q[k] = j < nvec ? __ldcs(ids + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      acc += est[q[k].x] + est[q[k].y] + est[q[k].z] + est[q[k].w];
    }
  }
  if (acc == 0xdeadbeef) atomicAdd(out, acc);
}

// same with ids < cache_n served from shared memory
template <int U>
__global__ void gather_cached(const uint4* __restrict__ ids, const uint16_t* __restrict__ est,
                              size_t nvec, uint32_t cache_n, unsigned long long* out) {
  extern __shared__ uint16_t s[];
  for (uint32_t i = threadIdx.x; i < cache_n; i += blockDim.x) s[i] = est[i];
  __syncthreads();
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nvec;
       i += (size_t)gridDim.x * blockDim.x * U) {
    uint4 q[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      size_t j = i + (size_t)k * gridDim.x * blockDim.x;
      q[k] = j < nvec ? __ldcs(ids + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      uint32_t v[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) acc += v[e] < cache_n ? s[v[e]] : est[v[e]];
    }
  }
  if (acc == 0xdeadbeef) atomicAdd(out, acc);
}

// atomics: atomicSub on u32 counters at the ids
__global__ void atomic_scatter(const uint4* __restrict__ ids, uint32_t* cnt, size_t nvec) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nvec; i += (size_t)gridDim.x * blockDim.x) {
    uint4 q = __ldcs(ids + i);
    atomicSub(cnt + q.x, 1u); atomicSub(cnt + q.y, 1u); atomicSub(cnt + q.z, 1u); atomicSub(cnt + q.w, 1u);
  }
}

__global__ void stream_only(const uint4* __restrict__ ids, size_t nvec, unsigned long long* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nvec; i += (size_t)gridDim.x * blockDim.x) {
    uint4 q = __ldcs(ids + i);
    acc += q.x ^ q.y ^ q.z ^ q.w;
  }
  if (acc == 0xdeadbeef) atomicAdd(out, acc);
}

static uint64_t rng = 88172645463325252ull;
static inline uint64_t xs() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; }

int main(int argc, char** argv) {
  const size_t nnz = 128u << 20;   // 128 M entries (512 MB of ids)
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint16_t* est; uint32_t* ids; uint32_t* cnt; unsigned long long* out;
  const size_t nmax = 64u << 20;
  CK(cudaMalloc(&est, nmax * 2)); CK(cudaMalloc(&ids, nnz * 4)); CK(cudaMalloc(&cnt, nmax * 4));
  CK(cudaMalloc(&out, 8)); CK(cudaMemset(est, 1, nmax * 2)); CK(cudaMemset(cnt, 0xff, nmax * 4));
  std::vector<uint32_t> h(nnz);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char* what, auto&& launch) {
    launch(); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a); launch(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
    }
    printf("%-58s %8.3f ms  %7.1f G entries/s\n", what, best, nnz / (best * 1e-3) / 1e9);
  };
  // patterns: uniform over n (n = 4M: 8 MB est, L2-resident; 64M: 128 MB, not),
  // skewed (power-law-ish: id = n * u^3, low ids hot), sorted runs of 64 (rows)
  struct Pat { const char* name; uint32_t n; int kind; };
  Pat pats[] = {{"uniform n=4M", 4u << 20, 0}, {"uniform n=64M", 64u << 20, 0},
                {"skew u^3 n=4M", 4u << 20, 1}, {"skew u^3 n=64M", 64u << 20, 1},
                {"skew u^3 n=4M rows of 64 sorted", 4u << 20, 2},
                {"skew u^3 n=64M rows of 64 sorted", 64u << 20, 2}};
  for (const Pat& p : pats) {
    for (size_t i = 0; i < nnz; ++i) {
      double u = (xs() >> 11) * (1.0 / 9007199254740992.0);
      h[i] = p.kind == 0 ? (uint32_t)(xs() % p.n) : (uint32_t)(p.n * u * u * u);
    }
    if (p.kind == 2)
      for (size_t i = 0; i < nnz; i += 64) std::sort(h.begin() + i, h.begin() + i + 64);
    CK(cudaMemcpy(ids, h.data(), nnz * 4, cudaMemcpyHostToDevice));
    const size_t nvec = nnz / 4;
    printf("--- %s\n", p.name);
    for (int tpb : {256, 512, 1024}) {
      int blocks = sms * (2048 / tpb);
      char buf[128];
      snprintf(buf, sizeof buf, "global gather U=4 tpb=%d", tpb);
      timeit(buf, [&] { gather_global<4><<<blocks, tpb>>>((const uint4*)ids, est, nvec, out); });
    }
    timeit("global gather U=8 tpb=512 x4 blocks/SM", [&] { gather_global<8><<<sms * 4, 512>>>((const uint4*)ids, est, nvec, out); });
    for (uint32_t cn : {24576u, 65536u, 98304u}) {
      char buf[128];
      snprintf(buf, sizeof buf, "smem cache %u ids (%u KB), U=4 tpb=1024 1 blk/SM", cn, cn * 2 / 1024);
      CK(cudaFuncSetAttribute(gather_cached<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, cn * 2));
      timeit(buf, [&] { gather_cached<4><<<sms, 1024, cn * 2>>>((const uint4*)ids, est, nvec, cn, out); });
    }
    timeit("atomicSub scatter tpb=512", [&] { atomic_scatter<<<sms * 4, 512>>>((const uint4*)ids, cnt, nvec); });
    timeit("id stream only", [&] { stream_only<<<sms * 4, 512>>>((const uint4*)ids, nvec, out); });
  }
  return 0;
}
