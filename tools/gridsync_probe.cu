// gridsync_probe.cu — cost of cooperative_groups grid.sync() on the full
// B200 (148 CTAs x 768 threads) vs a hand-rolled sense-reversal barrier
// (development probe: what a round's two barriers cost the solver).
#include <cooperative_groups.h>
#include <chrono>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(768, 1) cg_sync(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

__device__ unsigned int g_count = 0;
__device__ volatile unsigned int g_gen = 0;
__global__ void __launch_bounds__(768, 1) my_sync(int iters, unsigned long long* out) {
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned int gen = g_gen;
      __threadfence();
      if (atomicAdd(&g_count, 1u) == gridDim.x - 1) {
        g_count = 0;
        __threadfence();
        g_gen = gen + 1;
      } else {
        while (g_gen == gen) {}
      }
      __threadfence();
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  int iters = 2000;
  for (int k = 0; k < 2; ++k) {
    void* args[] = {&iters, &d};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel(k == 0 ? (void*)cg_sync : (void*)my_sync, sms, 768, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("%s: %.3f us per barrier (%d CTAs)\n", k == 0 ? "cg grid.sync" : "sense barrier",
           ms * 1000.f / iters, sms);
  }
  return 0;
}
