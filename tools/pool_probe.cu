// pool_probe.cu — does the default stream-ordered pool reuse a block freed on
// a stream that was then destroyed, when the next allocation comes from a new
// stream?  (development probe for the e2e path; prints per-call host times)
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
static double ms(std::chrono::steady_clock::time_point a) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
}
int main() {
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  uint64_t keep = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  const size_t bytes = 1560ull << 20;
  for (int mode = 0; mode < 2; ++mode) {
    for (int i = 0; i < 4; ++i) {
      cudaStream_t s;
      cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      auto t = std::chrono::steady_clock::now();
      void* p = nullptr;
      cudaMallocAsync(&p, bytes, s);
      cudaMemsetAsync(p, 0, 16, s);
      cudaStreamSynchronize(s);
      double a = ms(t);
      cudaFreeAsync(p, s);
      cudaStreamSynchronize(s);
      if (mode == 0) cudaStreamDestroy(s);
      std::printf("mode %s iter %d: malloc+touch %.3f ms\n", mode ? "same-stream-kept" : "new-stream", i, a);
      if (mode == 1) cudaStreamDestroy(s);
    }
  }
  return 0;
}
