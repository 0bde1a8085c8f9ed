// kc_stage.cu — host<->device copies of PAGEABLE host memory through pinned
// staging buffers.
//
// The reference's Graph keeps its CSR in std::vector (graph.hpp:72-73):
// pageable memory, which the CUDA driver copies through its own small
// bounce buffers at ~11 GB/s on the B200 box (profiles/r02/bench_*: 49.5 ms
// for R-MAT 22's 547 MB).  Here the bytes are copied into a ring of pinned
// slots by a few host threads (memcpy bandwidth scales with threads) while
// the copy engine drains the previous slot, so the PCIe link (~55 GB/s
// pinned) rather than one bounce buffer bounds the upload.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <cstdlib>
#include <thread>
#include <vector>

#include "kc_internal.h"

namespace kcb {
namespace {

constexpr size_t SLOT_BYTES = 32u << 20;  // one staging slot
constexpr int NSLOT = 4;                  // ring depth

// A fixed set of worker threads that split one memcpy between them.
class CopyPool {
 public:
  CopyPool() {
    unsigned hc = std::thread::hardware_concurrency();
    // measured on the 16-core B200 host (scripts/stage_ab.sh): R-MAT 26's 8.95 GB stage in
    // 333 / 275 / 221 / 200 ms with 4 / 8 / 12 / 16 threads (R-MAT 22: 19.7 / 15.6 / 16.3 / 16.3)
    nthreads_ = std::max(1u, std::min(16u, hc ? hc : 4u));
    if (const char* v = std::getenv("KC_STAGE_THREADS"))  // development override
      if (*v) nthreads_ = std::max(1u, std::min(64u, (unsigned)std::strtoul(v, nullptr, 10)));
    for (unsigned i = 1; i < nthreads_; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  // dst[0, n) = src[0, n), split over the pool (the caller takes part 0)
  void copy(void* dst, const void* src, size_t n) {
    if (n < (1u << 20) || nthreads_ == 1) {
      host_copy(dst, src, n);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(m_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      n_ = n;
      pending_ = nthreads_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    part(0);
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void part(unsigned i) {
    const size_t per = (n_ + nthreads_ - 1) / nthreads_;
    const size_t a = std::min(n_, per * i), b = std::min(n_, a + per);
    if (b > a) host_copy(dst_ + a, src_ + a, b - a);
  }
  void loop(unsigned i) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      part(i);
      {
        std::lock_guard<std::mutex> lk(m_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  unsigned nthreads_ = 1;
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  uint64_t gen_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_ = 0;
  unsigned pending_ = 0;
};

// The pinned ring, per process (one upload at a time uses it: `mu`).
struct Ring {
  std::mutex mu;
  void* slot[NSLOT] = {};
  cudaEvent_t done[NSLOT] = {};
  bool ready = false;
  CopyPool* pool = nullptr;
  cudaError_t init() {
    if (ready) return cudaSuccess;
    for (int i = 0; i < NSLOT; ++i) {
      cudaError_t e = cudaHostAlloc(&slot[i], SLOT_BYTES, cudaHostAllocPortable);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    pool = new CopyPool();
    ready = true;
    return cudaSuccess;
  }
};

Ring& ring() {
  static Ring* r = new Ring();  // process lifetime (no teardown-order issues)
  return *r;
}

}  // namespace

bool is_pageable(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

cudaError_t staged_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  Ring& r = ring();
  std::lock_guard<std::mutex> lk(r.mu);
  cudaError_t e = r.init();
  if (e != cudaSuccess) return e;
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  static int next = 0;  // ring position persists across calls
  for (size_t off = 0; off < bytes; off += SLOT_BYTES) {
    const size_t n = std::min(SLOT_BYTES, bytes - off);
    const int k = next;
    next = (next + 1) % NSLOT;
    e = cudaEventSynchronize(r.done[k]);  // the slot's previous DMA has drained
    if (e != cudaSuccess) return e;
    r.pool->copy(r.slot[k], in + off, n);
    e = cudaMemcpyAsync(out + off, r.slot[k], n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaEventRecord(r.done[k], s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t staged_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  Ring& r = ring();
  std::lock_guard<std::mutex> lk(r.mu);
  cudaError_t e = r.init();
  if (e != cudaSuccess) return e;
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  // DMA slot k while the host drains slot k-1 into the caller's memory
  const size_t nchunk = (bytes + SLOT_BYTES - 1) / SLOT_BYTES;
  for (size_t c = 0; c < nchunk + 1; ++c) {
    if (c < nchunk) {
      const int k = (int)(c % NSLOT);
      const size_t off = c * SLOT_BYTES, n = std::min(SLOT_BYTES, bytes - off);
      e = cudaEventSynchronize(r.done[k]);
      if (e == cudaSuccess) e = cudaMemcpyAsync(r.slot[k], in + off, n, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaEventRecord(r.done[k], s);
      if (e != cudaSuccess) return e;
    }
    if (c > 0) {
      const size_t p = c - 1;
      const int k = (int)(p % NSLOT);
      const size_t off = p * SLOT_BYTES, n = std::min(SLOT_BYTES, bytes - off);
      e = cudaEventSynchronize(r.done[k]);
      if (e != cudaSuccess) return e;
      r.pool->copy(out + off, r.slot[k], n);
    }
  }
  return cudaSuccess;
}

}  // namespace kcb
