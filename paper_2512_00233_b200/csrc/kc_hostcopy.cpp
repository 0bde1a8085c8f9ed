// kc_hostcopy.cpp — the host-side copy of the pageable staging path
// (kc_stage.cu): caller memory <-> pinned ring slots.  A plain memcpy reads
// the destination lines before overwriting them (write-allocate); with
// non-temporal stores the copy moves 2 bytes of DRAM traffic per byte instead
// of 3, next to the DMA engine reading the same slots.  AVX2 at run time
// (__builtin_cpu_supports), memcpy otherwise.  KC_STAGE_NT=0 disables it.
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <immintrin.h>

namespace kcb {

namespace {

__attribute__((target("avx2"))) void nt_copy_avx2(char* dst, const char* src, size_t n) {
  // head: up to the first 32-byte boundary of dst
  const size_t head = (32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31;
  if (head) {
    const size_t h = head < n ? head : n;
    std::memcpy(dst, src, h);
    dst += h;
    src += h;
    n -= h;
  }
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    _mm_prefetch(src + i + 1024, _MM_HINT_NTA);
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
    const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
  }
  _mm_sfence();
  if (i < n) std::memcpy(dst + i, src + i, n - i);
}

bool use_nt() {
  static const bool on = [] {
    const char* v = std::getenv("KC_STAGE_NT");
    if (v && *v == '0') return false;
    return __builtin_cpu_supports("avx2") != 0;
  }();
  return on;
}

}  // namespace

void host_copy(void* dst, const void* src, size_t n) {
  if (n >= (64u << 10) && use_nt())
    nt_copy_avx2(static_cast<char*>(dst), static_cast<const char*>(src), n);
  else
    std::memcpy(dst, src, n);
}

}  // namespace kcb
