// kc_count.cu — the counting-rule FastK solver's persistent cooperative
// kernel (every round in one launch, grid barriers between the phases).
// The code is kc_count_impl.cuh; this unit compiles it with the persistent
// kernel's CTA shape and register budget: 768 threads, 4-entry streams (one
// 128-bit id load per lane per step instead of two: the scans are chains of
// dependent round trips per vertex, and the registers the second load and its
// four gathers held are worth more as spill-free code — R-MAT 22 6.26 -> 5.78
// ms, R-MAT 26 60.5 -> 56.9 ms, profiles/r02/split_sweep3.txt).
#define KC_TU_SPLIT 0
#ifdef KC_COUNT_THREADS
#define KC_SOLVE_THREADS KC_COUNT_THREADS
#endif
#ifndef KC_COUNT_STREAM_K
#define KC_COUNT_STREAM_K 4
#endif
#define KC_STREAM_K KC_COUNT_STREAM_K
#ifdef KC_COUNT_STREAM_PREFETCH
#define KC_STREAM_PREFETCH KC_COUNT_STREAM_PREFETCH
#endif
#ifdef KC_COUNT_PHASE_INLINE
#define KC_PHASE_INLINE KC_COUNT_PHASE_INLINE
#endif
#include "kc_count_impl.cuh"
