// kc_count.cu — the counting-rule FastK solver's persistent cooperative
// kernel (every round in one launch, grid barriers between the phases).
// The code is kc_count_impl.cuh; this unit compiles it with the persistent
// kernel's CTA shape and register budget.
#define KC_TU_SPLIT 0
#ifdef KC_COUNT_THREADS
#define KC_SOLVE_THREADS KC_COUNT_THREADS
#endif
#ifdef KC_COUNT_STREAM_K
#define KC_STREAM_K KC_COUNT_STREAM_K
#endif
#ifdef KC_COUNT_STREAM_PREFETCH
#define KC_STREAM_PREFETCH KC_COUNT_STREAM_PREFETCH
#endif
#ifdef KC_COUNT_PHASE_INLINE
#define KC_PHASE_INLINE KC_COUNT_PHASE_INLINE
#endif
#include "kc_count_impl.cuh"
