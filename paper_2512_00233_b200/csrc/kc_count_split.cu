// kc_count_split.cu — the counting-rule FastK solver's per-phase kernels
// (EVALUATE, NOTIFY + APPLY of one round per launch) for the large rounds:
// kc_count_impl.cuh compiled with the phase functions inlined, each kernel
// with its own register budget, KC_SPLIT_CTAS CTAs of KC_SPLIT_THREADS
// threads per SM.
#define KC_TU_SPLIT 1
#ifndef KC_SPLIT_THREADS
#define KC_SPLIT_THREADS 512
#endif
#define KC_SOLVE_THREADS KC_SPLIT_THREADS
#ifdef KC_SPLIT_STREAM_K
#define KC_STREAM_K KC_SPLIT_STREAM_K
#endif
#ifdef KC_SPLIT_STREAM_PREFETCH
#define KC_STREAM_PREFETCH KC_SPLIT_STREAM_PREFETCH
#endif
#ifdef KC_SPLIT_PHASE_INLINE
#define KC_PHASE_INLINE KC_SPLIT_PHASE_INLINE
#endif
#include "kc_count_impl.cuh"
