// kc_count_split.cu — the counting-rule FastK solver's per-phase kernels
// (EVALUATE, NOTIFY + APPLY of one round per launch) for the large rounds:
// kc_count_impl.cuh compiled with the phase functions inlined (no ABI calls,
// no callee-save spills), each kernel with its own register budget, and more
// resident warps than the persistent kernel: 896 threads (72 registers, 44%
// of the warp slots), 4-entry streams.  Sweeps over threads per CTA x CTAs
// per SM x stream depth x prefetch: profiles/r02/split_sweep{1,2,3}.txt
// (R-MAT 22 5.78 -> 5.48 ms, R-MAT 26 56.9 -> 54.6 ms on top of kc_count.cu's
// 4-entry streams).
#define KC_TU_SPLIT 1
#ifndef KC_SPLIT_THREADS
#define KC_SPLIT_THREADS 896
#endif
#define KC_SOLVE_THREADS KC_SPLIT_THREADS
#ifndef KC_SPLIT_CTAS
#define KC_SPLIT_CTAS 1
#endif
#ifndef KC_SPLIT_STREAM_K
#define KC_SPLIT_STREAM_K 4
#endif
#define KC_STREAM_K KC_SPLIT_STREAM_K
#ifdef KC_SPLIT_STREAM_PREFETCH
#define KC_STREAM_PREFETCH KC_SPLIT_STREAM_PREFETCH
#endif
#ifndef KC_SPLIT_PHASE_INLINE
#define KC_SPLIT_PHASE_INLINE 1
#endif
#define KC_PHASE_INLINE KC_SPLIT_PHASE_INLINE
#include "kc_count_impl.cuh"
