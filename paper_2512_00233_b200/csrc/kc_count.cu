// kc_count.cu — the counting-rule FastK solver's persistent cooperative
// kernel (every round in one launch, grid barriers between the phases).
// The code is kc_count_impl.cuh; this unit compiles it with the persistent
// kernel's CTA shape and register budget.
#define KC_TU_SPLIT 0
#include "kc_count_impl.cuh"
