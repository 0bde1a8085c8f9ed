// kc_internal.h — shared declarations between the C-ABI host layer
// (kc_api.cu), the solver (kc_solve.cu), the layout pass (kc_prep.cu) and the
// synthetic-graph builder (kc_gen.cu).  Not installed; not part of the ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kcb {

// Degree classes.  Vertex ids are relabelled by descending degree at upload
// (kc_prep.cu), so class c is the id range [cls_begin[c], cls_begin[c+1]).
enum Cls : int { C_HUGE = 0, C_BLOCK = 1, C_WARP = 2, C_SUB = 3, C_THREAD = 4, NCLS = 5 };
constexpr uint32_t DEG_THREAD_MAX = 8;     // one thread per vertex, values in registers
constexpr uint32_t DEG_SUB_MAX = 64;       // 8-lane tile per vertex, 8 values per lane
constexpr uint32_t DEG_WARP_MAX = 1024;    // warp per vertex, 32 values per lane
constexpr uint32_t DEG_BLOCK_MAX = 32768;  // CTA per vertex, windowed histogram
                                           // (> DEG_BLOCK_MAX: CTA per vertex, same code)
constexpr int SOLVE_THREADS = 1024;
constexpr int HIST_BINS = 4096;            // windowed histogram, 16 KB of shared memory

// Activation rules (see include/kcore_b200.h kc_rule and SURVEY.md §7.3).
enum Rule : int { R_REF_EXT = 0, R_REF_PLAIN = 1, R_SNAP_EXT = 2, R_SNAP_PLAIN = 3 };

struct Ctl {                 // per round parity: work-grab cursors + drop count
  uint32_t grab[NCLS];
  uint32_t ndrops;
  uint32_t pad[2];
};

constexpr uint32_t STAT_SLOTS = 4096;  // rounds >= STAT_SLOTS-1 share the last slot

struct RoundStat {           // per round, accumulated with atomics
  unsigned long long evals, escan, drops, fires, frontier, active_after, tail, pad;
};

struct SolveBuffers {
  // layout (owned by kc_graph)
  const void* off;           // uint32 or uint64, n_nz + 1 (relabelled ids)
  const uint32_t* adj;       // relabelled neighbours
  void* est;                 // uint16 or uint32 [n_nz]
  uint32_t n_nz;
  uint32_t cls_begin[NCLS + 1];
  // frontier state
  uint32_t* queue[2];        // [n_nz] each, class c segment at cls_begin[c]
  uint32_t* qcnt;            // [2][NCLS]
  uint32_t* bm[2];           // dedup bitmaps, (n_nz + 31) / 32 words
  uint32_t* drop_u;          // [n_nz]
  void* drop_t;              // EstT [n_nz]
  void* drop_old;            // EstT [n_nz]
  Ctl* ctl;                  // [2]
  RoundStat* stats;          // [STAT_SLOTS]
  uint32_t* status;          // [0] rounds completed, [1] converged, [2] tail rounds
};

struct SolveConfig {
  int rule;
  uint32_t cache_n;          // ids cached in shared memory
  uint32_t max_rounds;
  uint32_t tail_threshold;   // frontier size below which one CTA finishes (0 = off)
  int num_sms;
};

// Launch rounds [r_begin, r_end) of the persistent solver on `stream`.
// est16: estimates are uint16 (else uint32); off64: offsets are uint64.
cudaError_t launch_rounds(const SolveBuffers& b, const SolveConfig& c, bool est16, bool off64,
                          uint32_t r_begin, uint32_t r_end, cudaStream_t stream);
// Initialise estimates (min(deg, H)), round-0 frontier, counters.
cudaError_t launch_init(const SolveBuffers& b, bool est16, bool off64, uint32_t h_graph,
                        uint32_t max_rounds, cudaStream_t stream);
// Max shared memory the solver may use for the estimate cache (bytes).
size_t solver_cache_bytes_max();

// On-device layout of an uploaded CSR (kc_prep.cu).
struct PrepOut {
  void* off;        // OffT [n_nz + 1]
  uint32_t* adj;    // [nnz]
  uint32_t* perm;   // [n] new id -> caller id
  uint32_t n_nz;    // non-isolated vertices (ids [0, n_nz))
  uint32_t h_graph; // h-index of the degree sequence
  uint32_t cls_begin[NCLS + 1];
  bool off64;
};
cudaError_t prep_layout(const uint64_t* off, const uint32_t* adj, uint32_t n, uint64_t nnz,
                        bool force_off64, cudaStream_t s, PrepOut* out);

}  // namespace kcb
