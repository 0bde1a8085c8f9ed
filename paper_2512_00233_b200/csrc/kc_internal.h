// kc_internal.h — shared declarations between the C-ABI host layer
// (kc_api.cu), the solver (kc_solve.cu), the layout pass (kc_prep.cu) and the
// synthetic-graph builder (kc_gen.cu).  Not installed; not part of the ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kcb {

// Degree classes.  Vertex ids are relabelled by descending degree at upload
// (kc_prep.cu), so class c is the id range [cls_begin[c], cls_begin[c+1]).
enum Cls : int { C_HUGE = 0, C_BIG = 1, C_WARP = 2, C_SUB = 3, C_THREAD = 4, NCLS = 5 };
constexpr uint32_t DEG_THREAD_MAX = 8;   // THREAD: one thread per vertex, values in registers
constexpr uint32_t DEG_SUB_MAX = 64;     // SUB:    8-lane tile per vertex, 8 values per lane
constexpr uint32_t DEG_WARP_MAX = 1020;  // WARP:   warp per vertex, 32 values per lane
                                         //         (1020: a misaligned row still fits
                                         //          8 aligned 128-bit loads per lane)
constexpr uint32_t DEG_BIG_MAX = 8192;   // BIG:    warp per vertex, streamed, warp histogram
                                         // HUGE:   CTA per vertex, streamed, CTA histogram
#ifndef KC_SOLVE_THREADS
#define KC_SOLVE_THREADS 768
#endif
constexpr int SOLVE_THREADS = KC_SOLVE_THREADS;
constexpr int HIST_BINS = 4096;          // CTA windowed histogram (16 KB of shared memory)
constexpr int WARP_BINS = 256;           // per-warp windowed histogram (32 x 1 KB)
constexpr uint32_t EST16_LIMIT = 32768;  // 16-bit estimates need H < 2^15 (packed compares)
constexpr uint32_t ADJ_PAD = 8;          // neighbours allocated with 8 spare entries
                                         // (aligned 128-bit loads may read past a row)

// Activation rules (see include/kcore_b200.h kc_rule and SURVEY.md §7.3).
//   R_REF_*   notified vertices are re-evaluated (fastk.cpp:156-163), flags
//   R_COUNT   support counters: only vertices that will drop are evaluated
enum Rule : int { R_REF_EXT = 0, R_REF_PLAIN = 1, R_COUNT = 2 };

struct Ctl {                 // per round parity
  uint32_t grab[NCLS];       // evaluate phase cursors, per class
  uint32_t grab2[NCLS];      // notify phase cursors, per class
  uint32_t qcnt[NCLS];       // active vertices of each class (compacted queue)
  uint32_t lqn[2], lqc[2], lqd[2];  // counting solver: long-scan queue per phase —
                                    // appended, consumed, CTAs done appending
  uint32_t pad[3];
};

constexpr uint32_t STAT_SLOTS = 4096;  // rounds >= STAT_SLOTS-1 share the last slot

struct RoundStat {           // per round, accumulated with atomics
  unsigned long long evals;  // vertex evaluations
  unsigned long long escan;  // sum of degrees over evaluations (E_scan)
  unsigned long long drops, fires;
  unsigned long long nscan;  // entries streamed by the notify phase
  unsigned long long ascan;  // entries streamed by the evaluate phase (lists: < escan)
  unsigned long long q01, q23, q4;  // queue sizes: HUGE | BIG<<32, WARP | SUB<<32, THREAD
};

struct SolveBuffers {
  // layout (owned by kc_graph)
  const void* off;           // uint32 or uint64, n_nz + 1 (relabelled ids)
  const uint32_t* adj;       // relabelled neighbours (+ ADJ_PAD)
  const uint32_t* dcut;      // degree cut table [dcut_n] (kc_count.cu DegCut)
  uint32_t dcut_n;
  bool rows_sorted;          // neighbour rows sorted ascending
  uint32_t n_nz;
  uint32_t cls_begin[NCLS + 1];
  // est[0] = E, the round's snapshot; est[1] = N, the settled values (N == E
  // at every round start; the evaluate phase lowers N, the notify phase
  // copies droppers' N back into E)
  void* est[2];              // uint16 or uint32 [n_pad] each
  uint32_t* cnt;             // R_COUNT: #neighbours w with est_w >= est_v [n_pad]
  uint8_t* flag[2];          // frontier byte flags; flag[r & 1] = round r's active set
  uint32_t* queue;           // [n_pad] round r's active ids, class c segment at cls_begin[c]
  uint32_t* queue2;          // counting rule: the other round parity's queue [n_pad]
  uint32_t* radj;            // counting rule: relevant-neighbour lists [nnz + ADJ_PAD]
  uint32_t* rlen;            // counting rule: list lengths [n_pad]
  void* rthr;                // counting rule: list thresholds (EstT) [n_pad]
  uint32_t* lq[2];           // counting rule: long-scan queues per phase [cls_begin[1]]
  uint8_t* pflag;            // counting rule: round-1 droppers found by the pull phase [n_pad]
                             // (zero between solves: the compaction clears what it takes)
  uint32_t* spec;            // counting rule: next-round evaluations [3][n_pad16]
                             // (round tag, level, count), n_pad16 = n_nz rounded to 16
  Ctl* ctl;                  // [2]
  uint32_t* anydrop;         // [3] "some estimate dropped in round r" (r % 3)
  RoundStat* stats;          // [STAT_SLOTS]
  uint32_t* status;          // [0] rounds completed, [1] converged, [2] stopped for the tail,
                             // [3] est buffer holding the current state
  unsigned long long* prof;  // optional phase timestamps [PROF_ROUNDS][prof_ctas][PROF_PHASES]
  uint32_t prof_ctas;        // CTAs per profile row (the SM count)
  unsigned long long* tailc; // hybrid tail (kc_tail.cu): counters [TAIL_SLOTS]
};
// kc_tail.cu counters (tailc[]): pops (tail_pops), evaluations, notifications,
// drops, adjacency entries scanned, "the tail ran"; slot 6 is scratch.
enum TailSlot : int { TAIL_POPS = 0, TAIL_EVALS, TAIL_FIRES, TAIL_DROPS, TAIL_ESCAN, TAIL_RAN,
                      TAIL_SCRATCH, TAIL_SLOTS = 8 };
// status[] slots; ST_HANDOFF: the per-phase kernels (kc_count_split.cu) met a small round and
// left the rest to the persistent kernel
enum StatusSlot : int { ST_ROUNDS = 0, ST_CONVERGED = 1, ST_TAIL = 2, ST_BUF = 3, ST_HANDOFF = 4,
                        ST_SLOTS = 8 };
constexpr uint32_t PROF_ROUNDS = 256;
constexpr uint32_t PROF_PHASES = 8;

struct SolveConfig {
  int rule;
  uint32_t clamp_drop;       // max degree > H (round 0 changed in the reference)
  uint32_t cache_n;          // ids cached in shared memory
  uint32_t max_rounds;
  uint32_t tail_threshold;   // reference rule + hybrid_tail: stop the rounds when a round
                             // starts with fewer active vertices (the batch, fastk.hpp:29-31)
                             // and leave the rest to the sequential tail (0 = off)
  int num_sms;
  uint32_t pull;             // counting rule: round 0's notify + round 1's evaluate as one
                             // pull phase (kc_count.cu PULL) when the launch covers rounds 0-1
  uint32_t split_rounds;     // counting rule, whole solves: rounds 1 .. split_rounds run one
                             // kernel per phase (kc_count_split.cu) while they start with at
  uint32_t split_min;        // least split_min active vertices (0 rounds: off)
  uint32_t split_cache;      // the per-phase kernels keep the shared-memory estimate cache
};

// Launch rounds [r_begin, r_end) of the persistent solver on `stream`.
// est16: estimates are uint16 (else uint32); off64: offsets are uint64.
cudaError_t launch_rounds(const SolveBuffers& b, const SolveConfig& c, bool est16, bool off64,
                          uint32_t r_begin, uint32_t r_end, cudaStream_t stream);
// The counting-rule solver (kc_count.cu): same contract.
cudaError_t launch_count_rounds(const SolveBuffers& b, const SolveConfig& c, bool est16, bool off64,
                                uint32_t r_begin, uint32_t r_end, cudaStream_t stream);
// Rounds [r_lo, r_hi] one kernel per phase (kc_count_split.cu), queued without host round
// trips; they return at once after convergence or the hand-off (ST_HANDOFF).
cudaError_t launch_count_phases(const SolveBuffers& b, const SolveConfig& c, bool est16, bool off64,
                                uint32_t r_lo, uint32_t r_hi, bool skip_first_eval,
                                cudaStream_t stream);
// FastK's sequential tail (fastk.cpp:28-55) on one CTA, after the rounds
// kernel stopped for it (status[2] == 1) — or, with force_flags >= 0, from
// the active set in flag[force_flags] (observed mode).  No-op otherwise.
cudaError_t launch_tail(const SolveBuffers& b, const uint32_t* perm, bool est16, bool off64,
                        int ext, int force_flags, int num_sms, cudaStream_t s);
cudaError_t launch_count_init(const SolveBuffers& b, bool est16, bool off64, uint32_t h_graph,
                              cudaStream_t stream);
// Initialise estimates (min(deg, H)), round-0 frontier, counters.
cudaError_t launch_init(const SolveBuffers& b, bool est16, bool off64, uint32_t h_graph,
                        uint32_t max_rounds, cudaStream_t stream);
// Max shared memory the solver may use for the estimate cache (bytes).
size_t solver_cache_bytes_max();

// The caller's current device is restored when a C-ABI entry point returns
// (every entry point that selects the graph's device holds one).
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      prev = -1;
      cudaGetLastError();
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Stream-ordered device allocation from the library's own memory pool (one
// per device, created on first use), kept (release threshold = max) so
// repeated upload / solve / free cycles do not pay cudaMalloc / cudaFree —
// without changing the device's default pool, which co-resident libraries
// (PyTorch, CuPy) may use (kc_api.cu).
cudaError_t dmalloc(void** p, size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s);
template <typename T>
inline cudaError_t dmalloc_n(T** p, size_t count, cudaStream_t s) {
  return dmalloc(reinterpret_cast<void**>(p), (count ? count : 1) * sizeof(T), s);
}

// Independent device peel + verify (kc_peel.cu).
struct PeelBuffers {
  const void* off;           // layout offsets (uint32 or uint64)
  const uint32_t* adj;
  uint32_t n_nz;
  uint32_t* deg;             // [n_nz] remaining degree
  uint32_t* core;            // [n_nz] peel level (layout ids)
  uint32_t* rem[2];          // [n_nz] remaining lists
  uint32_t* fr[2];           // [n_nz] frontier lists (warp rows)
  uint32_t* frb[2];          // [n_nz] frontier lists (grid rows)
  void* ctl;                 // peel_ctl_bytes()
};
size_t peel_ctl_bytes();
cudaError_t launch_peel(const PeelBuffers& b, bool off64, int num_sms, cudaStream_t s);
cudaError_t launch_peel_out(const PeelBuffers& b, const uint32_t* perm, uint32_t n, uint32_t* out,
                            int num_sms, cudaStream_t s);
cudaError_t launch_mismatch_count(const uint32_t* a, const uint32_t* b, uint32_t n,
                                  unsigned long long* count, int num_sms, cudaStream_t s);
cudaError_t launch_mismatch_list(const uint32_t* cand, const uint32_t* truth, uint32_t n,
                                 uint32_t* ids, uint32_t cap, cudaStream_t s);

// On-device layout of an uploaded CSR (kc_prep.cu).
struct PrepOut {
  void* off;        // OffT [n_nz + 1]
  uint32_t* adj;    // [nnz]
  uint32_t* perm;   // [n] new id -> caller id
  uint32_t* dcut;   // dcut[x] = #{ids of degree >= x}, x <= max_degree + 1
  bool rows_sorted; // rows sorted ascending (dcut then also splits every row)
  uint32_t n_nz;    // non-isolated vertices (ids [0, n_nz))
  uint32_t h_graph; // h-index of the degree sequence
  uint32_t max_degree;
  uint32_t cls_begin[NCLS + 1];
  bool off64;
  bool invalid;     // the input is not a CSR (offsets not 0..nnz non-decreasing, or a
                    // neighbour id >= n): nothing was laid out
};
// Pipelined upload (host CSR): the neighbours arrive in k chunks of old row
// ids [old_lo[c], old_lo[c+1]) (host array, k + 1 entries), chunk c complete
// when ready[c] fires; the layout relabels each chunk's rows as it lands.
struct AdjFeed {
  int k;
  const uint32_t* old_lo;
  const cudaEvent_t* ready;
  // staged (pageable) uploads: ready[c] is recorded by a host thread; the
  // layout first blocks until it has been (host_wait(ctx, c)), then waits on it
  void (*host_wait)(void* ctx, int c) = nullptr;
  void* ctx = nullptr;
};

// Pageable host memory (kc_stage.cu): copies through pinned staging slots
// filled by host threads while the copy engine drains the previous slot.
bool is_pageable(const void* p);
void host_copy(void* dst, const void* src, size_t n);  // kc_hostcopy.cpp: non-temporal stores
cudaError_t staged_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s);
cudaError_t staged_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s);
cudaError_t prep_layout(const uint64_t* off, const uint32_t* adj, uint32_t n, uint64_t nnz,
                        bool force_off64, bool sort_rows, cudaStream_t s, PrepOut* out,
                        const AdjFeed* feed = nullptr);

}  // namespace kcb
