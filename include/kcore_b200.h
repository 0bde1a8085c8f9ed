/*
 * kcore_b200.h — C-ABI of the B200 (sm_100a) FastK coreness path.
 *
 * Drop-in boundary for the reference entry point
 *     kcore::EngineResult kcore::fastk_run(const Graph&, const FastKOptions&,
 *                                          const Instrumentation*)
 * declared at /root/reference/proj/include/kcore/fastk.hpp:46-47 and defined at
 * src/fastk.cpp:57-187.  Undirected CSR in (the reference Graph's
 * offsets()/neighbors(), include/kcore/graph.hpp:53-59,72-73), per-vertex
 * coreness out (CorenessResult::coreness, include/kcore/oracle.hpp:10-14),
 * RunReport counters (include/kcore/report.hpp:17-23) in kc_stats.
 *
 * Plain C types only; no exceptions cross this boundary.  Every call is
 * synchronous with respect to the host.  A kc_graph handle owns one CUDA
 * stream and its device buffers; it is not thread-safe, distinct handles are.
 * There is no CPU fallback: without a usable sm_100 device every entry point
 * that needs one returns KC_ERR_NO_DEVICE.
 */
#ifndef KCORE_B200_H
#define KCORE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KC_ABI_VERSION 1

typedef enum kc_status {
  KC_OK = 0,
  KC_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument (fastk.cpp:58-59) */
  KC_ERR_NO_DEVICE = 2,        /* no CUDA device / not sm_100 */
  KC_ERR_OUT_OF_MEMORY = 3,    /* reference: std::bad_alloc */
  KC_ERR_CUDA = 4,             /* any other CUDA runtime error */
  KC_ERR_NOT_CONVERGED = 5,    /* round cap exceeded (never expected) */
  KC_ERR_CALLBACK = 6,         /* an inspector callback asked to stop */
  KC_ERR_PARSE = 7,            /* reference: kcore::ParseError (graph.hpp:13-23) */
  KC_ERR_IO = 8                /* reference: kcore::IoError (graph.hpp:25-28) */
} kc_status;

/* Which vertices a round re-evaluates.  Every rule follows
 * the same Jacobi estimate trajectory (shadow_run, tests/test_fastk.cpp:41-92)
 * and reaches the same unique fixed point. */
typedef enum kc_rule {
  /* fastk_run's rule: droppers notify neighbours with extended_notify judged
   * on SETTLED estimates (fastk.cpp:156-163); notified vertices are
   * re-evaluated.  The RunReport counters (iterations, messages_sent,
   * messages_drained, tail_pops) equal the reference's, with or without
   * hybrid_tail (kc_tail.cu runs the reference's sequential tail). */
  KC_RULE_REFERENCE = 0,
  /* support counters: cnt[v] = #{w in N(v) : est_w >= est_v}; a drop of u
   * across est_w (the extended rule on settled values) decrements cnt[w], and
   * w is re-evaluated iff cnt[w] < est_w — i.e. only vertices that WILL drop
   * are evaluated.  messages_sent counts decrements. */
  KC_RULE_COUNTING = 1,
  KC_RULE_AUTO = 2 /* the fastest rule (currently KC_RULE_COUNTING) */
} kc_rule;

/* FastKOptions (include/kcore/fastk.hpp:12-22) plus GPU knobs. */
typedef struct kc_options {
  uint32_t threads;        /* validated >= 1 like the reference; advisory on GPU */
  uint32_t batch;          /* validated >= 1; hybrid switch threshold (fastk.hpp:29-31) */
  int32_t extended_notify; /* fastk.hpp:18 */
  int32_t hybrid_tail;     /* fastk.hpp:21: KC_RULE_REFERENCE finishes with the sequential
                              tail once fewer than `batch` vertices are active */
  int32_t rule;            /* kc_rule */
  uint32_t max_rounds;     /* 0 = default safety cap */
  uint32_t smem_cache;     /* ids whose estimates are cached in shared memory per
                              round; 0 = default, 0xffffffff = disabled */
  uint32_t reserved[8];    /* reserved[0]: debug flags (KC_DEBUG_*) */
} kc_options;

#define KC_DEBUG_PHASE_TIMES 1u /* record per-CTA per-round phase timestamps */
#define KC_DEBUG_LEGACY_COUNT 2u /* counting rule on the flag-frontier solver (A/B) */
#define KC_DEBUG_VERIFY_PERTURB 4u /* kc_verify self-test: candidate[u] += 1 for u % 997 == 0 */
#define KC_DEBUG_NO_PULL 8u /* counting rule: push notify in round 0 (A/B of the pull phase) */

/* RunReport (report.hpp:17-23) + work counters and timings. */
typedef struct kc_stats {
  uint64_t iterations;       /* executed rounds incl. the final quiescent one */
  uint64_t messages_sent;    /* notifications fired */
  uint64_t messages_drained; /* vertex evaluations (incl. isolated vertices in round 0) */
  uint64_t tail_pops;        /* queue pops of the sequential tail (fastk.cpp:28-55) */
  uint64_t e_scan;           /* adjacency entries scanned by evaluations */
  uint64_t v_eval;           /* evaluations of non-isolated vertices */
  uint64_t drops;            /* estimate decreases */
  uint64_t tail_rounds;      /* 1 if the sequential tail ran */
  uint32_t k_max;            /* CorenessResult::k_max (oracle.hpp:12) */
  uint32_t h_graph;          /* h-index of the degree sequence */
  double k_avg;              /* CorenessResult::k_avg (oracle.hpp:13) */
  float t_upload_ms;         /* H2D of the CSR (kc_graph_upload) */
  float t_prep_ms;           /* on-device relabel / layout (kc_graph_upload) */
  float t_solve_ms;          /* init -> converged estimates, CSR resident */
  float t_download_ms;       /* permute-back + D2H of the coreness */
  uint32_t kernel_launches;  /* this library's kernels launched by the call (solve path) */
  uint32_t pad0;
  uint64_t scan_evaluate;    /* entries streamed with a gather by evaluations (lists < rows) */
  uint64_t scan_notify;      /* entries streamed with a gather by notify / pull scans */
  uint32_t reserved[2];
} kc_stats;

/* A borrowed view of an undirected simple CSR: offsets has n+1 entries,
 * neighbors has offsets[n] entries, each row strictly increasing, mirrored
 * (graph.hpp:31-36).  offsets/neighbors are HOST pointers unless stated. */
typedef struct kc_csr_view {
  uint32_t n;
  uint64_t nnz;
  const uint64_t* offsets;
  const uint32_t* neighbors;
} kc_csr_view;

typedef struct kc_graph kc_graph;

/* Per-round observation hook (report.hpp:33-39): called at iteration 0
 * (degrees) and after every executed round, with the estimates in the
 * caller's vertex ids.  Return non-zero to abort (KC_ERR_CALLBACK). */
typedef int (*kc_inspector_fn)(void* user, uint64_t iteration, const uint32_t* estimates,
                               uint32_t n, uint64_t active_count);

const char* kc_status_str(kc_status s);
int kc_abi_version(void);
void kc_default_options(kc_options* opt);
/* Last CUDA / validation error message of this thread ("" if none). */
const char* kc_last_error(void);

/* Upload a host CSR to `device` and lay it out for the solver (degree-sorted
 * relabel, 32-bit offsets when nnz < 2^32).  Validates the view shape. */
kc_status kc_graph_upload(const kc_csr_view* csr, int device, kc_graph** out);
/* Same, but `csr` points at DEVICE memory on `device` (e.g. a graph built by
 * kc_gen_*); the source buffers are only read. */
kc_status kc_graph_upload_device(const kc_csr_view* csr, int device, kc_graph** out);
/* Upload with layout flags (KC_UPLOAD_*); `on_device` selects the pointer
 * space of `csr` as above. */
#define KC_UPLOAD_FORCE_OFF64 1u /* 64-bit device offsets even when nnz < 2^32 */
#define KC_UPLOAD_FORCE_EST32 2u /* 32-bit estimates even when H < 2^15 */
#define KC_UPLOAD_UNSORTED_ROWS 4u /* keep relabelled rows in input order: skips the
                                      on-chip row sorts of the layout (A/B and tests;
                                      solves are 20-30% slower without the sorted-row
                                      degree cuts) */
kc_status kc_graph_upload_ex(const kc_csr_view* csr, int device, int on_device, uint32_t flags,
                             kc_graph** out);
void kc_graph_free(kc_graph* g);
uint32_t kc_graph_n(const kc_graph* g);
uint64_t kc_graph_nnz(const kc_graph* g);
/* The upload / prep timings of the handle (ms). */
kc_status kc_graph_timings(const kc_graph* g, float* t_upload_ms, float* t_prep_ms);

/* Converge on the device; write coreness[n] (caller's ids) to HOST memory. */
kc_status kc_solve(kc_graph* g, const kc_options* opt, uint32_t* coreness, kc_stats* stats);
/* Same, coreness written to DEVICE memory (no D2H; CSR and result resident). */
kc_status kc_solve_device(kc_graph* g, const kc_options* opt, uint32_t* coreness_dev,
                          kc_stats* stats);
/* Instrumented run: one round per launch, estimates copied out after each. */
kc_status kc_solve_observed(kc_graph* g, const kc_options* opt, kc_inspector_fn fn,
                            void* user, uint32_t* coreness, kc_stats* stats);

/* Convergence trace computed on the device (record_iteration,
 * /root/reference/proj/src/report.cpp:7-18; IterationStat, report.hpp:14-17):
 * one row per iteration boundary (iteration 0 = degrees, then every executed
 * round, plus the tail boundary under the hybrid tail), mean_error = mean of
 * (estimate - truth), active_fraction = active / n.  Per boundary only a
 * 16-byte reduction result crosses PCIe, never the estimates.  The gap is
 * summed exactly, so the doubles equal the reference's.  `truth` is a HOST
 * array of n coreness values (caller ids); rows beyond trace_cap are counted
 * in *trace_rows but not written. */
typedef struct kc_iteration_stat {
  double mean_error;
  double active_fraction;
} kc_iteration_stat;
kc_status kc_solve_traced(kc_graph* g, const kc_options* opt, const uint32_t* truth,
                          kc_iteration_stat* trace, uint64_t trace_cap, uint64_t* trace_rows,
                          uint32_t* coreness, kc_stats* stats);

/* ---- independent checker on the device ------------ */
/* kcore::peel_coreness (/root/reference/proj/src/oracle.cpp:21-66) as a
 * separate device algorithm (level-synchronous parallel peel, kc_peel.cu;
 * shares nothing with the FastK kernels but the layout).  coreness[n] to
 * HOST memory (caller ids); stats: iterations = peel levels (k_max + 1),
 * k_max, k_avg, t_solve_ms = device time of the peel. */
kc_status kc_peel(kc_graph* g, uint32_t* coreness, kc_stats* stats);
/* kcore::verify (oracle.cpp:68-75) on the device: FastK under `opt` and the
 * device peel on the same handle, compared on the device.  *count = number of
 * mismatching vertices; the first min(cap, count) in ascending node id go to
 * out[] (Mismatch, oracle.hpp:23-27).  Only the mismatches cross PCIe. */
typedef struct kc_mismatch {
  uint32_t node;
  uint32_t candidate;
  uint32_t truth;
} kc_mismatch;
kc_status kc_verify(kc_graph* g, const kc_options* opt, kc_mismatch* out, uint64_t cap,
                    uint64_t* count);

/* kcore::sequential_tail (fastk.hpp:38-39, fastk.cpp:28-55) on the device:
 * est[n] and active[n] (HOST, caller ids) in/out; pops the active vertices
 * in ascending (estimate, id) order exactly like the reference's min-heap
 * (kc_tail.cu).  stats: tail_pops, messages_drained, messages_sent of this
 * call; every flag is 0 on return. */
kc_status kc_sequential_tail(kc_graph* g, uint32_t* est, uint8_t* active, int extended_notify,
                             kc_stats* stats);

/* One-shot drop-in: upload (sorted layout, rows sorted while each chunk of the
 * host-to-device copy is relabelled) + solve + download + free (fastk_run
 * semantics). */
kc_status kc_fastk_run(const kc_csr_view* csr, const kc_options* opt, uint32_t* coreness,
                       kc_stats* stats);

/* The library keeps the device memory of freed handles and finished one-shot
 * solves for the next call (its own stream-ordered pool, plus large blocks
 * recycled by exact size).  kc_trim_memory hands all of it back to the
 * driver (current device); live handles are not touched. */
kc_status kc_trim_memory(void);

/* Debug: the host-side copy of the pageable staging path (non-temporal AVX2
 * stores where the CPU has them, memcpy otherwise); needs no device.  For
 * tests. */
void kc_debug_host_copy(void* dst, const void* src, uint64_t bytes);

/* The CUDA stream a handle runs on (cudaStream_t as void*), for callers that
 * want to time kc_solve_device with their own events. */
void* kc_graph_stream(kc_graph* g);

/* Debug: per-round, per-CTA %globaltimer stamps of the solver phases
 * (round start, cache filled, HUGE, BIG, WARP, SUB, THREAD done, round end)
 * from the last solve run with KC_DEBUG_PHASE_TIMES; layout
 * [256 rounds][grid][8].  *grid receives the CTA count. */
kc_status kc_debug_phase_times(kc_graph* g, unsigned long long* out, uint64_t cap,
                               uint32_t* grid);

/* Debug: per-round counters of the last solve, 9 x uint64 per round
 * (evaluations, sum of their degrees, drops, notifications, entries streamed
 * by notify, entries streamed by evaluate, queue sizes HUGE|BIG<<32,
 * WARP|SUB<<32, THREAD) for the first `rounds` rounds (at most 4096). */
kc_status kc_debug_round_stats(kc_graph* g, unsigned long long* out, uint32_t rounds);
/* Measurement probe (debug): `reps` passes of the solver's inner operation
 * alone over every adjacency entry — the id stream plus one estimate gather
 * each, no cache — after a solve; *ms_per_pass = device time per pass. */
kc_status kc_debug_gather_probe(kc_graph* g, int reps, float* ms_per_pass);
/* Debug: the handle's on-device layout copied to HOST arrays — offsets
 * [n_nz + 1] (widened to 64 bit), neighbours [nnz] in the relabelled ids, and
 * perm [n] (new id -> caller id).  *n_nz receives the number of non-isolated
 * vertices, *rows_sorted whether every row is ascending.  Any output may be
 * NULL.  For layout tests. */
kc_status kc_debug_layout(kc_graph* g, uint64_t* offsets, uint32_t* neighbors, uint32_t* perm,
                          uint32_t* n_nz, int* rows_sorted);

/* ---- synthetic inputs (BASELINE.json configs; the "kcgen v1" spec) ------ */
/* Build one of the five configs (1..5) — or a scaled variant — directly on
 * the device: CSR with uint64 offsets and uint32 neighbours in DEVICE memory
 * owned by the returned kc_csr_dev (free with kc_csr_dev_free).
 *   cfg 1: ER G(n, m)          p0 = n,     p1 = m
 *   cfg 2: grid side x side    p0 = side
 *   cfg 3/5: R-MAT             p0 = scale, p1 = edge factor
 *   cfg 4: Chung-Lu            p0 = n,     p1 = cliques, p2 = clique size */
typedef struct kc_csr_dev {
  kc_csr_view view; /* device pointers */
  int device;
  const uint64_t* original_ids; /* DEVICE, n entries: dense id -> source id
                                   (Graph::original_id, graph.hpp:57); NULL =
                                   identity (generated graphs) */
} kc_csr_dev;
kc_status kc_gen_config(int cfg, uint64_t p0, uint64_t p1, uint64_t p2, uint64_t seed,
                        int device, kc_csr_dev** out);
void kc_csr_dev_free(kc_csr_dev* g);
/* ---- edge-list ingest ------------------------------ */
/* kcore::load_edge_list (graph.hpp:76-84, graph.cpp:22-80, 141-199) on the
 * device: "u v" per line, '#' comments and blank lines skipped, ids are
 * arbitrary unsigned 64-bit and densified to the ranks of the ascending
 * distinct ids, self-loops dropped, duplicates collapsed, rows sorted.
 * `text` is HOST memory.  On malformed input returns KC_ERR_PARSE and fills
 * *err (may be NULL) with the 1-based line and the reference's message. */
typedef struct kc_parse_error {
  uint64_t line;
  char what[160];
} kc_parse_error;
kc_status kc_load_edge_list(const char* text, uint64_t len, int device, kc_csr_dev** out,
                            kc_parse_error* err);
/* Same from a file, gzip-compressed or plain (zlib's gzopen, as the
 * reference's load_edge_list_file, graph.cpp:200-226); KC_ERR_IO with the
 * reference's message if it cannot be opened or read. */
kc_status kc_load_edge_list_file(const char* path, int device, kc_csr_dev** out,
                                 kc_parse_error* err);
/* Host copy of the original ids of a device CSR (n entries). */
kc_status kc_csr_dev_original_ids(const kc_csr_dev* g, uint64_t* ids);

/* Copy a device CSR to host buffers (offsets n+1, neighbours nnz). */
kc_status kc_csr_dev_download(const kc_csr_dev* g, uint64_t* offsets, uint32_t* neighbors);

#ifdef __cplusplus
}
#endif
#endif /* KCORE_B200_H */
