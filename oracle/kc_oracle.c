/*
 * kc_oracle.c — CPU restatement of the reference's FastK coreness path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library, and
 * only as the checker or the reported CPU baseline.  The product path
 * (paper_2512_00233_b200, libkcore_b200.so) never links or calls it.
 *
 * Parity is pinned two ways (see tests/test_oracle.py):
 *   - against the reference compiled from /root/reference by oracle/Makefile
 *     (oracle/_ref/libkcore_ref.so): peel_coreness, compute_index and the full
 *     fastk_run counters on the same graphs;
 *   - against the known-answer tests of the reference's own suites
 *     (tests/test_kernel.cpp:30-44, tests/test_fastk.cpp:118-179,
 *     tests/test_oracle.cpp:43-67, tests/test_bench.cpp:166-176), replayed in
 *     tests/golden/ by oracle/make_golden.py.
 *
 * Everything here is plain C11 + OpenMP.  Each function cites the reference
 * file:line it restates (paths relative to /root/reference/proj).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <omp.h>

#define KCO_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Seeded counter-based PRNG ("kcgen v1").  Not from the reference: the      */
/* reference measures on SNAP files; BASELINE.json's synthetic configs stand */
/* in for them.  The same spec is implemented independently on the GPU      */
/* (paper_2512_00233_b200/csrc/kc_gen.cu) and the two are checked equal.     */
/* ------------------------------------------------------------------------ */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(seed * 0x9E3779B97F4A7C15ULL + mix64(stream + 0x632BE59BD9B4E019ULL));
}
static inline uint64_t rng_at(uint64_t key, uint64_t ctr) {
  return mix64(key + ctr * 0x9E3779B97F4A7C15ULL);
}
/* floor(x * n / 2^32) for a 32-bit uniform x: exact integer range reduction */
static inline uint32_t range32(uint32_t x, uint32_t n) {
  return (uint32_t)(((uint64_t)x * (uint64_t)n) >> 32);
}
static inline uint64_t mulhi64(uint64_t a, uint64_t b) {
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
}

KCO_API uint64_t kco_rng_at(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return rng_at(stream_key(seed, stream), ctr);
}

/* Bijective seeded hash on [0, 2^bits): the "seeded shuffle" of R-MAT ids.  */
static inline uint32_t perm_bits(uint32_t x, uint32_t bits, uint64_t key) {
  const uint32_t mask = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
  const uint32_t half = bits / 2 ? bits / 2 : 1;
  for (int r = 0; r < 4; ++r) {
    uint64_t k = rng_at(key, (uint64_t)r);
    x = (uint32_t)((x * ((uint32_t)k | 1u) + (uint32_t)(k >> 32)) & mask);
    x ^= x >> half;
    x &= mask;
  }
  return x;
}
KCO_API uint32_t kco_perm_bits(uint32_t x, uint32_t bits, uint64_t seed) {
  return perm_bits(x, bits, stream_key(seed, 9));
}

/* Config 1: G(n, m) — m uniform endpoint pairs; loops/dups removed later. */
KCO_API void kco_gen_er(uint32_t n, uint64_t m, uint64_t seed, uint32_t* pairs) {
  const uint64_t key = stream_key(seed, 1);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)m; ++i) {
    uint64_t r = rng_at(key, (uint64_t)i);
    pairs[2 * i] = range32((uint32_t)r, n);
    pairs[2 * i + 1] = range32((uint32_t)(r >> 32), n);
  }
}

/* Config 2: side x side grid, id = r*side + c.  Per vertex 3 candidate
 * edges (right p, down p, diagonal (r+1,c+1) p_diag); a rejected candidate is
 * emitted as a self-loop, which CSR construction drops (graph.cpp:93,102). */
KCO_API void kco_gen_grid(uint32_t side, uint32_t p_keep_q32, uint32_t p_diag_q32,
                          uint64_t seed, uint32_t* pairs) {
  const uint64_t k1 = stream_key(seed, 2), k2 = stream_key(seed, 3);
  const uint64_t n = (uint64_t)side * side;
#pragma omp parallel for schedule(static)
  for (int64_t id = 0; id < (int64_t)n; ++id) {
    uint32_t r = (uint32_t)(id / side), c = (uint32_t)(id % side);
    uint64_t h = rng_at(k1, (uint64_t)id), h2 = rng_at(k2, (uint64_t)id);
    uint32_t u = (uint32_t)id;
    uint32_t* p = pairs + 6 * id;
    p[0] = u; p[1] = (c + 1 < side && (uint32_t)h < p_keep_q32) ? u + 1 : u;
    p[2] = u; p[3] = (r + 1 < side && (uint32_t)(h >> 32) < p_keep_q32) ? u + side : u;
    p[4] = u; p[5] = (r + 1 < side && c + 1 < side && (uint32_t)h2 < p_diag_q32) ? u + side + 1 : u;
  }
}

/* Configs 3/5: R-MAT, `scale` quadrant draws per pair with integer
 * thresholds a, a+b, a+b+c (all scaled by 2^32), ids then permuted. */
KCO_API void kco_gen_rmat(uint32_t scale, uint64_t m, uint32_t ta, uint32_t tab, uint32_t tabc,
                          uint64_t seed, uint32_t* pairs) {
  const uint64_t key = stream_key(seed, 4), pkey = stream_key(seed, 9);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)m; ++i) {
    uint32_t u = 0, v = 0;
    uint64_t h = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      if ((l & 1) == 0) h = rng_at(key, (uint64_t)i * 16 + l / 2);
      uint32_t x = (l & 1) ? (uint32_t)(h >> 32) : (uint32_t)h;
      uint32_t bu = x >= tab, bv = (x >= ta && x < tab) || x >= tabc;
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    pairs[2 * i] = perm_bits(u, scale, pkey);
    pairs[2 * i + 1] = perm_bits(v, scale, pkey);
  }
}

/* Config 4: Chung–Lu weights.  w_i = x_min * (1-U_i)^(-1/(gamma-1)),
 * truncated at w_max, x_min bisected so mean(w) = mean_target; weights are
 * quantized to integers W_i = llround(w_i * 1024) so sampling is exact
 * integer arithmetic on both CPU and GPU.  Returns x_min. */
KCO_API double kco_chunglu_weights(uint32_t n, double gamma, double mean_target, double w_max,
                                   uint64_t seed, uint64_t* wq) {
  const uint64_t key = stream_key(seed, 5);
  double* g = (double*)malloc(sizeof(double) * (n ? n : 1));
  const double ex = -1.0 / (gamma - 1.0);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    double U = (double)(rng_at(key, (uint64_t)i) >> 11) * 0x1.0p-53;
    g[i] = pow(1.0 - U, ex);
  }
  /* deterministic chunked mean (fixed chunk order, independent of threads) */
  const int64_t CH = 1 << 16;
  const int64_t nch = ((int64_t)n + CH - 1) / CH;
  double* part = (double*)malloc(sizeof(double) * (nch ? nch : 1));
  double lo = 0.0, hi = mean_target;
  for (int it = 0; it < 100; ++it) {
    double x = 0.5 * (lo + hi);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nch; ++c) {
      double s = 0.0;
      int64_t e = (c + 1) * CH < (int64_t)n ? (c + 1) * CH : (int64_t)n;
      for (int64_t i = c * CH; i < e; ++i) {
        double w = x * g[i];
        s += w < w_max ? w : w_max;
      }
      part[c] = s;
    }
    double s = 0.0;
    for (int64_t c = 0; c < nch; ++c) s += part[c];
    if (s / (double)n < mean_target) lo = x; else hi = x;
  }
  double xm = 0.5 * (lo + hi);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    double w = xm * g[i];
    w = w < w_max ? w : w_max;
    wq[i] = (uint64_t)llround(w * 1024.0);
  }
  free(part);
  free(g);
  return xm;
}

/* Chung–Lu pairs: endpoints drawn with P(i) ∝ W_i by inverse CDF over the
 * exclusive prefix sums `pre` (length n+1), then `cliques` planted cliques of
 * `csize` uniformly chosen vertices (all pairs).  pairs has
 * 2*(m + cliques*csize*(csize-1)/2) slots. */
static inline uint32_t cdf_search(const uint64_t* pre, uint32_t n, uint64_t target) {
  /* largest i with pre[i] <= target, i in [0, n) */
  uint32_t lo = 0, hi = n; /* invariant: pre[lo] <= target < pre[hi] */
  while (hi - lo > 1) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (pre[mid] <= target) lo = mid; else hi = mid;
  }
  return lo;
}
KCO_API void kco_gen_chunglu(uint32_t n, const uint64_t* pre, uint64_t m, uint32_t cliques,
                             uint32_t csize, uint64_t seed, uint32_t* pairs) {
  const uint64_t key = stream_key(seed, 6), ckey = stream_key(seed, 7);
  const uint64_t total = pre[n];
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)m; ++i) {
    pairs[2 * i] = cdf_search(pre, n, mulhi64(rng_at(key, 2 * (uint64_t)i), total));
    pairs[2 * i + 1] = cdf_search(pre, n, mulhi64(rng_at(key, 2 * (uint64_t)i + 1), total));
  }
  const uint64_t per = (uint64_t)csize * (csize - 1) / 2;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < (int64_t)cliques; ++c) {
    uint32_t* out = pairs + 2 * (m + (uint64_t)c * per);
    uint64_t k = 0;
    for (uint32_t a = 0; a < csize; ++a) {
      uint32_t ua = range32((uint32_t)rng_at(ckey, (uint64_t)c * csize + a), n);
      for (uint32_t b = a + 1; b < csize; ++b) {
        uint32_t ub = range32((uint32_t)rng_at(ckey, (uint64_t)c * csize + b), n);
        out[2 * k] = ua;
        out[2 * k + 1] = ub;
        ++k;
      }
    }
  }
}

/* ------------------------------------------------------------------------ */
/* CSR construction — restates build_csr, src/graph.cpp:85-128: drop        */
/* self-loops, count both directions, scatter, sort each row, drop          */
/* duplicates, compact.  Parallel here, but the output is a pure function of */
/* the edge multiset, like the reference's.  `nbr` must hold 2*m entries.    */
/* Returns nnz.                                                             */
/* ------------------------------------------------------------------------ */
static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}
static void sort_u32(uint32_t* a, uint64_t len) {
  if (len < 2) return;
  if (len <= 32) { /* insertion sort for short rows */
    for (uint64_t i = 1; i < len; ++i) {
      uint32_t x = a[i];
      uint64_t j = i;
      while (j > 0 && a[j - 1] > x) { a[j] = a[j - 1]; --j; }
      a[j] = x;
    }
    return;
  }
  qsort(a, len, sizeof(uint32_t), cmp_u32);
}

KCO_API uint64_t kco_build_csr(uint32_t n, const uint32_t* pairs, uint64_t m, uint64_t* off,
                               uint32_t* nbr) {
  uint64_t* cnt = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)m; ++i) {
    uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    if (u == v) continue;
#pragma omp atomic
    cnt[u + 1]++;
#pragma omp atomic
    cnt[v + 1]++;
  }
  for (uint64_t i = 1; i <= n; ++i) cnt[i] += cnt[i - 1];
  uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
  memcpy(cur, cnt, sizeof(uint64_t) * ((size_t)n + 1));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)m; ++i) {
    uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    if (u == v) continue;
    uint64_t pu, pv;
#pragma omp atomic capture
    pu = cur[u]++;
#pragma omp atomic capture
    pv = cur[v]++;
    nbr[pu] = v;
    nbr[pv] = u;
  }
  /* sort + dedup each row in place; record kept length */
  uint64_t* keep = cur; /* reuse: keep[u] = unique count of row u */
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t u = 0; u < (int64_t)n; ++u) {
    uint32_t* row = nbr + cnt[u];
    uint64_t len = cnt[u + 1] - cnt[u];
    sort_u32(row, len);
    uint64_t w = 0;
    for (uint64_t i = 0; i < len; ++i)
      if (i == 0 || row[i] != row[i - 1]) row[w++] = row[i];
    keep[u] = w;
  }
  off[0] = 0;
  for (uint64_t u = 0; u < n; ++u) off[u + 1] = off[u] + keep[u];
  /* compact rows leftwards (off[u] <= cnt[u]); sequential in row order */
  for (uint64_t u = 0; u < n; ++u) {
    if (off[u] != cnt[u]) memmove(nbr + off[u], nbr + cnt[u], sizeof(uint32_t) * keep[u]);
  }
  uint64_t nnz = off[n];
  free(cnt);
  free(cur);
  return nnz;
}

/* ------------------------------------------------------------------------ */
/* Capped h-index — restates compute_index_over, include/kcore/kernel.hpp:27-42: */
/* histogram of min(e, cap) into cap+1 bins, suffix scan from cap down.      */
/* ------------------------------------------------------------------------ */
KCO_API uint32_t kco_compute_index(const uint32_t* est, uint64_t count, uint32_t cap) {
  if (cap == 0) return 0; /* kernel.hpp:30 */
  uint32_t* counts = (uint32_t*)calloc((size_t)cap + 1, sizeof(uint32_t));
  for (uint64_t i = 0; i < count; ++i) { /* kernel.hpp:32-35 */
    uint32_t e = est[i];
    ++counts[e < cap ? e : cap];
  }
  uint32_t seen = 0, res = 0;
  for (uint32_t t = cap; t > 0; --t) { /* kernel.hpp:36-40 */
    seen += counts[t];
    if (seen >= t) { res = t; break; }
  }
  free(counts);
  return res;
}

/* Same arithmetic over a vertex's neighbours (recompute_node, src/fastk.cpp:15-20),
 * with the histogram clamped to min(cap, deg) bins: the result t <= deg, so
 * counts at levels <= min(cap, deg) are unchanged (identical result). */
static uint32_t recompute(const uint64_t* off, const uint32_t* nbr, const uint32_t* est,
                          uint32_t u, uint32_t cap, uint32_t* scratch) {
  if (cap == 0) return 0;
  uint64_t b = off[u], e = off[u + 1];
  uint64_t deg = e - b;
  uint32_t m = deg < cap ? (uint32_t)deg : cap;
  if (m == 0) return 0;
  memset(scratch, 0, sizeof(uint32_t) * ((size_t)m + 1));
  for (uint64_t i = b; i < e; ++i) {
    uint32_t x = est[nbr[i]];
    ++scratch[x < m ? x : m];
  }
  uint32_t seen = 0;
  for (uint32_t t = m; t > 0; --t) {
    seen += scratch[t];
    if (seen >= t) return t;
  }
  return 0;
}

/* should_notify / useful — include/kcore/fastk.hpp:25-27, src/fastk.cpp:22-24 */
static inline int should_notify(uint32_t nc, uint32_t oc, uint32_t ev) { return nc < ev && oc >= ev; }
static inline int useful(uint32_t nc, uint32_t oc, uint32_t ev, int ext) {
  return ext ? should_notify(nc, oc, ev) : ev > nc;
}
KCO_API int kco_should_notify(uint32_t nc, uint32_t oc, uint32_t ev) { return should_notify(nc, oc, ev); }

/* ------------------------------------------------------------------------ */
/* Bucket peel — restates peel_coreness, src/oracle.cpp:21-66 (Batagelj–     */
/* Zaversnik).  Single-threaded, O(V+E), the parity ground truth.            */
/* ------------------------------------------------------------------------ */
KCO_API void kco_peel(uint32_t n, const uint64_t* off, const uint32_t* nbr, uint32_t* core) {
  if (n == 0) return;
  uint32_t max_deg = 0;
  for (uint32_t u = 0; u < n; ++u) { /* oracle.cpp:26-30 */
    core[u] = (uint32_t)(off[u + 1] - off[u]);
    if (core[u] > max_deg) max_deg = core[u];
  }
  uint32_t* bin = (uint32_t*)calloc((size_t)max_deg + 2, sizeof(uint32_t));
  for (uint32_t u = 0; u < n; ++u) ++bin[core[u] + 1]; /* oracle.cpp:32-35 */
  for (uint32_t d = 1; d <= max_deg + 1; ++d) bin[d] += bin[d - 1];
  uint32_t* vert = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* pos = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* nxt = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)max_deg + 1));
  memcpy(nxt, bin, sizeof(uint32_t) * ((size_t)max_deg + 1));
  for (uint32_t u = 0; u < n; ++u) { /* oracle.cpp:37-45 */
    pos[u] = nxt[core[u]]++;
    vert[pos[u]] = u;
  }
  for (uint32_t i = 0; i < n; ++i) { /* oracle.cpp:47-64 */
    uint32_t v = vert[i];
    for (uint64_t j = off[v]; j < off[v + 1]; ++j) {
      uint32_t u = nbr[j];
      if (core[u] <= core[v]) continue;
      uint32_t du = core[u], pu = pos[u], pw = bin[du];
      uint32_t w = vert[pw];
      if (u != w) {
        vert[pu] = w; vert[pw] = u;
        pos[u] = pw; pos[w] = pu;
      }
      ++bin[du];
      --core[u];
    }
  }
  free(bin); free(vert); free(pos); free(nxt);
}

/* h-index of the degree sequence: bounds every estimate
 * after iteration 0. */
KCO_API uint32_t kco_degree_hindex(uint32_t n, const uint64_t* off) {
  uint64_t maxd = 0;
  for (uint32_t u = 0; u < n; ++u) { uint64_t d = off[u + 1] - off[u]; if (d > maxd) maxd = d; }
  uint64_t lim = maxd < n ? maxd : n;
  uint64_t* c = (uint64_t*)calloc(lim + 2, sizeof(uint64_t));
  for (uint32_t u = 0; u < n; ++u) { uint64_t d = off[u + 1] - off[u]; ++c[d < lim ? d : lim]; }
  uint64_t seen = 0; uint32_t h = 0;
  for (uint64_t t = lim; t > 0; --t) { seen += c[t]; if (seen >= t) { h = (uint32_t)t; break; } }
  free(c);
  return h;
}

/* ------------------------------------------------------------------------ */
/* Jacobi replay of the FastK round — the shadow_run semantics of           */
/* tests/test_fastk.cpp:41-92 (full-snapshot evaluation, updates applied     */
/* after the pass), restricted to the active set exactly as fastk_run's      */
/* process phase (src/fastk.cpp:128-149) with the activation rule chosen by  */
/* `rule`:                                                                  */
/*   0 REF_EXT   extended rule judged on settled values (fastk.cpp:156-163)  */
/*   1 REF_PLAIN plain guard on settled values (fastk.cpp:206-207, ext off)  */
/*   2 SNAP_PLAIN plain guard est_snapshot[v] > t in the same pass (SURVEY B) */
/*   3 SNAP_EXT  self-activation + extended rule on the snapshot (SURVEY C)  */
/* Counters follow RunReport (include/kcore/report.hpp:17-23): iterations    */
/* includes the final quiescent round; drained = evaluations; sent = fires.  */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t iterations, messages_sent, messages_drained, tail_pops;
  uint64_t e_scan;        /* sum of deg over evaluations */
  uint64_t notify_scan;   /* rule 0/1: adjacency entries re-read by the notify pass */
  uint64_t drops;         /* number of estimate decreases */
} kco_stats;

KCO_API int kco_jacobi(uint32_t n, const uint64_t* off, const uint32_t* nbr, int rule,
                       int clamp_h, uint32_t* est_out, kco_stats* st,
                       uint32_t* snapshots, uint64_t max_snap, uint64_t* active_counts,
                       uint64_t* scanned_per_iter, uint64_t max_iter_rec) {
  memset(st, 0, sizeof(*st));
  uint32_t H = clamp_h ? kco_degree_hindex(n, off) : 0xffffffffu;
  uint32_t* est = est_out;
  uint32_t maxdeg = 0;
  for (uint32_t u = 0; u < n; ++u) {
    uint32_t d = (uint32_t)(off[u + 1] - off[u]);
    est[u] = d < H ? d : H;
    if (d > maxdeg) maxdeg = d;
  }
  uint32_t* list = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* newv = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint8_t* flag = (uint8_t*)calloc(n ? n : 1, 1);
  uint64_t nact = n;
  for (uint32_t u = 0; u < n; ++u) list[u] = u;
  uint64_t it = 0;
  if (snapshots && max_snap > 0) memcpy(snapshots, est, sizeof(uint32_t) * n);
  if (active_counts && max_iter_rec > 0) active_counts[0] = n;
  int nth = omp_get_max_threads();
  uint32_t** scratch = (uint32_t**)malloc(sizeof(uint32_t*) * nth);
  for (int t = 0; t < nth; ++t) scratch[t] = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)maxdeg + 2));
  for (;;) {
    uint64_t scanned = 0, drops = 0, sent = 0;
    int any = 0;
#pragma omp parallel reduction(+ : scanned, drops, sent) reduction(| : any)
    {
      uint32_t* sc = scratch[omp_get_thread_num()];
#pragma omp for schedule(dynamic, 256)
      for (int64_t i = 0; i < (int64_t)nact; ++i) {
        uint32_t u = list[i];
        uint32_t cap = est[u];
        scanned += off[u + 1] - off[u];
        uint32_t t = recompute(off, nbr, est, u, cap, sc);
        newv[i] = t;
        if (t < cap) {
          any = 1;
          ++drops;
          if (rule >= 2) { /* single-pass activation on the snapshot */
            if (rule == 3) __atomic_store_n(&flag[u], 1, __ATOMIC_RELAXED);
            for (uint64_t j = off[u]; j < off[u + 1]; ++j) {
              uint32_t v = nbr[j];
              uint32_t ev = est[v];
              int fire = rule == 3 ? should_notify(t, cap, ev) : ev > t;
              if (fire) { __atomic_store_n(&flag[v], 1, __ATOMIC_RELAXED); ++sent; }
            }
          }
        }
      }
    }
    st->e_scan += scanned;
    st->messages_drained += nact;
    st->drops += drops;
    /* apply (fastk.cpp:153); rules 0/1 remember the old value in newv's place */
    uint32_t* oldv = NULL;
    if (rule <= 1) {
      oldv = (uint32_t*)malloc(sizeof(uint32_t) * (nact ? nact : 1));
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)nact; ++i) {
      uint32_t u = list[i];
      if (oldv) oldv[i] = est[u];
      est[u] = newv[i];
    }
    if (rule <= 1) { /* notify on settled values (fastk.cpp:156-163) */
      uint64_t ns = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : sent, ns)
      for (int64_t i = 0; i < (int64_t)nact; ++i) {
        uint32_t u = list[i];
        uint32_t t = newv[i], oc = oldv[i];
        if (t >= oc) continue;
        ns += off[u + 1] - off[u];
        for (uint64_t j = off[u]; j < off[u + 1]; ++j) {
          uint32_t v = nbr[j];
          if (useful(t, oc, est[v], rule == 0)) { __atomic_store_n(&flag[v], 1, __ATOMIC_RELAXED); ++sent; }
        }
      }
      st->notify_scan += ns;
      free(oldv);
    }
    st->messages_sent += sent;
    /* next active list in id order */
    uint64_t k = 0;
    for (uint32_t u = 0; u < n; ++u) if (flag[u]) { flag[u] = 0; list[k++] = u; }
    nact = k;
    ++it;
    if (scanned_per_iter && it - 1 < max_iter_rec) scanned_per_iter[it - 1] = scanned;
    if (active_counts && it < max_iter_rec) active_counts[it] = nact;
    if (snapshots && it < max_snap) memcpy(snapshots + it * (uint64_t)n, est, sizeof(uint32_t) * n);
    if (!any) break;
  }
  st->iterations = it;
  for (int t = 0; t < nth; ++t) free(scratch[t]);
  free(scratch); free(list); free(newv); free(flag);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Sequential tail — restates sequential_tail, src/fastk.cpp:28-55: min-heap */
/* of (estimate at push, node) ordered lexicographically (std::greater on a  */
/* pair), lazy deletion of stale entries.                                    */
/* ------------------------------------------------------------------------ */
typedef struct { uint32_t key, u; } heap_ent;
static inline int ent_less(heap_ent a, heap_ent b) { return a.key < b.key || (a.key == b.key && a.u < b.u); }
typedef struct { heap_ent* a; uint64_t len, cap; } heap_t;
static void heap_push(heap_t* h, heap_ent e) {
  if (h->len == h->cap) { h->cap = h->cap ? 2 * h->cap : 64; h->a = (heap_ent*)realloc(h->a, sizeof(heap_ent) * h->cap); }
  uint64_t i = h->len++;
  while (i > 0) {
    uint64_t p = (i - 1) / 2;
    if (!ent_less(e, h->a[p])) break;
    h->a[i] = h->a[p]; i = p;
  }
  h->a[i] = e;
}
static heap_ent heap_pop(heap_t* h) {
  heap_ent top = h->a[0], last = h->a[--h->len];
  uint64_t i = 0;
  for (;;) {
    uint64_t l = 2 * i + 1, r = l + 1, m = i;
    heap_ent best = last;
    if (l < h->len && ent_less(h->a[l], best)) { m = l; best = h->a[l]; }
    if (r < h->len && ent_less(h->a[r], best)) { m = r; }
    if (m == i) break;
    h->a[i] = h->a[m]; i = m;
  }
  if (h->len) h->a[i] = last;
  return top;
}

KCO_API void kco_sequential_tail(uint32_t n, const uint64_t* off, const uint32_t* nbr, uint32_t* est,
                                 uint8_t* active, int ext, kco_stats* st) {
  heap_t h = {0, 0, 0};
  uint32_t maxdeg = 0;
  for (uint32_t u = 0; u < n; ++u) { uint32_t d = (uint32_t)(off[u + 1] - off[u]); if (d > maxdeg) maxdeg = d; }
  uint32_t* sc = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)maxdeg + 2));
  for (uint32_t u = 0; u < n; ++u) if (active[u]) heap_push(&h, (heap_ent){est[u], u}); /* fastk.cpp:31-32 */
  while (h.len) { /* fastk.cpp:35-54 */
    heap_ent e = heap_pop(&h);
    ++st->tail_pops;
    uint32_t u = e.u;
    if (!active[u]) continue;
    active[u] = 0;
    ++st->messages_drained;
    uint32_t cap = est[u];
    st->e_scan += off[u + 1] - off[u];
    uint32_t t = recompute(off, nbr, est, u, cap, sc);
    if (t >= cap) continue;
    est[u] = t;
    for (uint64_t j = off[u]; j < off[u + 1]; ++j) {
      uint32_t v = nbr[j];
      uint32_t ev = est[v];
      if (!useful(t, cap, ev, ext)) continue;
      active[v] = 1;
      heap_push(&h, (heap_ent){ev, v});
      ++st->messages_sent;
    }
  }
  free(sc); free(h.a);
}

/* Full fastk_run restatement (src/fastk.cpp:57-187) at T=1: the reference is
 * bit-identical across thread counts (tests/test_fastk.cpp:205-230), so one
 * thread pins every counter.  batch only matters through the hybrid switch
 * (fastk.hpp:29-31). */
KCO_API int kco_fastk(uint32_t n, const uint64_t* off, const uint32_t* nbr, uint32_t batch,
                      int ext, int hybrid, uint32_t* est, kco_stats* st) {
  if (batch == 0) return -1; /* fastk.cpp:58-59 */
  memset(st, 0, sizeof(*st));
  uint32_t maxdeg = 0;
  for (uint32_t u = 0; u < n; ++u) { /* fastk.cpp:67-70 */
    est[u] = (uint32_t)(off[u + 1] - off[u]);
    if (est[u] > maxdeg) maxdeg = est[u];
  }
  uint8_t* active = (uint8_t*)malloc(n ? n : 1);
  memset(active, 1, n ? n : 1);
  uint32_t* sc = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)maxdeg + 2));
  typedef struct { uint32_t v, nc, oc; } pend_t;
  uint32_t* upd_u = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* upd_t = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  pend_t* pend = NULL; uint64_t pcap = 0;
  uint64_t active_count = n;
  int tail = 0;
  for (;;) {
    uint64_t nu = 0, np = 0;
    int changed = 0;
    int64_t delta = 0;
    for (uint32_t u = 0; u < n; ++u) { /* process, fastk.cpp:128-149 */
      if (!active[u]) continue;
      active[u] = 0; --delta; ++st->messages_drained;
      uint32_t cap = est[u];
      st->e_scan += off[u + 1] - off[u];
      uint32_t t = recompute(off, nbr, est, u, cap, sc);
      if (t >= cap) continue;
      upd_u[nu] = u; upd_t[nu] = t; ++nu; changed = 1;
      for (uint64_t j = off[u]; j < off[u + 1]; ++j) {
        uint32_t v = nbr[j];
        if (est[v] > t) {
          if (np == pcap) { pcap = pcap ? 2 * pcap : 1024; pend = (pend_t*)realloc(pend, sizeof(pend_t) * pcap); }
          pend[np++] = (pend_t){v, t, cap};
        }
      }
    }
    for (uint64_t i = 0; i < nu; ++i) est[upd_u[i]] = upd_t[i]; /* apply, fastk.cpp:153 */
    for (uint64_t i = 0; i < np; ++i) { /* notify, fastk.cpp:156-162 */
      pend_t p = pend[i];
      int fire = ext ? should_notify(p.nc, p.oc, est[p.v]) : est[p.v] > p.nc;
      if (!fire) continue;
      ++st->messages_sent;
      if (!active[p.v]) { active[p.v] = 1; ++delta; }
    }
    active_count = (uint64_t)((int64_t)active_count + delta);
    ++st->iterations; /* completion, fastk.cpp:102-118 */
    if (!changed) break;
    if (hybrid && active_count < batch) { tail = 1; break; }
  }
  if (tail) kco_sequential_tail(n, off, nbr, est, active, ext, st);
  free(active); free(sc); free(upd_u); free(upd_t); free(pend);
  return 0;
}
