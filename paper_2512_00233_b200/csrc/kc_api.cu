// kc_api.cu — the C-ABI (include/kcore_b200.h) over the sm_100a solver.
//
// Host side of the drop-in for kcore::fastk_run (reference
// include/kcore/fastk.hpp:46-47, src/fastk.cpp:57-187): validation with the
// reference's error behaviour (threads/batch == 0 rejected before any work,
// fastk.cpp:58-59), CSR upload, on-device layout (kc_prep.cu), the persistent
// round kernel (kc_solve.cu), permute-back + download, RunReport counters.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <new>
#include <string>
#include <atomic>
#include <unordered_map>
#include <vector>

#include "../../include/kcore_b200.h"
#include "kc_internal.h"

using namespace kcb;

namespace {

thread_local std::string g_last_error;

}  // namespace

namespace kcb {
static cudaMemPool_t g_pools[64];
void pool_debug(const char* what) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool = g_pools[dev & 63];
  if (!pool) return;
  uint64_t res = 0, used = 0, hi = 0;
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &hi);
  std::fprintf(stderr, "[kc host] pool %-12s reserved %.1f MB used %.1f MB high %.1f MB\n", what,
               res / 1e6, used / 1e6, hi / 1e6);
}
// Large blocks are recycled by exact size in front of the pool.  The pool
// keeps its memory (release threshold), but when the sizes are not page
// multiples (n = 20,000,000: 80,000,000-byte arrays, 1,557,878,200-byte
// adjacency) it re-maps the reserved pages into a fresh address range on
// every call: 0.6 ms per 80 MB, 6-10 ms per 1.5 GB — 22 ms of a 64 ms
// one-shot solve of the Chung-Lu graph, none on the power-of-two R-MAT sizes.
// A one-shot solve of the same graph size asks for the same sizes in the same
// order, so every request finds the block the previous call returned.  A
// returned block carries an event recorded on the stream that freed it and
// the next owner's stream waits on it (stream-ordered like cudaFreeAsync).
// Blocks not asked for during two consecutive uploads (another graph size)
// go back to the pool at the next miss, and all of them do when the pool
// runs out of memory.
namespace blockcache {
constexpr size_t CACHE_MIN_BYTES = 1u << 20;
struct IdleBlock {
  void* p;
  cudaEvent_t ev;
  uint64_t gen;  // upload generation it was returned in
};
struct BlockCache {
  std::mutex m;
  std::unordered_map<void*, size_t> live;              // handed out: pointer -> bytes
  std::unordered_multimap<size_t, IdleBlock> idle;     // returned, by exact size
};
BlockCache g_cache[64];
std::atomic<uint64_t> g_gen{2};  // bumped per uploaded handle (upload_common)
bool cache_on() {
  static const bool on = [] {
    const char* v = std::getenv("KC_BLOCK_CACHE");
    return !(v && *v == '0');
  }();
  return on;
}
}  // namespace blockcache
using namespace blockcache;

cudaError_t dmalloc(void** p, size_t bytes, cudaStream_t s) {
  // the library's own pool per device (not the device's default pool: its
  // release threshold is process-wide state other libraries rely on)
  static std::once_flag once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once[dev & 63], [dev] {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;  // keep freed blocks for the next solve
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      g_pools[dev & 63] = pool;
    } else {
      cudaGetLastError();
      g_pools[dev & 63] = nullptr;  // fall back to the default pool, untouched
    }
  });
  static const bool dbg = std::getenv("KC_DEBUG_HOST") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  if (!bytes) bytes = 1;
  BlockCache& bc = g_cache[dev & 63];
  const bool big = bytes >= CACHE_MIN_BYTES && cache_on();
  auto release = [s](const std::vector<IdleBlock>& v) {  // back to the pool, after their last use
    for (const IdleBlock& b : v) {
      cudaStreamWaitEvent(s, b.ev, 0);
      cudaEventDestroy(b.ev);
      cudaFreeAsync(b.p, s);
    }
  };
  if (big) {
    std::vector<IdleBlock> stale;
    IdleBlock hit{nullptr, nullptr, 0};
    {
      std::lock_guard<std::mutex> lk(bc.m);
      auto it = bc.idle.find(bytes);
      if (it != bc.idle.end()) {
        hit = it->second;
        bc.idle.erase(it);
        bc.live[hit.p] = bytes;
      } else {
        const uint64_t cur = g_gen.load();
        for (auto i = bc.idle.begin(); i != bc.idle.end();)
          if (i->second.gen + 2 <= cur) {
            stale.push_back(i->second);
            i = bc.idle.erase(i);
          } else {
            ++i;
          }
      }
    }
    if (hit.p) {
      cudaError_t e = cudaStreamWaitEvent(s, hit.ev, 0);
      cudaEventDestroy(hit.ev);
      if (e != cudaSuccess) return e;
      *p = hit.p;
      return cudaSuccess;
    }
    if (dbg && !stale.empty())
      std::fprintf(stderr, "[kc host] block cache: %zu stale blocks released\n", stale.size());
    release(stale);
  }
  cudaMemPool_t pool = g_pools[dev & 63];
  cudaError_t e = pool ? cudaMallocFromPoolAsync(p, bytes, pool, s) : cudaMallocAsync(p, bytes, s);
  if (e == cudaErrorMemoryAllocation) {  // hand every idle block back and retry
    cudaGetLastError();
    std::vector<IdleBlock> all;
    {
      std::lock_guard<std::mutex> lk(bc.m);
      for (auto& kv : bc.idle) all.push_back(kv.second);
      bc.idle.clear();
    }
    release(all);
    cudaStreamSynchronize(s);
    e = pool ? cudaMallocFromPoolAsync(p, bytes, pool, s) : cudaMallocAsync(p, bytes, s);
  }
  if (e == cudaSuccess && big) {
    std::lock_guard<std::mutex> lk(bc.m);
    bc.live[*p] = bytes;
  }
  if (dbg) {
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > 0.5) std::fprintf(stderr, "[kc host] dmalloc %zu bytes: %.3f ms\n", bytes, ms);
  }
  return e;
}
cudaError_t trim_memory() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  BlockCache& bc = g_cache[dev & 63];
  std::vector<IdleBlock> all;
  {
    std::lock_guard<std::mutex> lk(bc.m);
    for (auto& kv : bc.idle) all.push_back(kv.second);
    bc.idle.clear();
  }
  for (const IdleBlock& b : all) {
    cudaEventSynchronize(b.ev);
    cudaEventDestroy(b.ev);
    cudaFreeAsync(b.p, nullptr);
  }
  if ((e = cudaStreamSynchronize(nullptr)) != cudaSuccess) return e;
  if (g_pools[dev & 63]) return cudaMemPoolTrimTo(g_pools[dev & 63], 0);
  return cudaSuccess;
}
void dfree(void* p, cudaStream_t s) {
  if (!p) return;
  int dev = 0;
  cudaGetDevice(&dev);
  BlockCache& bc = g_cache[dev & 63];
  size_t bytes = 0;
  {
    std::lock_guard<std::mutex> lk(bc.m);
    auto it = bc.live.find(p);
    if (it != bc.live.end()) {
      bytes = it->second;
      bc.live.erase(it);
    }
  }
  if (bytes) {  // a large block: keep it for the next request of this size
    cudaEvent_t ev = nullptr;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess &&
        cudaEventRecord(ev, s) == cudaSuccess) {
      std::lock_guard<std::mutex> lk(bc.m);
      bc.idle.emplace(bytes, IdleBlock{p, ev, g_gen.load()});
      return;
    }
    if (ev) cudaEventDestroy(ev);
    cudaGetLastError();
  }
  cudaFreeAsync(p, s);
}
}  // namespace kcb

namespace {

kc_status fail(kc_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

kc_status cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear sticky-less errors
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  if (e == cudaErrorMemoryAllocation) return fail(KC_ERR_OUT_OF_MEMORY, m);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver || e == cudaErrorInvalidDevice)
    return fail(KC_ERR_NO_DEVICE, m);
  return fail(KC_ERR_CUDA, m);
}

#define CK(x)                                      \
  do {                                             \
    cudaError_t e_ = (x);                          \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
  } while (0)

kc_status check_device(int device, int* num_sms) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(KC_ERR_NO_DEVICE, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  if (device < 0 || device >= count) return fail(KC_ERR_NO_DEVICE, "device index out of range");
  // single attributes (cudaGetDeviceProperties costs milliseconds per call)
  int major = 0, sms = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  if (major != 10) {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    return fail(KC_ERR_NO_DEVICE, std::string("device is not sm_100 (Blackwell): ") + prop.name);
  }
  CK(cudaSetDevice(device));
  if (num_sms) *num_sms = sms;
  return KC_OK;
}

__global__ void permute_back_kernel(const void* est, bool est16, const uint32_t* perm,
                                    uint32_t n, uint32_t n_nz, uint32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t v = 0;
    if (i < n_nz) v = est16 ? ((const uint16_t*)est)[i] : ((const uint32_t*)est)[i];
    out[perm[i]] = v;
  }
}

// Measurement probe (kc_debug_gather_probe): one pass over every adjacency
// entry of the layout — the 128-bit id stream with the solver's L2
// evict-first hint, and one gather of the entry's estimate from `est` (no
// shared-memory cache) — i.e. the solver's inner operation with nothing
// else.  Its ncu L2 hit rate, with the id sectors (read once: misses)
// taken out, is the hit rate of the estimate gathers; its time is the
// gather rate this graph allows.
template <typename EstT>
__global__ void est_gather_probe_kernel(const uint32_t* __restrict__ adj, uint64_t nnz,
                                        const EstT* __restrict__ est,
                                        unsigned long long* out) {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const uint64_t nvec = nnz / 4;
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 q;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                 : "l"(adj + 4 * i), "l"(pol));
    acc += (uint32_t)est[q.x] + (uint32_t)est[q.y] + (uint32_t)est[q.z] + (uint32_t)est[q.w];
  }
  if (acc == 0x7fffffffu) atomicAdd(out, 1ull);  // keeps the loads
}

template <typename OffT>
__global__ void degree_back_kernel(const OffT* off, const uint32_t* perm, uint32_t n,
                                   uint32_t n_nz, uint32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[perm[i]] = i < n_nz ? (uint32_t)(off[i + 1] - off[i]) : 0u;
}

// Number of set byte flags (observed mode's active_count).
__global__ void count_flags_kernel(const uint8_t* f, uint32_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    c += f[i] != 0;
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage t;
  const unsigned long long b = BR(t).Sum(c);
  if (threadIdx.x == 0 && b) atomicAdd(out, b);
}

// k_max and sum of estimates (n_nz entries).
__global__ void kstats_kernel(const void* est, bool est16, uint32_t n_nz,
                              unsigned long long* out /* [0]=max, [1]=sum */) {
  uint32_t mx = 0;
  unsigned long long sm = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_nz; i += gridDim.x * blockDim.x) {
    uint32_t v = est16 ? ((const uint16_t*)est)[i] : ((const uint32_t*)est)[i];
    mx = v > mx ? v : mx;
    sm += v;
  }
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage t1;
  __shared__ typename BR::TempStorage t2;
  unsigned long long bmx = BR(t1).Reduce((unsigned long long)mx, cub::Max());
  unsigned long long bsm = BR(t2).Sum(sm);
  if (threadIdx.x == 0) {
    atomicMax(&out[0], bmx);
    atomicAdd(&out[1], bsm);
  }
}

}  // namespace

struct kc_graph {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  uint32_t n = 0;
  uint64_t nnz = 0;
  PrepOut lay{};
  bool est16 = true;
  float t_upload = 0.f, t_prep = 0.f;
  // solver state (allocated at first solve)
  bool solver_ready = false;
  uint32_t max_rounds = 0;
  SolveBuffers sb{};
  uint32_t* d_out = nullptr;      // coreness in caller ids [n]
  unsigned long long* d_prof = nullptr;  // phase timestamps (debug)
  unsigned long long* d_count = nullptr; // observed mode: active-flag count
  uint32_t state_buf = 0;                // est buffer holding the current state
  uint32_t round_launches = 1;           // solver kernels queued by the last run_rounds
  unsigned long long* d_k = nullptr;
  // independent peel / verify (allocated at first use)
  bool peel_ready = false;
  PeelBuffers pb{};
  uint32_t* d_cand = nullptr;            // verify: FastK coreness (caller ids)
};

namespace {

void free_peel(kc_graph* g) {
  if (!g->peel_ready) return;
  dfree(g->pb.deg, g->stream);
  dfree(g->pb.core, g->stream);
  for (int i = 0; i < 2; ++i) {
    dfree(g->pb.rem[i], g->stream);
    dfree(g->pb.fr[i], g->stream);
    dfree(g->pb.frb[i], g->stream);
  }
  dfree(g->pb.ctl, g->stream);
  dfree(g->d_cand, g->stream);
  g->d_cand = nullptr;
  std::memset(&g->pb, 0, sizeof(g->pb));
  g->peel_ready = false;
}

void free_solver(kc_graph* g) {
  if (!g->solver_ready) return;
  dfree(g->sb.est[0], g->stream);
  dfree(g->sb.est[1], g->stream);
  dfree(g->sb.cnt, g->stream);
  dfree(g->sb.queue, g->stream);
  dfree(g->sb.queue2, g->stream);
  dfree(g->sb.radj, g->stream);
  dfree(g->sb.rlen, g->stream);
  dfree(g->sb.rthr, g->stream);
  dfree(g->sb.spec, g->stream);
  dfree(g->sb.pflag, g->stream);
  dfree(g->sb.lq[0], g->stream);
  dfree(g->sb.lq[1], g->stream);
  dfree(g->sb.flag[0], g->stream);
  dfree(g->sb.flag[1], g->stream);
  dfree(g->sb.ctl, g->stream);
  dfree(g->sb.anydrop, g->stream);
  dfree(g->sb.stats, g->stream);
  dfree(g->sb.status, g->stream);
  dfree(g->sb.tailc, g->stream);
  dfree(g->d_out, g->stream);
  dfree(g->d_k, g->stream);
  dfree(g->d_prof, g->stream);
  dfree(g->d_count, g->stream);
  g->d_prof = nullptr;
  g->d_count = nullptr;
  g->d_out = nullptr;
  g->d_k = nullptr;
  std::memset(&g->sb, 0, sizeof(g->sb));
  g->solver_ready = false;
}

kc_status ensure_solver(kc_graph* g, uint32_t max_rounds) {
  (void)max_rounds;
  if (g->solver_ready) return KC_OK;
  struct Mark {
    bool on = std::getenv("KC_DEBUG_HOST") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    ~Mark() {
      if (on)
        std::fprintf(stderr, "[kc host] ensure_solver allocs %8.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
  } mark;
  const uint32_t n_nz = g->lay.n_nz;
  const size_t es = g->est16 ? 2 : 4;
  const size_t n_pad = (((size_t)n_nz + 15) & ~(size_t)15) + 16;  // 16-byte vectors + slack
  SolveBuffers& b = g->sb;
  std::memset(&b, 0, sizeof(b));
  b.off = g->lay.off;
  b.adj = g->lay.adj;
  b.dcut = g->lay.dcut;
  b.dcut_n = g->lay.dcut ? g->lay.max_degree + 2 : 0u;
  b.rows_sorted = g->lay.rows_sorted;
  b.n_nz = n_nz;
  for (int c = 0; c <= NCLS; ++c) b.cls_begin[c] = g->lay.cls_begin[c];
  g->solver_ready = true;  // so that partial allocations get freed
  CK(dmalloc((void**)&b.est[0], n_pad * es, g->stream));
  CK(dmalloc((void**)&b.est[1], n_pad * es, g->stream));
  CK(dmalloc((void**)&b.cnt, n_pad * sizeof(uint32_t), g->stream));
  CK(dmalloc((void**)&b.queue, n_pad * sizeof(uint32_t), g->stream));
  CK(dmalloc((void**)&b.queue2, n_pad * sizeof(uint32_t), g->stream));
  CK(dmalloc((void**)&b.rlen, n_pad * sizeof(uint32_t), g->stream));
  CK(dmalloc((void**)&b.rthr, n_pad * es, g->stream));
  CK(dmalloc((void**)&b.radj, ((size_t)g->nnz + ADJ_PAD) * sizeof(uint32_t), g->stream));
  CK(cudaMemsetAsync(b.radj + g->nnz, 0, ADJ_PAD * sizeof(uint32_t), g->stream));
  CK(dmalloc((void**)&b.spec, 3 * ((((size_t)n_nz + 15) & ~(size_t)15) + 16) * sizeof(uint32_t),
             g->stream));
  for (int ph = 0; ph < 2; ++ph) {  // slots hold 0xffffffff while empty
    CK(dmalloc((void**)&b.lq[ph], ((size_t)b.cls_begin[1] + 1) * sizeof(uint32_t), g->stream));
    CK(cudaMemsetAsync(b.lq[ph], 0xff, ((size_t)b.cls_begin[1] + 1) * sizeof(uint32_t), g->stream));
  }
  CK(dmalloc((void**)&b.pflag, n_pad, g->stream));
  CK(cudaMemsetAsync(b.pflag, 0, n_pad, g->stream));
  CK(dmalloc((void**)&b.flag[0], n_pad, g->stream));
  CK(dmalloc((void**)&b.flag[1], n_pad, g->stream));
  CK(cudaMemsetAsync(b.est[0], 0, n_pad * es, g->stream));
  CK(cudaMemsetAsync(b.est[1], 0, n_pad * es, g->stream));
  CK(cudaMemsetAsync(b.flag[0], 0, n_pad, g->stream));
  CK(cudaMemsetAsync(b.flag[1], 0, n_pad, g->stream));
  CK(dmalloc((void**)&b.ctl, 2 * sizeof(Ctl), g->stream));
  CK(dmalloc((void**)&b.anydrop, 4 * sizeof(uint32_t), g->stream));
  CK(dmalloc((void**)&b.stats, (size_t)STAT_SLOTS * sizeof(RoundStat), g->stream));
  CK(dmalloc((void**)&b.status, ST_SLOTS * sizeof(uint32_t), g->stream));
  CK(cudaMemsetAsync(b.status, 0, ST_SLOTS * sizeof(uint32_t), g->stream));
  CK(dmalloc((void**)&b.tailc, TAIL_SLOTS * sizeof(unsigned long long), g->stream));
  if (!g->d_out) CK(dmalloc((void**)&g->d_out, (g->n ? g->n : 1) * sizeof(uint32_t), g->stream));
  if (!g->d_k) CK(dmalloc((void**)&g->d_k, 2 * sizeof(unsigned long long), g->stream));
  CK(dmalloc((void**)&g->d_count, sizeof(unsigned long long), g->stream));
  g->max_rounds = max_rounds;
  return KC_OK;
}

int map_rule(const kc_options& o) {
  const bool ref = o.rule == KC_RULE_REFERENCE;
  if (ref) return o.extended_notify ? R_REF_EXT : R_REF_PLAIN;
  return R_COUNT;  // exact activation: extended_notify cannot change it
}

kc_status validate(const kc_options* opt, kc_options* o) {
  if (opt) *o = *opt; else kc_default_options(o);
  // fastk.cpp:58-59 — rejected before any work
  if (o->threads == 0) return fail(KC_ERR_INVALID_ARGUMENT, "fastk: threads must be >= 1");
  if (o->batch == 0) return fail(KC_ERR_INVALID_ARGUMENT, "fastk: batch must be >= 1");
  if (o->rule < 0 || o->rule > KC_RULE_AUTO) return fail(KC_ERR_INVALID_ARGUMENT, "unknown rule");
  if (o->rule == KC_RULE_AUTO) o->rule = KC_RULE_COUNTING;
  // Every round with a drop lowers sum(est) by >= 1, so the loop terminates;
  // 0 means no cap (paths need ~n/2 Jacobi rounds).
  if (o->max_rounds == 0) o->max_rounds = 0xffffffffu;
  return KC_OK;
}

// The reference rule with hybrid_tail finishes like fastk_run: once fewer
// than `batch` vertices are active, the sequential tail (kc_tail.cu).  The
// counting rule has no use for it (its rounds only hold droppers).
bool uses_tail(const kc_options& o) { return o.hybrid_tail && map_rule(o) != R_COUNT; }

// The counting rule runs on kc_count.cu's solver (lists + direct queues)
// unless the legacy flag-frontier solver is requested for A/B runs.
bool uses_count_kernel(const kc_options& o) {
  return map_rule(o) == R_COUNT && !(o.reserved[0] & KC_DEBUG_LEGACY_COUNT);
}

uint32_t cache_entries(const kc_graph* g, const kc_options& o) {
  if (o.smem_cache == 0xffffffffu) return 0;
  const size_t es = g->est16 ? 2 : 4;
  size_t want = o.smem_cache ? o.smem_cache : solver_cache_bytes_max() / es;
  size_t maxe = solver_cache_bytes_max() / es;
  if (want > maxe) want = maxe;
  size_t n_pad = ((size_t)g->lay.n_nz + 15) & ~(size_t)15;
  if (want > n_pad) want = n_pad;
  want &= ~(size_t)15;  // 16-entry multiple (16-byte vectors for either width)
  return (uint32_t)want;
}

#ifndef KC_SPLIT_ROUNDS_DEFAULT
#define KC_SPLIT_ROUNDS_DEFAULT 16u   // rounds 1 .. 16 one kernel per phase while they are large
#endif                                // (24 from 1e9 entries: the rounds stay large longer; a
                                      // launch after the hand-off is a ~4 us no-op)
#ifndef KC_SPLIT_MIN_BIG_ROWS
#define KC_SPLIT_MIN_BIG_ROWS 65536u  // ... on graphs with at least this many rows of degree > 64
#endif
uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* v = std::getenv(name);
  return v && *v ? (uint32_t)std::strtoul(v, nullptr, 10) : dflt;
}

// Run the solver to convergence (or one round when `one_round`), leaving the
// estimates on the device.  Fills the counters of `st`.
kc_status run_rounds(kc_graph* g, const kc_options& o, uint32_t r_begin, uint32_t r_end,
                     bool tail_switch) {
  if ((o.reserved[0] & KC_DEBUG_PHASE_TIMES) && !g->d_prof) {
    CK(dmalloc((void**)&g->d_prof, (size_t)PROF_ROUNDS * g->num_sms * PROF_PHASES * 8, g->stream));
    CK(cudaMemsetAsync(g->d_prof, 0, (size_t)PROF_ROUNDS * g->num_sms * PROF_PHASES * 8, g->stream));
  }
  g->sb.prof = (o.reserved[0] & KC_DEBUG_PHASE_TIMES) ? g->d_prof : nullptr;
  SolveConfig c{};
  c.rule = map_rule(o);
  c.clamp_drop = g->lay.max_degree > g->lay.h_graph ? 1u : 0u;
  c.cache_n = cache_entries(g, o);
  c.max_rounds = o.max_rounds;
  c.tail_threshold = tail_switch ? o.batch : 0u;
  c.num_sms = g->num_sms;
  c.pull = (o.reserved[0] & KC_DEBUG_NO_PULL) ? 0u : 1u;
  // Per-phase kernels (kc_count_split.cu) for the large rounds of a whole
  // solve: on by default for graphs with enough vertices of degree > 64 (the
  // warp / CTA list scans they speed up); each of their launches costs ~4 us,
  // which small graphs do not earn back (ER: 0.52 -> 0.79 ms with them).
  // KC_SPLIT_ROUNDS (0: off) / KC_SPLIT_MIN / KC_SPLIT_CACHE override.
  static const char* split_env = std::getenv("KC_SPLIT_ROUNDS");
  static const uint32_t split_rounds_env = env_u32("KC_SPLIT_ROUNDS", 0u);
  const uint32_t split_rounds = (split_env && *split_env) ? split_rounds_env
                                : g->nnz >= 1000000000ull ? KC_SPLIT_ROUNDS_DEFAULT + 8u
                                                          : KC_SPLIT_ROUNDS_DEFAULT;
  static const uint32_t split_min = env_u32("KC_SPLIT_MIN", 1024u);
  static const uint32_t split_cache = env_u32("KC_SPLIT_CACHE", 1u);
  const bool split_fits = g->lay.cls_begin[C_SUB] >= KC_SPLIT_MIN_BIG_ROWS;
  c.split_rounds = (split_env && *split_env) || split_fits ? split_rounds : 0u;
  c.split_min = split_min;
  c.split_cache = split_cache;
  g->sb.prof_ctas = (uint32_t)g->num_sms;
  // solver kernels this call queues (kc_stats.kernel_launches): the persistent kernel, or
  // persistent + 2 per per-phase round + persistent again (launch_count_rounds)
  g->round_launches = 1u;
  if (uses_count_kernel(o) && c.split_rounds && r_begin == 0 && r_end > 2)
    g->round_launches = 2u + 2u * (c.split_rounds < r_end - 1 ? c.split_rounds : r_end - 1);
  if (uses_count_kernel(o))
    CK(launch_count_rounds(g->sb, c, g->est16, g->lay.off64, r_begin, r_end, g->stream));
  else
    CK(launch_rounds(g->sb, c, g->est16, g->lay.off64, r_begin, r_end, g->stream));
  return KC_OK;
}

kc_status init_state(kc_graph* g, const kc_options& o) {
  CK(cudaMemsetAsync(g->sb.tailc, 0, TAIL_SLOTS * sizeof(unsigned long long), g->stream));
  if (uses_count_kernel(o))
    CK(launch_count_init(g->sb, g->est16, g->lay.off64, g->lay.h_graph, g->stream));
  else
    CK(launch_init(g->sb, g->est16, g->lay.off64, g->lay.h_graph, o.max_rounds, g->stream));
  return KC_OK;
}

kc_status collect(kc_graph* g, const kc_options& o, kc_stats* st, bool* converged) {
  uint32_t status[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(status, g->sb.status, sizeof(status), cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  const uint32_t rounds = status[0];
  *converged = status[1] != 0;
  g->state_buf = status[3] & 1;
  if (!st) return KC_OK;
  const uint32_t slots = rounds < STAT_SLOTS ? rounds : STAT_SLOTS;
  std::vector<RoundStat> rs(slots);
  if (slots)
    CK(cudaMemcpy(rs.data(), g->sb.stats, slots * sizeof(RoundStat), cudaMemcpyDeviceToHost));
  st->iterations = rounds;
  st->messages_sent = st->messages_drained = st->e_scan = st->v_eval = st->drops = 0;
  st->scan_evaluate = st->scan_notify = 0;
  for (const RoundStat& r : rs) {
    st->scan_evaluate += r.ascan;
    st->scan_notify += r.nscan;
    st->messages_sent += r.fires;
    st->v_eval += r.evals;
    st->e_scan += r.escan;
    st->drops += r.drops;
  }
  // isolated vertices are evaluated once in round 0 by the reference
  // (fastk.cpp:128-149 sweeps all ids); they cost nothing here.
  st->messages_drained = st->v_eval + (rounds ? (uint64_t)(g->n - g->lay.n_nz) : 0);
  st->tail_pops = 0;
  st->tail_rounds = 0;
  if (uses_tail(o)) {  // fastk.cpp:175-185: the tail's pops, evaluations, notifications
    unsigned long long tc[TAIL_SLOTS];
    CK(cudaMemcpy(tc, g->sb.tailc, sizeof(tc), cudaMemcpyDeviceToHost));
    st->tail_pops = tc[TAIL_POPS];
    st->messages_sent += tc[TAIL_FIRES];
    st->v_eval += tc[TAIL_EVALS];
    st->messages_drained += tc[TAIL_EVALS];
    st->e_scan += tc[TAIL_ESCAN];
    st->drops += tc[TAIL_DROPS];
    st->tail_rounds = tc[TAIL_RAN];
  }
  return KC_OK;
}

kc_status kstats(kc_graph* g, kc_stats* st) {
  if (!st) return KC_OK;
  unsigned long long k[2] = {0, 0};
  CK(cudaMemsetAsync(g->d_k, 0, 2 * sizeof(unsigned long long), g->stream));
  if (g->lay.n_nz) {
    kstats_kernel<<<g->num_sms * 2, 256, 0, g->stream>>>(g->sb.est[g->state_buf], g->est16,
                                                        g->lay.n_nz, g->d_k);
    CK(cudaGetLastError());
  }
  CK(cudaMemcpyAsync(k, g->d_k, sizeof(k), cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  st->k_max = (uint32_t)k[0];
  st->k_avg = g->n ? (double)k[1] / (double)g->n : 0.0;
  st->h_graph = g->lay.h_graph;
  return KC_OK;
}

kc_status permute_back(kc_graph* g) {
  if (!g->n) return KC_OK;
  permute_back_kernel<<<g->num_sms * 4, 256, 0, g->stream>>>(g->sb.est[g->state_buf], g->est16,
                                                             g->lay.perm,
                                                             g->n, g->lay.n_nz, g->d_out);
  CK(cudaGetLastError());
  return KC_OK;
}

// KC_DEBUG_HOST=1: host wall-clock milestones of the upload (stderr).
struct HostClock {
  bool on = std::getenv("KC_DEBUG_HOST") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[kc host] %-22s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t0).count());
  }
};

kc_status upload_common(const kc_csr_view* csr, int device, bool on_device, uint32_t flags,
                        kc_graph** out) {
  kcb::DeviceGuard device_guard;  // restore the caller's current device
  HostClock hc;
  kcb::blockcache::g_gen.fetch_add(1);  // (the block cache ages its idle blocks by uploads)
  if (!out) return fail(KC_ERR_INVALID_ARGUMENT, "out is null");
  *out = nullptr;
  if (!csr) return fail(KC_ERR_INVALID_ARGUMENT, "csr view is null");
  if (csr->n > 0 && (!csr->offsets || (csr->nnz > 0 && !csr->neighbors)))
    return fail(KC_ERR_INVALID_ARGUMENT, "csr view has null arrays");
  int sms = 0;
  kc_status s = check_device(device, &sms);
  if (s != KC_OK) return s;
  hc.mark("check_device");
  kc_graph* g = new (std::nothrow) kc_graph();
  if (!g) return fail(KC_ERR_OUT_OF_MEMORY, "host allocation failed");
  g->device = device;
  g->num_sms = sms;
  g->n = csr->n;
  g->nnz = csr->nnz;
  auto bail = [&](kc_status st) {
    kc_graph_free(g);
    return st;
  };
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking)) != cudaSuccess)
    return bail(cuda_fail(e, "cudaStreamCreate"));
  for (auto& ev : g->ev)
    if ((e = cudaEventCreate(&ev)) != cudaSuccess) return bail(cuda_fail(e, "cudaEventCreate"));
  hc.mark("stream+events");
  if (g->n == 0) {
    *out = g;
    return KC_OK;
  }
  uint64_t* d_off = nullptr;
  uint32_t* d_adj = nullptr;
  struct Stage {  // the staged (pageable) neighbour upload's host thread
    std::thread th;
    std::mutex m;
    std::condition_variable cv;
    int recorded = 0;
    cudaError_t err = cudaSuccess;
  } stage;
  // pipelined neighbours (host path): chunks of old rows on a copy stream,
  // each relabelled by the layout as soon as it lands
  cudaStream_t cs = nullptr;
  std::vector<cudaEvent_t> ready;
  std::vector<uint32_t> old_lo;
  AdjFeed feed{0, nullptr, nullptr};
  auto drop_feed = [&]() {
    for (cudaEvent_t ev : ready)
      if (ev) cudaEventDestroy(ev);
    ready.clear();
    if (cs) cudaStreamDestroy(cs);
    cs = nullptr;
  };
  if (!on_device) {
    if (csr->offsets[0] != 0 || csr->offsets[csr->n] != csr->nnz)
      return bail(fail(KC_ERR_INVALID_ARGUMENT, "offsets[0] != 0 or offsets[n] != nnz"));
    cudaEventRecord(g->ev[0], g->stream);
    if ((e = dmalloc_n(&d_off, (size_t)g->n + 1, g->stream)) != cudaSuccess)
      return bail(cuda_fail(e, "cudaMallocAsync offsets"));
    if ((e = dmalloc_n(&d_adj, g->nnz, g->stream)) != cudaSuccess) {
      dfree(d_off, g->stream);
      return bail(cuda_fail(e, "cudaMallocAsync neighbors"));
    }
    // pageable host arrays (a reference Graph's std::vectors) go through the
    // pinned staging ring (kc_stage.cu); pinned ones straight to the DMA engine
    const bool pageable = is_pageable(csr->offsets) || is_pageable(csr->neighbors);
    if (pageable)
      e = staged_h2d(d_off, csr->offsets, ((size_t)g->n + 1) * sizeof(uint64_t), g->stream);
    else
      e = cudaMemcpyAsync(d_off, csr->offsets, ((size_t)g->n + 1) * sizeof(uint64_t),
                          cudaMemcpyHostToDevice, g->stream);
    // chunks of ~64 MB of neighbours, cut at row boundaries (at most 16)
    const uint64_t bytes = g->nnz * sizeof(uint32_t);
    uint64_t k = (bytes + (64ull << 20) - 1) / (64ull << 20);
    k = k < 1 ? 1 : k > 16 ? 16 : k;
    old_lo.push_back(0);
    // cut points in 1/(4k) of the entries: k equal chunks; when a chunk is
    // large (>= 256 MB) the last one is cut again into 1/2, 1/4, 1/4 — only the
    // last chunk's layout is not hidden under a copy
    std::vector<uint64_t> cuts;
    for (uint64_t c = 1; c < k; ++c) cuts.push_back(4 * c);
    if (bytes / k >= (256ull << 20)) {
      cuts.push_back(4 * k - 2);
      cuts.push_back(4 * k - 1);
    }
    for (uint64_t q : cuts) {  // first row whose start is >= q/(4k) of the entries
      const uint64_t target = (uint64_t)((unsigned __int128)g->nnz * q / (4 * k));
      uint32_t lo = old_lo.back(), hi = g->n;
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (csr->offsets[mid] < target) lo = mid + 1; else hi = mid;
      }
      if (lo > old_lo.back() && lo < g->n) old_lo.push_back(lo);
    }
    old_lo.push_back(g->n);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    cudaEvent_t alloc_done = nullptr;
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&alloc_done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(alloc_done, g->stream);  // stream-ordered allocations
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, alloc_done, 0);
    if (alloc_done) cudaEventDestroy(alloc_done);
    const size_t nchunks = old_lo.size() - 1;
    for (size_t c = 0; e == cudaSuccess && c < nchunks; ++c) {
      cudaEvent_t ev = nullptr;
      e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e == cudaSuccess) ready.push_back(ev);
    }
    // chunk c: its neighbours on the copy stream, then ready[c]
    auto copy_chunk = [&, cs](size_t c) -> cudaError_t {
      const uint64_t b0 = csr->offsets[old_lo[c]], b1 = csr->offsets[old_lo[c + 1]];
      cudaError_t ce = cudaSuccess;
      if (b1 > b0)
        ce = pageable ? staged_h2d(d_adj + b0, csr->neighbors + b0, (b1 - b0) * sizeof(uint32_t), cs)
                      : cudaMemcpyAsync(d_adj + b0, csr->neighbors + b0,
                                        (b1 - b0) * sizeof(uint32_t), cudaMemcpyHostToDevice, cs);
      if (ce == cudaSuccess) ce = cudaEventRecord(ready[c], cs);
      return ce;
    };
    if (e == cudaSuccess && !pageable) {
      for (size_t c = 0; e == cudaSuccess && c < nchunks; ++c) e = copy_chunk(c);
      if (e == cudaSuccess) e = cudaEventRecord(g->ev[1], cs);
    } else if (e == cudaSuccess) {
      // staged: a host thread fills the pinned ring chunk by chunk while this
      // thread lays out the chunks already recorded (AdjFeed::host_wait)
      stage.recorded = 0;
      stage.err = cudaSuccess;
      stage.th = std::thread([&, copy_chunk, nchunks] {
        cudaSetDevice(g->device);
        for (size_t c = 0; c < nchunks; ++c) {
          cudaError_t ce = stage.err == cudaSuccess ? copy_chunk(c) : stage.err;
          if (ce == cudaSuccess && c + 1 == nchunks) ce = cudaEventRecord(g->ev[1], cs);
          {
            std::lock_guard<std::mutex> lk(stage.m);
            if (ce != cudaSuccess) stage.err = ce;
            stage.recorded = (int)c + 1;
          }
          stage.cv.notify_all();
        }
      });
    }
    if (e != cudaSuccess) {
      cudaStreamSynchronize(g->stream);
      if (cs) cudaStreamSynchronize(cs);
      drop_feed();
      dfree(d_off, g->stream);
      dfree(d_adj, g->stream);
      return bail(cuda_fail(e, "cudaMemcpy H2D"));
    }
    feed = AdjFeed{(int)ready.size(), old_lo.data(), ready.data()};
    if (pageable) {
      feed.host_wait = [](void* ctx, int c) {
        Stage* st = static_cast<Stage*>(ctx);
        std::unique_lock<std::mutex> lk(st->m);
        st->cv.wait(lk, [&] { return st->recorded > c; });
      };
      feed.ctx = &stage;
    }
    hc.mark("H2D enqueued");
  } else {
    d_off = const_cast<uint64_t*>(csr->offsets);
    d_adj = const_cast<uint32_t*>(csr->neighbors);
    cudaEventRecord(g->ev[0], g->stream);
    cudaEventRecord(g->ev[1], g->stream);
  }
  e = prep_layout(d_off, d_adj, g->n, g->nnz, (flags & KC_UPLOAD_FORCE_OFF64) != 0,
                  (flags & KC_UPLOAD_UNSORTED_ROWS) == 0, g->stream, &g->lay,
                  on_device ? nullptr : &feed);
  hc.mark("layout returned");
  if (stage.th.joinable()) {
    stage.th.join();
    if (stage.err != cudaSuccess && e == cudaSuccess) e = stage.err;
  }
  if (cs) cudaStreamWaitEvent(g->stream, g->ev[1], 0);  // every chunk copied (error paths too)
  cudaEventRecord(g->ev[2], g->stream);
  cudaStreamSynchronize(g->stream);
  if (cs) cudaStreamSynchronize(cs);
  drop_feed();
  hc.mark("synced");
  if (!on_device) {
    dfree(d_off, g->stream);
    dfree(d_adj, g->stream);
  }
  if (e != cudaSuccess) return bail(cuda_fail(e, "layout"));
  if (g->lay.invalid)
    return bail(fail(KC_ERR_INVALID_ARGUMENT,
                     "not a CSR: offsets must run 0..nnz non-decreasing and every neighbour id "
                     "must be < n (graph.hpp:37-75)"));
  cudaEventElapsedTime(&g->t_upload, g->ev[0], g->ev[1]);
  cudaEventElapsedTime(&g->t_prep, g->ev[1], g->ev[2]);
  g->est16 = g->lay.h_graph < EST16_LIMIT && !(flags & KC_UPLOAD_FORCE_EST32);
  *out = g;
  return KC_OK;
}

}  // namespace

extern "C" {

const char* kc_status_str(kc_status s) {
  switch (s) {
    case KC_OK: return "ok";
    case KC_ERR_INVALID_ARGUMENT: return "invalid argument";
    case KC_ERR_NO_DEVICE: return "no usable sm_100 CUDA device";
    case KC_ERR_OUT_OF_MEMORY: return "out of device memory";
    case KC_ERR_CUDA: return "CUDA error";
    case KC_ERR_NOT_CONVERGED: return "round cap exceeded before convergence";
    case KC_ERR_CALLBACK: return "inspector callback aborted the run";
    case KC_ERR_PARSE: return "malformed edge list";
    case KC_ERR_IO: return "edge list could not be read";
  }
  return "unknown status";
}

int kc_abi_version(void) { return KC_ABI_VERSION; }

const char* kc_last_error(void) { return g_last_error.c_str(); }

void kc_default_options(kc_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->threads = 16;  // FastKOptions defaults, fastk.hpp:12-22
  o->batch = 256;
  o->extended_notify = 1;
  o->hybrid_tail = 1;
  o->rule = KC_RULE_AUTO;
  o->max_rounds = 0;
  o->smem_cache = 0;
}

kc_status kc_graph_upload(const kc_csr_view* csr, int device, kc_graph** out) {
  g_last_error.clear();
  return upload_common(csr, device, false, 0u, out);
}

kc_status kc_graph_upload_device(const kc_csr_view* csr, int device, kc_graph** out) {
  g_last_error.clear();
  return upload_common(csr, device, true, 0u, out);
}

kc_status kc_graph_upload_ex(const kc_csr_view* csr, int device, int on_device, uint32_t flags,
                             kc_graph** out) {
  g_last_error.clear();
  if (flags & ~(KC_UPLOAD_FORCE_OFF64 | KC_UPLOAD_FORCE_EST32 | KC_UPLOAD_UNSORTED_ROWS))
    return fail(KC_ERR_INVALID_ARGUMENT, "unknown upload flags");
  return upload_common(csr, device, on_device != 0, flags, out);
}

void kc_graph_free(kc_graph* g) {
  kcb::DeviceGuard device_guard;  // restore the caller's current device
  if (!g) return;
  HostClock hc;
  cudaSetDevice(g->device);
  free_solver(g);
  free_peel(g);
  dfree(g->d_out, g->stream);  // when only the peel ran
  dfree(g->d_k, g->stream);
  dfree(g->lay.off, g->stream);
  dfree(g->lay.adj, g->stream);
  dfree(g->lay.perm, g->stream);
  dfree(g->lay.dcut, g->stream);
  if (g->stream) cudaStreamSynchronize(g->stream);
  for (auto& ev : g->ev)
    if (ev) cudaEventDestroy(ev);
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
  hc.mark("graph_free");
  if (hc.on) kcb::pool_debug("after free");
}

uint32_t kc_graph_n(const kc_graph* g) { return g ? g->n : 0; }
uint64_t kc_graph_nnz(const kc_graph* g) { return g ? g->nnz : 0; }
kc_status kc_trim_memory(void) {
  g_last_error.clear();
  int cur = 0, sms = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) {
    cudaGetLastError();
    return fail(KC_ERR_NO_DEVICE, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  kc_status s = check_device(cur, &sms);
  if (s != KC_OK) return s;
  CK(kcb::trim_memory());
  return KC_OK;
}

void kc_debug_host_copy(void* dst, const void* src, uint64_t bytes) {
  kcb::host_copy(dst, src, (size_t)bytes);
}

void* kc_graph_stream(kc_graph* g) { return g ? (void*)g->stream : nullptr; }

kc_status kc_graph_timings(const kc_graph* g, float* tu, float* tp) {
  if (!g) return fail(KC_ERR_INVALID_ARGUMENT, "null graph");
  if (tu) *tu = g->t_upload;
  if (tp) *tp = g->t_prep;
  return KC_OK;
}

static kc_status solve_impl(kc_graph* g, const kc_options* opt, uint32_t* out, bool out_dev,
                            kc_stats* st) {
  kcb::DeviceGuard device_guard;  // restore the caller's current device
  g_last_error.clear();
  if (!g) return fail(KC_ERR_INVALID_ARGUMENT, "null graph");
  kc_options o;
  kc_status s = validate(opt, &o);
  if (s != KC_OK) return s;
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->t_upload_ms = g->t_upload;
    st->t_prep_ms = g->t_prep;
  }
  CK(cudaSetDevice(g->device));
  if (g->n == 0) {  // empty graph: one (empty) round, tests/test_fastk.cpp:156-159
    if (st) st->iterations = 1;
    return KC_OK;
  }
  if (g->lay.n_nz == 0) {  // edgeless: one round evaluates every vertex to 0
    if (out_dev) CK(cudaMemsetAsync(out, 0, g->n * sizeof(uint32_t), g->stream));
    else std::memset(out, 0, g->n * sizeof(uint32_t));
    CK(cudaStreamSynchronize(g->stream));
    if (st) {
      st->iterations = 1;
      st->messages_drained = g->n;
      st->h_graph = 0;
    }
    return KC_OK;
  }
  HostClock hc;
  s = ensure_solver(g, o.max_rounds);
  if (s != KC_OK) return s;
  hc.mark("solve: ensure_solver");
  CK(cudaEventRecord(g->ev[0], g->stream));
  s = init_state(g, o);
  if (s != KC_OK) return s;
  s = run_rounds(g, o, 0, o.max_rounds, uses_tail(o));
  if (s != KC_OK) return s;
  if (uses_tail(o))  // a no-op unless the rounds stopped for the tail
    CK(launch_tail(g->sb, g->lay.perm, g->est16, g->lay.off64, o.extended_notify != 0, -1,
                   g->num_sms, g->stream));
  CK(cudaEventRecord(g->ev[1], g->stream));
  bool conv = false;
  s = collect(g, o, st, &conv);
  if (s != KC_OK) return s;
  if (!conv) return fail(KC_ERR_NOT_CONVERGED, "round cap reached");
  s = kstats(g, st);
  if (s != KC_OK) return s;
  CK(cudaEventRecord(g->ev[2], g->stream));
  s = permute_back(g);
  if (s != KC_OK) return s;
  if (out_dev)
    CK(cudaMemcpyAsync(out, g->d_out, g->n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, g->stream));
  else if (g->n >= (1u << 20) && is_pageable(out))  // through the pinned ring (kc_stage.cu)
    CK(staged_d2h(out, g->d_out, g->n * sizeof(uint32_t), g->stream));
  else
    CK(cudaMemcpyAsync(out, g->d_out, g->n * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
  CK(cudaEventRecord(g->ev[3], g->stream));
  CK(cudaStreamSynchronize(g->stream));
  hc.mark("solve: done");
  if (st) {
    // init + solver kernels (+ tail list + tail) + k stats + permute-back
    st->kernel_launches = 1u + g->round_launches + (uses_tail(o) ? 2u : 0u) + 2u;
    cudaEventElapsedTime(&st->t_solve_ms, g->ev[0], g->ev[1]);
    cudaEventElapsedTime(&st->t_download_ms, g->ev[2], g->ev[3]);
  }
  return KC_OK;
}

kc_status kc_solve(kc_graph* g, const kc_options* opt, uint32_t* coreness, kc_stats* st) {
  if (g && g->n && !coreness) return fail(KC_ERR_INVALID_ARGUMENT, "coreness is null");
  return solve_impl(g, opt, coreness, false, st);
}

kc_status kc_solve_device(kc_graph* g, const kc_options* opt, uint32_t* coreness_dev,
                          kc_stats* st) {
  if (g && g->n && !coreness_dev) return fail(KC_ERR_INVALID_ARGUMENT, "coreness is null");
  return solve_impl(g, opt, coreness_dev, true, st);
}

}  // extern "C"

namespace {

// What the one-round-per-launch loop hands out at each iteration boundary
// (instrument_boundary, report.cpp:20-29): the estimates to an inspector
// (one D2H of est per boundary), and/or a record_iteration row
// (report.cpp:7-18) computed on the device — a sum of the estimates, so a
// trace costs one 16-byte copy per boundary.  The gap sum is an exact
// integer, so mean_error is bit-identical to the reference's double sum.
struct Boundaries {
  kc_inspector_fn fn = nullptr;
  void* user = nullptr;
  bool trace = false;
  uint64_t truth_sum = 0;
  kc_iteration_stat* rows = nullptr;
  uint64_t cap = 0;
  uint64_t count = 0;
};

kc_status boundary(kc_graph* g, Boundaries& b, uint64_t it, uint64_t active,
                   std::vector<uint32_t>& snap, bool degrees) {
  if (b.fn) {
    if (degrees) {  // iteration 0: the reference reports est = degree (fastk.cpp:67-68, 93)
      if (g->lay.off64)
        degree_back_kernel<uint64_t><<<g->num_sms * 4, 256, 0, g->stream>>>(
            (const uint64_t*)g->lay.off, g->lay.perm, g->n, g->lay.n_nz, g->d_out);
      else
        degree_back_kernel<uint32_t><<<g->num_sms * 4, 256, 0, g->stream>>>(
            (const uint32_t*)g->lay.off, g->lay.perm, g->n, g->lay.n_nz, g->d_out);
      CK(cudaGetLastError());
    } else {
      kc_status s = permute_back(g);
      if (s != KC_OK) return s;
    }
    CK(cudaMemcpyAsync(snap.data(), g->d_out, g->n * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                       g->stream));
    CK(cudaStreamSynchronize(g->stream));
    if (b.fn(b.user, it, snap.data(), g->n, active)) return fail(KC_ERR_CALLBACK, "inspector");
  }
  if (b.trace) {
    uint64_t sum = g->nnz;  // iteration 0: sum of degrees
    if (!degrees) {
      unsigned long long k[2] = {0, 0};
      CK(cudaMemsetAsync(g->d_k, 0, sizeof(k), g->stream));
      kstats_kernel<<<g->num_sms * 2, 256, 0, g->stream>>>(g->sb.est[g->state_buf], g->est16,
                                                          g->lay.n_nz, g->d_k);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(k, g->d_k, sizeof(k), cudaMemcpyDeviceToHost, g->stream));
      CK(cudaStreamSynchronize(g->stream));
      sum = k[1];
    }
    if (b.count < b.cap) {
      const double n = (double)g->n;
      b.rows[b.count].mean_error = g->n ? (double)((int64_t)sum - (int64_t)b.truth_sum) / n : 0.0;
      b.rows[b.count].active_fraction = g->n ? (double)active / n : 0.0;
    }
    ++b.count;
  }
  return KC_OK;
}

kc_status observed_impl(kc_graph* g, const kc_options* opt, Boundaries& b, uint32_t* coreness,
                        kc_stats* st) {
  kcb::DeviceGuard device_guard;  // restore the caller's current device
  g_last_error.clear();
  if (!g) return fail(KC_ERR_INVALID_ARGUMENT, "null graph");
  kc_options o;
  kc_status s = validate(opt, &o);
  if (s != KC_OK) return s;
  if (g->n && !coreness) return fail(KC_ERR_INVALID_ARGUMENT, "coreness is null");
  if (st) std::memset(st, 0, sizeof(*st));
  CK(cudaSetDevice(g->device));
  std::vector<uint32_t> snap(b.fn ? g->n : 0);
  if (g->n == 0 || g->lay.n_nz == 0) {
    // iteration 0 (degrees = 0) and the single quiescent round
    if (b.fn && b.fn(b.user, 0, snap.data(), g->n, g->n)) return fail(KC_ERR_CALLBACK, "inspector");
    if (b.fn && b.fn(b.user, 1, snap.data(), g->n, 0)) return fail(KC_ERR_CALLBACK, "inspector");
    for (uint64_t it = 0; b.trace && it < 2; ++it) {
      if (b.count < b.cap) {
        const double n = g->n ? (double)g->n : 1.0;
        b.rows[b.count].mean_error = -(double)b.truth_sum / n;
        b.rows[b.count].active_fraction = it == 0 && g->n ? 1.0 : 0.0;
      }
      ++b.count;
    }
    if (g->n) std::memset(coreness, 0, g->n * sizeof(uint32_t));
    if (st) {
      st->iterations = 1;
      st->messages_drained = g->n;
    }
    return KC_OK;
  }
  s = ensure_solver(g, o.max_rounds);
  if (s != KC_OK) return s;
  s = init_state(g, o);
  if (s != KC_OK) return s;
  s = boundary(g, b, 0, g->n, snap, true);
  if (s != KC_OK) return s;
  bool conv = false;
  for (uint32_t r = 0; r < o.max_rounds && !conv; ++r) {
    s = run_rounds(g, o, r, r + 1, false);
    if (s != KC_OK) return s;
    s = collect(g, o, nullptr, &conv);
    if (s != KC_OK) return s;
    unsigned long long active = 0;
    if (!conv && uses_count_kernel(o)) {  // round r+1's queue sizes
      Ctl ctl;
      CK(cudaMemcpyAsync(&ctl, g->sb.ctl + ((r + 1) & 1), sizeof(Ctl), cudaMemcpyDeviceToHost,
                         g->stream));
      CK(cudaStreamSynchronize(g->stream));
      for (int c = 0; c < NCLS; ++c) active += ctl.qcnt[c];
    } else if (!conv) {  // flags collected for round r+1 (the reference's active_count)
      CK(cudaMemsetAsync(g->d_count, 0, sizeof(unsigned long long), g->stream));
      count_flags_kernel<<<g->num_sms * 2, 256, 0, g->stream>>>(g->sb.flag[(r + 1) & 1],
                                                                g->lay.n_nz, g->d_count);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(&active, g->d_count, sizeof(active), cudaMemcpyDeviceToHost, g->stream));
      CK(cudaStreamSynchronize(g->stream));
    }
    s = boundary(g, b, (uint64_t)r + 1, active, snap, false);
    if (s != KC_OK) return s;
    if (!conv && uses_tail(o) && active < o.batch) {
      // hybrid switch after round r (fastk.cpp:113-115): the sequential tail
      // from round r+1's active flags, then one more boundary with nothing
      // active (fastk.cpp:180-183)
      CK(launch_tail(g->sb, g->lay.perm, g->est16, g->lay.off64, o.extended_notify != 0,
                     (int)((r + 1) & 1), g->num_sms, g->stream));
      s = boundary(g, b, (uint64_t)r + 2, 0, snap, false);
      if (s != KC_OK) return s;
      conv = true;
    }
  }
  if (!conv) return fail(KC_ERR_NOT_CONVERGED, "round cap reached");
  s = collect(g, o, st, &conv);
  if (s != KC_OK) return s;
  s = kstats(g, st);
  if (s != KC_OK) return s;
  s = permute_back(g);
  if (s != KC_OK) return s;
  CK(cudaMemcpyAsync(coreness, g->d_out, g->n * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                     g->stream));
  CK(cudaStreamSynchronize(g->stream));
  return KC_OK;
}

}  // namespace

extern "C" {

kc_status kc_solve_observed(kc_graph* g, const kc_options* opt, kc_inspector_fn fn, void* user,
                            uint32_t* coreness, kc_stats* st) {
  Boundaries b;
  b.fn = fn;
  b.user = user;
  return observed_impl(g, opt, b, coreness, st);
}

kc_status kc_solve_traced(kc_graph* g, const kc_options* opt, const uint32_t* truth,
                          kc_iteration_stat* trace, uint64_t trace_cap, uint64_t* trace_rows,
                          uint32_t* coreness, kc_stats* st) {
  if (!g) return fail(KC_ERR_INVALID_ARGUMENT, "null graph");
  if (g->n && !truth) return fail(KC_ERR_INVALID_ARGUMENT, "truth is null");
  if (trace_cap && !trace) return fail(KC_ERR_INVALID_ARGUMENT, "trace is null");
  Boundaries b;
  b.trace = true;
  for (uint32_t u = 0; u < g->n; ++u) b.truth_sum += truth[u];
  b.rows = trace;
  b.cap = trace_cap;
  kc_status s = observed_impl(g, opt, b, coreness, st);
  if (trace_rows) *trace_rows = b.count;
  return s;
}



kc_status kc_debug_phase_times(kc_graph* g, unsigned long long* out, uint64_t cap,
                               uint32_t* grid) {
  if (!g || !out || !grid) return fail(KC_ERR_INVALID_ARGUMENT, "null argument");
  *grid = (uint32_t)g->num_sms;
  if (!g->d_prof) return fail(KC_ERR_INVALID_ARGUMENT, "no phase times recorded");
  const uint64_t total = (uint64_t)PROF_ROUNDS * g->num_sms * PROF_PHASES;
  CK(cudaMemcpy(out, g->d_prof, (cap < total ? cap : total) * 8, cudaMemcpyDeviceToHost));
  return KC_OK;
}

kc_status kc_debug_round_stats(kc_graph* g, unsigned long long* out, uint32_t rounds) {
  if (!g || !out) return fail(KC_ERR_INVALID_ARGUMENT, "null argument");
  if (!g->sb.stats) return fail(KC_ERR_INVALID_ARGUMENT, "no solve has run");
  const uint32_t k = rounds < STAT_SLOTS ? rounds : STAT_SLOTS;
  CK(cudaMemcpy(out, g->sb.stats, (size_t)k * sizeof(RoundStat), cudaMemcpyDeviceToHost));
  return KC_OK;
}

kc_status kc_debug_gather_probe(kc_graph* g, int reps, float* ms_per_pass) {
  kcb::DeviceGuard device_guard;
  if (!g || !ms_per_pass) return fail(KC_ERR_INVALID_ARGUMENT, "null argument");
  if (!g->sb.est[0]) return fail(KC_ERR_INVALID_ARGUMENT, "no solve has run");
  CK(cudaSetDevice(g->device));
  const uint64_t nnz = g->nnz & ~(uint64_t)3;
  CK(cudaEventRecord(g->ev[0], g->stream));
  for (int r = 0; r < (reps > 0 ? reps : 1); ++r) {
    if (g->est16)
      est_gather_probe_kernel<uint16_t><<<g->num_sms * 8, 256, 0, g->stream>>>(
          g->lay.adj, nnz, (const uint16_t*)g->sb.est[0], g->d_count);
    else
      est_gather_probe_kernel<uint32_t><<<g->num_sms * 8, 256, 0, g->stream>>>(
          g->lay.adj, nnz, (const uint32_t*)g->sb.est[0], g->d_count);
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(g->ev[1], g->stream));
  CK(cudaEventSynchronize(g->ev[1]));
  float ms = 0;
  cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]);
  *ms_per_pass = ms / (reps > 0 ? reps : 1);
  return KC_OK;
}

kc_status kc_debug_layout(kc_graph* g, uint64_t* offsets, uint32_t* neighbors, uint32_t* perm,
                          uint32_t* n_nz, int* rows_sorted) {
  kcb::DeviceGuard device_guard;
  if (!g) return fail(KC_ERR_INVALID_ARGUMENT, "null argument");
  CK(cudaSetDevice(g->device));
  if (n_nz) *n_nz = g->n ? g->lay.n_nz : 0u;
  if (rows_sorted) *rows_sorted = g->n && g->lay.rows_sorted ? 1 : 0;
  if (g->n == 0) return KC_OK;
  CK(cudaStreamSynchronize(g->stream));
  const size_t m = (size_t)g->lay.n_nz + 1;
  if (offsets) {
    if (g->lay.off64) {
      CK(cudaMemcpy(offsets, g->lay.off, m * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    } else {
      std::vector<uint32_t> tmp(m);
      CK(cudaMemcpy(tmp.data(), g->lay.off, m * sizeof(uint32_t), cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < m; ++i) offsets[i] = tmp[i];
    }
  }
  if (neighbors && g->nnz)
    CK(cudaMemcpy(neighbors, g->lay.adj, g->nnz * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  if (perm) CK(cudaMemcpy(perm, g->lay.perm, (size_t)g->n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return KC_OK;
}

static kc_status ensure_peel(kc_graph* g) {
  if (g->peel_ready) return KC_OK;
  const size_t m = (size_t)g->lay.n_nz + 1;
  PeelBuffers& b = g->pb;
  std::memset(&b, 0, sizeof(b));
  b.off = g->lay.off;
  b.adj = g->lay.adj;
  b.n_nz = g->lay.n_nz;
  g->peel_ready = true;  // partial allocations get freed
  CK(dmalloc_n(&b.deg, m, g->stream));
  CK(dmalloc_n(&b.core, m, g->stream));
  for (int i = 0; i < 2; ++i) {
    CK(dmalloc_n(&b.rem[i], m, g->stream));
    CK(dmalloc_n(&b.fr[i], m, g->stream));
    CK(dmalloc_n(&b.frb[i], m, g->stream));
  }
  CK(dmalloc(&b.ctl, peel_ctl_bytes(), g->stream));
  CK(dmalloc_n(&g->d_cand, (size_t)g->n + 1, g->stream));
  if (!g->d_out) CK(dmalloc_n(&g->d_out, (size_t)g->n + 1, g->stream));
  if (!g->d_k) CK(dmalloc_n(&g->d_k, 2, g->stream));
  return KC_OK;
}

// Peel on the device into g->d_out (caller ids); levels and time in st.
static kc_status peel_device(kc_graph* g, kc_stats* st) {
  kc_status s = ensure_peel(g);
  if (s != KC_OK) return s;
  CK(cudaEventRecord(g->ev[0], g->stream));
  CK(launch_peel(g->pb, g->lay.off64, g->num_sms, g->stream));
  CK(cudaEventRecord(g->ev[1], g->stream));
  CK(launch_peel_out(g->pb, g->lay.perm, g->n, g->d_out, g->num_sms, g->stream));
  if (st) {
    uint32_t levels = 0;
    unsigned long long k[2] = {0, 0};
    CK(cudaMemcpyAsync(&levels, (const char*)g->pb.ctl + peel_ctl_bytes() - sizeof(uint32_t),
                       sizeof(levels), cudaMemcpyDeviceToHost, g->stream));
    CK(cudaMemsetAsync(g->d_k, 0, sizeof(k), g->stream));
    kstats_kernel<<<g->num_sms * 2, 256, 0, g->stream>>>(g->d_out, false, g->n, g->d_k);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(k, g->d_k, sizeof(k), cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    st->iterations = g->lay.n_nz ? levels : 1;
    st->k_max = (uint32_t)k[0];
    st->k_avg = g->n ? (double)k[1] / (double)g->n : 0.0;
    st->h_graph = g->lay.h_graph;
    cudaEventElapsedTime(&st->t_solve_ms, g->ev[0], g->ev[1]);
  }
  return KC_OK;
}

__global__ void perturb_kernel(uint32_t* c, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (i % 997u == 0) c[i] += 1;
}

__global__ void mismatch_gather_kernel(const uint32_t* ids, uint32_t m, const uint32_t* cand,
                                       const uint32_t* truth, kc_mismatch* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const uint32_t u = ids[i];
    out[i].node = u;
    out[i].candidate = cand[u];
    out[i].truth = truth[u];
  }
}

kc_status kc_peel(kc_graph* g, uint32_t* coreness, kc_stats* st) {
  kcb::DeviceGuard device_guard;  // restore the caller's current device
  g_last_error.clear();
  if (!g) return fail(KC_ERR_INVALID_ARGUMENT, "null graph");
  if (g->n && !coreness) return fail(KC_ERR_INVALID_ARGUMENT, "coreness is null");
  if (st) std::memset(st, 0, sizeof(*st));
  CK(cudaSetDevice(g->device));
  if (g->n == 0) {
    if (st) st->iterations = 1;
    return KC_OK;
  }
  kc_status s = peel_device(g, st);
  if (s != KC_OK) return s;
  CK(cudaMemcpyAsync(coreness, g->d_out, g->n * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                     g->stream));
  CK(cudaStreamSynchronize(g->stream));
  return KC_OK;
}

// Standalone sequential tail (kcore::sequential_tail, fastk.hpp:38-39): the
// caller's estimates and active flags (caller ids) in, the device tail, the
// estimates out.  Isolated vertices never interact: an active one pops once
// and its estimate becomes 0 (compute_index_over of no values).
__global__ void tail_in_kernel(const uint32_t* est, const uint8_t* active, const uint32_t* perm,
                               uint32_t n, uint32_t n_nz, uint32_t* E, uint32_t* N, uint8_t* flag,
                               uint32_t* est_out, unsigned long long* iso) {
  unsigned long long c = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t old = perm[i];
    if (i < n_nz) {
      E[i] = N[i] = est[old];
      flag[i] = active[old] != 0;
    } else {
      est_out[old] = active[old] ? 0u : est[old];
      c += active[old] != 0;
    }
  }
  if (c) atomicAdd(iso, c);
}

__global__ void tail_out_kernel(const uint32_t* E, const uint32_t* perm, uint32_t n_nz,
                                uint32_t* est_out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_nz; i += gridDim.x * blockDim.x)
    est_out[perm[i]] = E[i];
}

kc_status kc_sequential_tail(kc_graph* g, uint32_t* est, uint8_t* active, int extended_notify,
                             kc_stats* st) {
  kcb::DeviceGuard device_guard;  // restore the caller's current device
  g_last_error.clear();
  if (!g) return fail(KC_ERR_INVALID_ARGUMENT, "null graph");
  if (g->n && (!est || !active)) return fail(KC_ERR_INVALID_ARGUMENT, "est / active is null");
  if (st) std::memset(st, 0, sizeof(*st));
  if (g->n == 0) return KC_OK;
  CK(cudaSetDevice(g->device));
  kc_status s = ensure_solver(g, 0);
  if (s != KC_OK) return s;
  const uint32_t n = g->n, n_nz = g->lay.n_nz;
  uint32_t *d_est = nullptr, *d_out = nullptr, *E = nullptr, *N = nullptr;
  uint8_t* d_act = nullptr;
  unsigned long long* d_iso = nullptr;
  auto cleanup = [&]() {
    dfree(d_est, g->stream);
    dfree(d_out, g->stream);
    dfree(E, g->stream);
    dfree(N, g->stream);
    dfree(d_act, g->stream);
    dfree(d_iso, g->stream);
  };
  cudaError_t e = cudaSuccess;
  if ((e = dmalloc_n(&d_est, n, g->stream)) != cudaSuccess ||
      (e = dmalloc_n(&d_out, n, g->stream)) != cudaSuccess ||
      (e = dmalloc_n(&E, (size_t)n_nz + 16, g->stream)) != cudaSuccess ||
      (e = dmalloc_n(&N, (size_t)n_nz + 16, g->stream)) != cudaSuccess ||
      (e = dmalloc_n(&d_act, n, g->stream)) != cudaSuccess ||
      (e = dmalloc_n(&d_iso, 1, g->stream)) != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "cudaMallocAsync");
  }
  unsigned long long iso = 0, tc[TAIL_SLOTS] = {};
  // 32-bit estimates whatever the handle's width: the caller's values are
  // arbitrary (fastk.hpp:38-39 takes any est), the tail compares them exactly
  SolveBuffers b = g->sb;
  b.est[0] = E;
  b.est[1] = N;
  e = cudaMemcpyAsync(d_est, est, (size_t)n * 4, cudaMemcpyHostToDevice, g->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_act, active, n, cudaMemcpyHostToDevice, g->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_iso, 0, 8, g->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(g->sb.tailc, 0, TAIL_SLOTS * 8, g->stream);
  if (e == cudaSuccess) {
    tail_in_kernel<<<g->num_sms * 4, 256, 0, g->stream>>>(d_est, d_act, g->lay.perm, n, n_nz, E, N,
                                                         g->sb.flag[0], d_out, d_iso);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && n_nz)
    e = launch_tail(b, g->lay.perm, false, g->lay.off64, extended_notify != 0, 0, g->num_sms,
                    g->stream);
  if (e == cudaSuccess) {
    tail_out_kernel<<<g->num_sms * 4, 256, 0, g->stream>>>(E, g->lay.perm, n_nz, d_out);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(est, d_out, (size_t)n * 4, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&iso, d_iso, 8, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(tc, g->sb.tailc, sizeof(tc), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  cleanup();
  if (e != cudaSuccess) return cuda_fail(e, "sequential tail");
  std::memset(active, 0, n);  // every pushed entry was popped: nothing stays active
  if (st) {
    st->tail_pops = (n_nz ? tc[TAIL_POPS] : 0) + iso;
    st->messages_drained = (n_nz ? tc[TAIL_EVALS] : 0) + iso;
    st->messages_sent = n_nz ? tc[TAIL_FIRES] : 0;
    st->drops = n_nz ? tc[TAIL_DROPS] : 0;
    st->e_scan = n_nz ? tc[TAIL_ESCAN] : 0;
    st->tail_rounds = 1;
  }
  return KC_OK;
}

kc_status kc_verify(kc_graph* g, const kc_options* opt, kc_mismatch* out, uint64_t cap,
                    uint64_t* count) {
  kcb::DeviceGuard device_guard;  // restore the caller's current device
  g_last_error.clear();
  if (!g) return fail(KC_ERR_INVALID_ARGUMENT, "null graph");
  if (!count) return fail(KC_ERR_INVALID_ARGUMENT, "count is null");
  if (cap && !out) return fail(KC_ERR_INVALID_ARGUMENT, "out is null");
  *count = 0;
  CK(cudaSetDevice(g->device));
  if (g->n == 0) return KC_OK;
  kc_status s = ensure_peel(g);
  if (s != KC_OK) return s;
  // candidate: FastK, coreness kept on the device
  s = kc_solve_device(g, opt, g->d_cand, nullptr);
  if (s != KC_OK) return s;
  if (opt && (opt->reserved[0] & KC_DEBUG_VERIFY_PERTURB)) {
    perturb_kernel<<<g->num_sms, 256, 0, g->stream>>>(g->d_cand, g->n);
    CK(cudaGetLastError());
  }
  s = peel_device(g, nullptr);  // truth into d_out
  if (s != KC_OK) return s;
  unsigned long long c = 0;
  CK(cudaMemsetAsync(g->d_k, 0, sizeof(unsigned long long), g->stream));
  CK(launch_mismatch_count(g->d_cand, g->d_out, g->n, g->d_k, g->num_sms, g->stream));
  CK(cudaMemcpyAsync(&c, g->d_k, sizeof(c), cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  *count = c;
  const uint64_t m = c < cap ? c : cap;
  if (m) {
    uint32_t* ids = nullptr;
    kc_mismatch* d_mm = nullptr;
    CK(dmalloc_n(&ids, m, g->stream));
    CK(dmalloc_n(&d_mm, m, g->stream));
    CK(launch_mismatch_list(g->d_cand, g->d_out, g->n, ids, (uint32_t)m, g->stream));
    mismatch_gather_kernel<<<g->num_sms, 256, 0, g->stream>>>(ids, (uint32_t)m, g->d_cand,
                                                             g->d_out, d_mm);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, d_mm, m * sizeof(kc_mismatch), cudaMemcpyDeviceToHost, g->stream));
    dfree(ids, g->stream);
    dfree(d_mm, g->stream);
    CK(cudaStreamSynchronize(g->stream));
  }
  return KC_OK;
}

#ifndef KC_ONESHOT_SORT
#define KC_ONESHOT_SORT 1  // 0: keep the relabelled rows in input order (A/B)
#endif
kc_status kc_fastk_run(const kc_csr_view* csr, const kc_options* opt, uint32_t* coreness,
                       kc_stats* st) {
  kc_options o;
  kc_status s = validate(opt, &o);  // invalid options rejected before any work
  if (s != KC_OK) return s;
  kc_graph* g = nullptr;
  // sorted layout: the rows are sorted on chip while each upload chunk is
  // relabelled (kc_prep.cu), under the copy of the next chunk
  s = kc_graph_upload_ex(csr, 0, 0, KC_ONESHOT_SORT ? 0u : KC_UPLOAD_UNSORTED_ROWS, &g);
  if (s != KC_OK) return s;
  s = kc_solve(g, &o, coreness, st);
  kc_graph_free(g);
  return s;
}

}  // extern "C"
