// kc_ingest.cu — SNAP-style text edge lists parsed and densified on the
// device: the GPU form of the reference's loader,
// /root/reference/proj/src/graph.cpp:
//   EdgeListParser (22-80)  one "u v" pair per line; ' ', '\t', '\r' are
//                           blanks; blank lines and lines whose first
//                           non-blank character is '#' are skipped; ids are
//                           unsigned 64-bit decimals; errors name the
//                           1-based line ("malformed token 'x'", "expected
//                           two ids, got one", "expected two ids per line")
//   densify (141-182)       dense ids = ranks of the ascending distinct ids
//                           that appear; original ids kept
//   build_csr (85-128)      self-loops dropped, duplicates collapsed, sorted
//                           rows — kc_gen.cu's build_csr_dev
// Pipeline: line starts (one flag per byte, compacted), one thread per line
// parses, valid pairs compacted, endpoints radix-sorted and uniqued, every
// endpoint ranked by binary search, CSR built on the device.  The first
// malformed line (lowest line number, as the streaming reference throws) is
// re-parsed on the host only to word the error exactly like ParseError.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/kcore_b200.h"
#include "kc_internal.h"

#include <zlib.h>

namespace kcb {

// kc_gen.cu
kc_status build_csr_dev_public(uint32_t n, const uint2* pairs, uint64_t m, cudaStream_t s,
                               uint64_t** off_out, uint32_t** nbr_out, uint64_t* nnz_out);
const char* gen_last_error();

namespace {

enum LineKind : uint32_t { L_SKIP = 0, L_EDGE = 1, L_BAD_TOKEN = 2, L_ONE_ID = 3, L_TOO_MANY = 4 };

__host__ __device__ inline bool is_blank(char c) { return c == ' ' || c == '\t' || c == '\r'; }

// One line [p, end) (graph.cpp:66-79).  Token errors report the token span.
__host__ __device__ inline uint32_t parse_line(const char* p, const char* end, uint64_t& u,
                                               uint64_t& v, const char** tb, const char** te) {
  while (end > p && is_blank(*(end - 1))) --end;
  while (p < end && is_blank(*p)) ++p;
  if (p == end || *p == '#') return L_SKIP;
  uint64_t val[2];
  for (int k = 0; k < 2; ++k) {
    const char* tok = p;
    while (p < end && !is_blank(*p)) ++p;
    // std::from_chars on an unsigned 64-bit integer: decimal digits only,
    // the whole token consumed, no overflow (graph.cpp:56-62)
    uint64_t x = 0;
    bool ok = true;
    for (const char* c = tok; c < p; ++c) {
      if (*c < '0' || *c > '9') {
        ok = false;
        break;
      }
      const uint64_t d = (uint64_t)(*c - '0');
      if (x > (~0ull - d) / 10) {
        ok = false;
        break;
      }
      x = x * 10 + d;
    }
    if (!ok) {
      *tb = tok;
      *te = p;
      return L_BAD_TOKEN;
    }
    val[k] = x;
    while (p < end && is_blank(*p)) ++p;
    if (k == 0 && p == end) return L_ONE_ID;
  }
  if (p != end) return L_TOO_MANY;
  u = val[0];
  v = val[1];
  return L_EDGE;
}

struct LineStart {
  const char* text;
  __device__ bool operator()(uint64_t i) const { return i == 0 || text[i - 1] == '\n'; }
};

__global__ void parse_kernel(const char* text, uint64_t len, const uint64_t* starts, uint64_t L,
                             ulonglong2* pairs, uint8_t* is_edge, unsigned long long* first_bad) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < L;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = starts[k];
    uint64_t e = k + 1 < L ? starts[k + 1] - 1 : len;
    if (k + 1 == L && e > b && text[e - 1] == '\n') --e;
    uint64_t u = 0, v = 0;
    const char *tb = nullptr, *te = nullptr;
    const uint32_t kind = parse_line(text + b, text + e, u, v, &tb, &te);
    pairs[k] = make_ulonglong2(u, v);
    is_edge[k] = kind == L_EDGE;
    if (kind >= L_BAD_TOKEN) atomicMin(first_bad, (unsigned long long)k);
  }
}

__global__ void endpoints_kernel(const ulonglong2* e, uint64_t m, uint64_t* ends) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    ends[2 * i] = e[i].x;
    ends[2 * i + 1] = e[i].y;
  }
}

__device__ __forceinline__ uint32_t rank_of(const uint64_t* ids, uint32_t n, uint64_t x) {
  uint32_t lo = 0, hi = n;  // lower_bound (graph.cpp:170-172)
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (ids[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void densify_kernel(const ulonglong2* e, uint64_t m, const uint64_t* ids, uint32_t n,
                               uint2* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = make_uint2(rank_of(ids, n, e[i].x), rank_of(ids, n, e[i].y));
}

thread_local std::string g_ingest_error;

struct DBuf {  // device buffer freed on scope exit
  void* p = nullptr;
  ~DBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 1); }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

kc_status cfail(cudaError_t e, const char* what) {
  cudaGetLastError();
  g_ingest_error = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? KC_ERR_OUT_OF_MEMORY : KC_ERR_CUDA;
}

#define IK(x)                                     \
  do {                                            \
    cudaError_t e_ = (x);                         \
    if (e_ != cudaSuccess) return cfail(e_, #x);  \
  } while (0)

void set_parse_error(kc_parse_error* err, uint64_t line, const std::string& what) {
  g_ingest_error = "line " + std::to_string(line) + ": " + what;
  if (!err) return;
  err->line = line;
  std::snprintf(err->what, sizeof(err->what), "%s", what.c_str());
}

// Word the error of line k (0-based) like ParseError (graph.cpp:56-79).
void describe(const char* text, uint64_t len, uint64_t b, uint64_t e, uint64_t k,
              kc_parse_error* err) {
  uint64_t u, v;
  const char *tb = nullptr, *te = nullptr;
  const uint32_t kind = parse_line(text + b, text + e, u, v, &tb, &te);
  (void)len;
  if (kind == L_BAD_TOKEN)
    set_parse_error(err, k + 1, "malformed token '" + std::string(tb, te) + "'");
  else if (kind == L_ONE_ID)
    set_parse_error(err, k + 1, "expected two ids, got one");
  else
    set_parse_error(err, k + 1, "expected two ids per line");
}

kc_status ingest(const char* host_text, uint64_t len, int device, kc_csr_dev** out,
                 kc_parse_error* err) {
  kcb::DeviceGuard device_guard;  // restore the caller's current device
  *out = nullptr;
  if (err) {
    err->line = 0;
    err->what[0] = 0;
  }
  int count = 0;  // no CPU fallback: the loader runs on the device or not at all
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0 || device < 0 || device >= count) {
    cudaGetLastError();
    g_ingest_error = "no CUDA device available (the B200 path has no CPU fallback)";
    return KC_ERR_NO_DEVICE;
  }
  IK(cudaSetDevice(device));
  cudaStream_t s = 0;
  const int G = 148 * 8, B = 256;
  DBuf text, starts, nsel, pairs, isedge, bad, edges, ends, ids, idsu, tmp, dense;
  uint64_t L = 0, m = 0, n = 0;
  if (len) {
    IK(text.alloc(len + 1));
    IK(cudaMemcpy(text.p, host_text, len, cudaMemcpyHostToDevice));
    IK(starts.alloc(len * sizeof(uint64_t)));
    IK(nsel.alloc(sizeof(uint64_t)));
    // line starts: position 0 and every position after a '\n'
    cub::CountingInputIterator<uint64_t> pos(0);
    size_t need = 0;
    IK(cub::DeviceSelect::If(nullptr, need, pos, starts.as<uint64_t>(), nsel.as<uint64_t>(),
                             (int64_t)len, LineStart{text.as<char>()}, s));
    IK(tmp.alloc(need));
    IK(cub::DeviceSelect::If(tmp.p, need, pos, starts.as<uint64_t>(), nsel.as<uint64_t>(),
                             (int64_t)len, LineStart{text.as<char>()}, s));
    IK(cudaMemcpy(&L, nsel.p, sizeof(L), cudaMemcpyDeviceToHost));
    cudaFree(tmp.p);
    tmp.p = nullptr;
    IK(pairs.alloc(L * sizeof(ulonglong2)));
    IK(isedge.alloc(L));
    IK(bad.alloc(sizeof(unsigned long long)));
    IK(cudaMemset(bad.p, 0xff, sizeof(unsigned long long)));
    parse_kernel<<<G, B, 0, s>>>(text.as<char>(), len, starts.as<uint64_t>(), L,
                                 pairs.as<ulonglong2>(), isedge.as<uint8_t>(),
                                 bad.as<unsigned long long>());
    IK(cudaGetLastError());
    unsigned long long first_bad = 0;
    IK(cudaMemcpy(&first_bad, bad.p, sizeof(first_bad), cudaMemcpyDeviceToHost));
    if (first_bad != ~0ull) {
      uint64_t se[2] = {0, len};
      IK(cudaMemcpy(&se[0], starts.as<uint64_t>() + first_bad, 8, cudaMemcpyDeviceToHost));
      if (first_bad + 1 < L) {
        IK(cudaMemcpy(&se[1], starts.as<uint64_t>() + first_bad + 1, 8, cudaMemcpyDeviceToHost));
        se[1] -= 1;
      } else if (se[1] > se[0] && host_text[se[1] - 1] == '\n') {
        se[1] -= 1;
      }
      describe(host_text, len, se[0], se[1], first_bad, err);
      return KC_ERR_PARSE;
    }
    // the lines that hold an edge, in line order
    IK(edges.alloc(L * sizeof(ulonglong2)));
    need = 0;
    IK(cub::DeviceSelect::Flagged(nullptr, need, pairs.as<ulonglong2>(), isedge.as<uint8_t>(),
                                  edges.as<ulonglong2>(), nsel.as<uint64_t>(), (int64_t)L, s));
    IK(tmp.alloc(need));
    IK(cub::DeviceSelect::Flagged(tmp.p, need, pairs.as<ulonglong2>(), isedge.as<uint8_t>(),
                                  edges.as<ulonglong2>(), nsel.as<uint64_t>(), (int64_t)L, s));
    IK(cudaMemcpy(&m, nsel.p, sizeof(m), cudaMemcpyDeviceToHost));
    cudaFree(tmp.p);
    tmp.p = nullptr;
  }
  kc_csr_dev* g = new (std::nothrow) kc_csr_dev();
  if (!g) return KC_ERR_OUT_OF_MEMORY;
  g->device = device;
  if (m == 0) {  // graph.cpp:142: no edges -> the empty graph
    uint64_t* off = nullptr;
    if (cudaMalloc(&off, sizeof(uint64_t)) != cudaSuccess ||
        cudaMemset(off, 0, sizeof(uint64_t)) != cudaSuccess) {
      delete g;
      return cfail(cudaErrorMemoryAllocation, "cudaMalloc");
    }
    g->view.offsets = off;
    *out = g;
    return KC_OK;
  }
  auto bail = [&](kc_status st) {
    kc_csr_dev_free(g);
    return st;
  };
  // densify (graph.cpp:141-182): ascending distinct ids, ranks by lower_bound
  const uint64_t m2 = 2 * m;
  if (ends.alloc(m2 * 8) != cudaSuccess || ids.alloc(m2 * 8) != cudaSuccess)
    return bail(cfail(cudaErrorMemoryAllocation, "cudaMalloc endpoints"));
  endpoints_kernel<<<G, B, 0, s>>>(edges.as<ulonglong2>(), m, ends.as<uint64_t>());
  size_t need = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, need, ends.as<uint64_t>(), ids.as<uint64_t>(), (int64_t)m2,
                                 0, 64, s);
  if (tmp.alloc(need) != cudaSuccess) return bail(cfail(cudaErrorMemoryAllocation, "cudaMalloc"));
  if (cub::DeviceRadixSort::SortKeys(tmp.p, need, ends.as<uint64_t>(), ids.as<uint64_t>(),
                                     (int64_t)m2, 0, 64, s) != cudaSuccess)
    return bail(cfail(cudaGetLastError(), "radix sort"));
  cudaFree(tmp.p);
  tmp.p = nullptr;
  if (idsu.alloc(m2 * 8) != cudaSuccess) return bail(cfail(cudaErrorMemoryAllocation, "cudaMalloc"));
  need = 0;
  cub::DeviceSelect::Unique(nullptr, need, ids.as<uint64_t>(), idsu.as<uint64_t>(),
                            nsel.as<uint64_t>(), (int64_t)m2, s);
  if (tmp.alloc(need) != cudaSuccess) return bail(cfail(cudaErrorMemoryAllocation, "cudaMalloc"));
  if (cub::DeviceSelect::Unique(tmp.p, need, ids.as<uint64_t>(), idsu.as<uint64_t>(),
                                nsel.as<uint64_t>(), (int64_t)m2, s) != cudaSuccess)
    return bail(cfail(cudaGetLastError(), "unique"));
  if (cudaMemcpy(&n, nsel.p, sizeof(n), cudaMemcpyDeviceToHost) != cudaSuccess)
    return bail(cfail(cudaGetLastError(), "cudaMemcpy"));
  if (n > 0xffffffffull) {  // graph.cpp:165-166
    set_parse_error(err, 0, "more than 2^32 distinct node ids");
    return bail(KC_ERR_PARSE);
  }
  if (dense.alloc(m * sizeof(uint2)) != cudaSuccess)
    return bail(cfail(cudaErrorMemoryAllocation, "cudaMalloc"));
  densify_kernel<<<G, B, 0, s>>>(edges.as<ulonglong2>(), m, idsu.as<uint64_t>(), (uint32_t)n,
                                 dense.as<uint2>());
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(cfail(cudaGetLastError(), "densify"));
  cudaFree(edges.p);
  edges.p = nullptr;
  cudaFree(ends.p);
  ends.p = nullptr;
  uint64_t* off = nullptr;
  uint32_t* nbr = nullptr;
  uint64_t nnz = 0;
  kc_status st = build_csr_dev_public((uint32_t)n, dense.as<uint2>(), m, s, &off, &nbr, &nnz);
  if (st != KC_OK) {
    g_ingest_error = gen_last_error();
    return bail(st);
  }
  g->view.n = (uint32_t)n;
  g->view.nnz = nnz;
  g->view.offsets = off;
  g->view.neighbors = nbr;
  g->original_ids = idsu.as<uint64_t>();  // dense id -> source id (n entries)
  idsu.p = nullptr;
  *out = g;
  return KC_OK;
}

}  // namespace

const char* ingest_last_error() { return g_ingest_error.c_str(); }

}  // namespace kcb

extern "C" {

kc_status kc_load_edge_list(const char* text, uint64_t len, int device, kc_csr_dev** out,
                            kc_parse_error* err) {
  if (!out || (len && !text)) return KC_ERR_INVALID_ARGUMENT;
  return kcb::ingest(text, len, device, out, err);
}

kc_status kc_load_edge_list_file(const char* path, int device, kc_csr_dev** out,
                                 kc_parse_error* err) {
  if (!out || !path) return KC_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  // kcore::load_edge_list_file (graph.cpp:200-226): gzopen reads gzip-compressed
  // and plain files alike; the same IoError messages
  gzFile gz = gzopen(path, "rb");
  if (!gz) {
    kcb::set_parse_error(err, 0, std::string("cannot open '") + path + "': " + std::strerror(errno));
    return KC_ERR_IO;
  }
  gzbuffer(gz, 1 << 20);
  std::vector<char> buf;
  std::vector<char> chunk(1 << 20);
  for (;;) {
    const int got = gzread(gz, chunk.data(), (unsigned)chunk.size());
    if (got < 0) {
      int errnum = 0;
      const char* msg = gzerror(gz, &errnum);
      kcb::set_parse_error(err, 0, std::string("error reading '") + path + "': " + msg);
      gzclose(gz);
      return KC_ERR_IO;
    }
    if (got == 0) break;
    buf.insert(buf.end(), chunk.data(), chunk.data() + got);
  }
  gzclose(gz);
  return kcb::ingest(buf.data(), buf.size(), device, out, err);
}

kc_status kc_csr_dev_original_ids(const kc_csr_dev* g, uint64_t* ids) {
  kcb::DeviceGuard device_guard;  // restore the caller's current device
  if (!g || (g->view.n && !ids)) return KC_ERR_INVALID_ARGUMENT;
  if (!g->view.n) return KC_OK;
  if (cudaSetDevice(g->device) != cudaSuccess) return KC_ERR_CUDA;
  if (!g->original_ids) {  // generated graphs: identity
    for (uint32_t i = 0; i < g->view.n; ++i) ids[i] = i;
    return KC_OK;
  }
  return cudaMemcpy(ids, g->original_ids, (size_t)g->view.n * 8, cudaMemcpyDeviceToHost) ==
                 cudaSuccess
             ? KC_OK
             : KC_ERR_CUDA;
}

}  // extern "C"
