// kcore_gpu.cpp — see kcore_gpu.hpp.  Host-side adapter over the C-ABI.
#include "kcore_gpu.hpp"

#include <cstring>
#include <new>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "kcore/oracle.hpp"
#include "kcore_b200.h"

namespace kcore::gpu {

namespace {

[[noreturn]] void raise(kc_status s, const char* where) {
  const std::string msg = std::string(where) + ": " + kc_status_str(s) + " (" + kc_last_error() + ")";
  if (s == KC_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (s == KC_ERR_OUT_OF_MEMORY) throw std::bad_alloc();
  throw std::runtime_error(msg);
}

kc_csr_view view_of(const Graph& g) {
  kc_csr_view view{};
  view.n = g.node_count();
  view.nnz = g.offsets().back();
  view.offsets = g.offsets().data();
  view.neighbors = (view.n > 0 && view.nnz > 0) ? g.neighbors(0).data() : nullptr;
  return view;
}

// Owns a kc_graph handle for the duration of one call.
struct Handle {
  kc_graph* h = nullptr;
  explicit Handle(const Graph& g, uint32_t flags) {
    const kc_csr_view view = view_of(g);
    kc_status s = kc_graph_upload_ex(&view, 0, 0, flags, &h);
    if (s != KC_OK) raise(s, "kc_graph_upload_ex");
  }
  ~Handle() { kc_graph_free(h); }
};

struct HookCtx {
  RunReport* report;
  const Instrumentation* instr;
};

// Engines call instrument_boundary (report.cpp:20-29) at every boundary;
// the C-ABI inspector delivers exactly those boundaries.
int on_boundary(void* user, uint64_t iteration, const uint32_t* est, uint32_t n,
                uint64_t active) {
  auto* c = static_cast<HookCtx*>(user);
  instrument_boundary(*c->report, c->instr, iteration, std::span<const uint32_t>(est, n), active);
  return 0;
}

}  // namespace

EngineResult fastk_run(const Graph& g, const FastKOptions& opt, const Instrumentation* instr,
                       Rule rule) {
  if (opt.threads == 0) throw std::invalid_argument("fastk: threads must be >= 1");
  if (opt.batch == 0) throw std::invalid_argument("fastk: batch must be >= 1");

  const uint32_t n = g.node_count();
  kc_csr_view view{};
  view.n = n;
  view.nnz = g.offsets().back();
  view.offsets = g.offsets().data();
  // neighbors(0) is only valid when n > 0 (offsets_ == {0} for the empty graph)
  view.neighbors = (n > 0 && view.nnz > 0) ? g.neighbors(0).data() : nullptr;

  kc_options o;
  kc_default_options(&o);
  o.threads = opt.threads;
  o.batch = opt.batch;
  o.extended_notify = opt.extended_notify ? 1 : 0;
  o.hybrid_tail = opt.hybrid_tail ? 1 : 0;
  o.rule = static_cast<int32_t>(rule);

  EngineResult out;
  std::vector<uint32_t> core(n);
  kc_stats st{};
  kc_graph* h = nullptr;
  // one solve per call: unsorted rows (the row sort costs more than it saves)
  kc_status s = kc_graph_upload_ex(&view, 0, 0, KC_UPLOAD_UNSORTED_ROWS, &h);
  if (s != KC_OK) raise(s, "kc_graph_upload_ex");
  const bool observed = instr && (instr->trace_convergence || instr->inspector);
  if (observed && !instr->inspector) {
    // trace only: record_iteration's rows reduced on the device
    if (!instr->truth) {
      kc_graph_free(h);
      throw std::invalid_argument("fastk: trace_convergence requires truth");
    }
    std::vector<kc_iteration_stat> rows(4096);
    uint64_t nrows = 0;
    s = kc_solve_traced(h, &o, instr->truth->coreness.data(), rows.data(), rows.size(), &nrows,
                        core.data(), &st);
    if (s == KC_OK && nrows > rows.size()) {
      rows.resize(nrows);
      s = kc_solve_traced(h, &o, instr->truth->coreness.data(), rows.data(), rows.size(), &nrows,
                          core.data(), &st);
    }
    for (uint64_t i = 0; s == KC_OK && i < nrows; ++i)
      out.report.trace.push_back(IterationStat{rows[i].mean_error, rows[i].active_fraction});
  } else if (observed) {
    HookCtx ctx{&out.report, instr};
    s = kc_solve_observed(h, &o, &on_boundary, &ctx, core.data(), &st);
  } else {
    s = kc_solve(h, &o, core.data(), &st);
  }
  kc_graph_free(h);
  if (s != KC_OK) raise(s, "kc_solve");

  out.report.iterations = st.iterations;
  out.report.messages_sent = st.messages_sent;
  out.report.messages_drained = st.messages_drained;
  out.report.tail_pops = st.tail_pops;
  out.result.coreness = std::move(core);
  out.result.k_max = st.k_max;
  out.result.k_avg = st.k_avg;
  return out;
}

CorenessResult peel_coreness(const Graph& g) {
  const uint32_t n = g.node_count();
  std::vector<uint32_t> core(n);
  if (n == 0) return make_coreness_result(std::move(core));
  Handle h(g, KC_UPLOAD_UNSORTED_ROWS);
  kc_stats st{};
  kc_status s = kc_peel(h.h, core.data(), &st);
  if (s != KC_OK) raise(s, "kc_peel");
  return make_coreness_result(std::move(core));
}

std::vector<Mismatch> verify_fastk(const Graph& g, const FastKOptions& opt, Rule rule) {
  if (opt.threads == 0) throw std::invalid_argument("fastk: threads must be >= 1");
  if (opt.batch == 0) throw std::invalid_argument("fastk: batch must be >= 1");
  std::vector<Mismatch> out;
  if (g.node_count() == 0) return out;
  kc_options o;
  kc_default_options(&o);
  o.threads = opt.threads;
  o.batch = opt.batch;
  o.extended_notify = opt.extended_notify ? 1 : 0;
  o.hybrid_tail = opt.hybrid_tail ? 1 : 0;
  o.rule = static_cast<int32_t>(rule);
  Handle h(g, 0);
  uint64_t count = 0;
  std::vector<kc_mismatch> mm(1024);
  kc_status s = kc_verify(h.h, &o, mm.data(), mm.size(), &count);
  if (s == KC_OK && count > mm.size()) {
    mm.resize(count);
    s = kc_verify(h.h, &o, mm.data(), mm.size(), &count);
  }
  if (s != KC_OK) raise(s, "kc_verify");
  for (uint64_t i = 0; i < count; ++i) out.push_back({mm[i].node, mm[i].candidate, mm[i].truth});
  return out;
}

void sequential_tail(const Graph& g, std::vector<std::uint32_t>& est, ActiveFlags& active,
                     bool extended_notify, RunReport& report) {
  const uint32_t n = g.node_count();
  if (n == 0) return;
  std::vector<uint8_t> flags(n);
  for (uint32_t u = 0; u < n; ++u) flags[u] = active[u].load(std::memory_order_relaxed);
  Handle h(g, KC_UPLOAD_UNSORTED_ROWS);
  kc_stats st{};
  kc_status s = kc_sequential_tail(h.h, est.data(), flags.data(), extended_notify ? 1 : 0, &st);
  if (s != KC_OK) raise(s, "kc_sequential_tail");
  for (uint32_t u = 0; u < n; ++u) active[u].store(flags[u], std::memory_order_relaxed);
  report.tail_pops += st.tail_pops;
  report.messages_drained += st.messages_drained;
  report.messages_sent += st.messages_sent;
}

}  // namespace kcore::gpu
