// ref_shim.cpp — extern "C" wrappers around the UNMODIFIED reference library
// compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libkcore_ref.so.  TEST/BASELINE INFRASTRUCTURE ONLY: loaded by
// tests/ (to pin oracle/kc_oracle.c) and by bench.py's --impl reference /
// cpu_baseline leg, never by the product.
//
// kcore::Graph keeps its CSR private (include/kcore/graph.hpp:66-74) and the
// only public builder is the single-threaded Graph::from_edges
// (graph.hpp:43-44, src/graph.cpp:130-137).  For large graphs we install an
// already-built CSR directly through the standard explicit-instantiation
// member-access idiom, so the reference's own fastk_run / peel_coreness run on
// the byte-identical CSR the GPU sees.  Small graphs can still go through
// from_edges (ref_graph_from_edges) to exercise the reference builder.
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "kcore/fastk.hpp"
#include "kcore/graph.hpp"
#include "kcore/kernel.hpp"
#include "kcore/oracle.hpp"
#include "kcore/report.hpp"

namespace {

template <class Tag, typename Tag::type M>
struct Rob {
  friend typename Tag::type get(Tag) { return M; }
};
struct NodeCountTag { using type = std::uint32_t kcore::Graph::*; friend type get(NodeCountTag); };
struct EdgeCountTag { using type = std::uint64_t kcore::Graph::*; friend type get(EdgeCountTag); };
struct OffsetsTag { using type = std::vector<std::uint64_t> kcore::Graph::*; friend type get(OffsetsTag); };
struct NeighborsTag { using type = std::vector<kcore::NodeId> kcore::Graph::*; friend type get(NeighborsTag); };
struct OrigTag { using type = std::vector<std::uint64_t> kcore::Graph::*; friend type get(OrigTag); };
template struct Rob<NodeCountTag, &kcore::Graph::node_count_>;
template struct Rob<EdgeCountTag, &kcore::Graph::edge_count_>;
template struct Rob<OffsetsTag, &kcore::Graph::offsets_>;
template struct Rob<NeighborsTag, &kcore::Graph::neighbors_>;
template struct Rob<OrigTag, &kcore::Graph::original_ids_>;

struct RefStats {
  std::uint64_t iterations, messages_sent, messages_drained, tail_pops;
};

void fill(const kcore::EngineResult& r, std::uint32_t* core, RefStats* st) {
  if (core && !r.result.coreness.empty())
    std::memcpy(core, r.result.coreness.data(), r.result.coreness.size() * sizeof(std::uint32_t));
  if (st) {
    st->iterations = r.report.iterations;
    st->messages_sent = r.report.messages_sent;
    st->messages_drained = r.report.messages_drained;
    st->tail_pops = r.report.tail_pops;
  }
}

}  // namespace

extern "C" {

// Install a CSR (offsets n+1, neighbours offsets[n]) as a kcore::Graph.
void* ref_graph_from_csr(std::uint32_t n, const std::uint64_t* off, const std::uint32_t* nbr) {
  auto* g = new kcore::Graph();
  g->*get(NodeCountTag{}) = n;
  g->*get(OffsetsTag{}) = std::vector<std::uint64_t>(off, off + n + 1);
  g->*get(NeighborsTag{}) = std::vector<kcore::NodeId>(nbr, nbr + off[n]);
  g->*get(EdgeCountTag{}) = off[n] / 2;
  std::vector<std::uint64_t> ids(n);
  for (std::uint32_t i = 0; i < n; ++i) ids[i] = i;
  g->*get(OrigTag{}) = std::move(ids);
  return g;
}

// Build through the reference's own from_edges (graph.cpp:130-137 → build_csr 85-128).
void* ref_graph_from_edges(std::uint32_t n, const std::uint32_t* pairs, std::uint64_t m) {
  std::vector<std::pair<kcore::NodeId, kcore::NodeId>> e(m);
  for (std::uint64_t i = 0; i < m; ++i) e[i] = {pairs[2 * i], pairs[2 * i + 1]};
  return new kcore::Graph(kcore::Graph::from_edges(n, e));
}

void ref_graph_free(void* g) { delete static_cast<kcore::Graph*>(g); }

// kcore::load_edge_list (graph.cpp:186-199) over an in-memory text.  Returns
// null on ParseError / IoError with the message in err and the line in *line.
void* ref_load_edge_list(const char* text, std::uint64_t len, char* err, std::uint64_t errcap,
                         std::uint64_t* line) {
  try {
    std::istringstream in(std::string(text, len));
    return new kcore::Graph(kcore::load_edge_list(in));
  } catch (const kcore::ParseError& e) {
    std::snprintf(err, errcap, "%s", e.what());
    *line = e.line();
  } catch (const std::exception& e) {
    std::snprintf(err, errcap, "%s", e.what());
    *line = 0;
  }
  return nullptr;
}

std::uint32_t ref_graph_n(const void* g) { return static_cast<const kcore::Graph*>(g)->node_count(); }

void ref_graph_original_ids(const void* gp, std::uint64_t* out) {
  const auto* g = static_cast<const kcore::Graph*>(gp);
  for (std::uint32_t u = 0; u < g->node_count(); ++u) out[u] = g->original_id(u);
}

std::uint64_t ref_graph_nnz(const void* g) {
  return static_cast<const kcore::Graph*>(g)->offsets().back();
}

// Copy the reference-built CSR out (offsets n+1, neighbours nnz).
void ref_graph_csr(const void* gp, std::uint64_t* off, std::uint32_t* nbr) {
  const auto* g = static_cast<const kcore::Graph*>(gp);
  const auto& o = g->offsets();
  std::memcpy(off, o.data(), o.size() * sizeof(std::uint64_t));
  if (g->node_count() > 0 && o.back() > 0)
    std::memcpy(nbr, g->neighbors(0).data(), o.back() * sizeof(std::uint32_t));
}

// kcore::peel_coreness (src/oracle.cpp:21-66).  Returns k_max.
std::uint32_t ref_peel(const void* g, std::uint32_t* core, double* k_avg) {
  kcore::CorenessResult r = kcore::peel_coreness(*static_cast<const kcore::Graph*>(g));
  if (!r.coreness.empty()) std::memcpy(core, r.coreness.data(), r.coreness.size() * 4);
  if (k_avg) *k_avg = r.k_avg;
  return r.k_max;
}

// kcore::fastk_run (src/fastk.cpp:57-187).  Returns 0, or -1 when the
// reference threw std::invalid_argument (threads/batch == 0).
int ref_fastk(const void* g, unsigned threads, std::uint32_t batch, int ext, int hybrid,
              std::uint32_t* core, RefStats* st) {
  kcore::FastKOptions o;
  o.threads = threads;
  o.batch = batch;
  o.extended_notify = ext != 0;
  o.hybrid_tail = hybrid != 0;
  try {
    fill(kcore::fastk_run(*static_cast<const kcore::Graph*>(g), o), core, st);
  } catch (const std::invalid_argument&) {
    return -1;
  }
  return 0;
}

// fastk_run with an Instrumentation inspector (report.hpp:33-39): records
// every boundary's estimate snapshot and active count.  snaps has room for
// max_snap * n values; returns the number of boundaries observed.
std::uint64_t ref_fastk_observed(const void* gp, unsigned threads, std::uint32_t batch, int ext,
                                 int hybrid, std::uint32_t* core, RefStats* st,
                                 std::uint32_t* snaps, std::uint64_t* actives,
                                 std::uint64_t max_snap) {
  const auto* g = static_cast<const kcore::Graph*>(gp);
  const std::uint32_t n = g->node_count();
  std::uint64_t seen = 0;
  kcore::Instrumentation instr;
  instr.inspector = [&](std::uint64_t, std::span<const std::uint32_t> est, std::uint64_t active) {
    if (seen < max_snap) {
      if (n) std::memcpy(snaps + seen * n, est.data(), n * sizeof(std::uint32_t));
      actives[seen] = active;
    }
    ++seen;
  };
  kcore::FastKOptions o;
  o.threads = threads;
  o.batch = batch;
  o.extended_notify = ext != 0;
  o.hybrid_tail = hybrid != 0;
  fill(kcore::fastk_run(*g, o, &instr), core, st);
  return seen;
}

// fastk_run with trace_convergence (report.cpp:7-18): mean_error and
// active_fraction per boundary, as the kcbench trace command prints them.
std::uint64_t ref_fastk_trace(const void* gp, unsigned threads, std::uint32_t batch, int ext,
                              int hybrid, double* mean_err, double* active_frac,
                              std::uint64_t max_rows) {
  const auto* g = static_cast<const kcore::Graph*>(gp);
  kcore::CorenessResult truth = kcore::peel_coreness(*g);
  kcore::Instrumentation instr;
  instr.truth = &truth;
  instr.trace_convergence = true;
  kcore::FastKOptions o;
  o.threads = threads;
  o.batch = batch;
  o.extended_notify = ext != 0;
  o.hybrid_tail = hybrid != 0;
  kcore::EngineResult r = kcore::fastk_run(*g, o, &instr);
  std::uint64_t k = 0;
  for (const auto& row : r.report.trace) {
    if (k < max_rows) {
      mean_err[k] = row.mean_error;
      active_frac[k] = row.active_fraction;
    }
    ++k;
  }
  return k;
}

// kcore::compute_index (src/kernel.cpp:7-16 → kernel.hpp:27-42).
std::uint32_t ref_compute_index(const std::uint32_t* est, std::uint64_t count, std::uint32_t cap) {
  return kcore::compute_index(std::span<const std::uint32_t>(est, count), cap);
}

int ref_should_notify(std::uint32_t nc, std::uint32_t oc, std::uint32_t ev) {
  return kcore::should_notify(nc, oc, ev) ? 1 : 0;
}

int ref_switch_condition(std::uint64_t active, std::uint32_t batch) {
  return kcore::switch_condition(active, batch) ? 1 : 0;
}

// kcore::sequential_tail (src/fastk.cpp:28-55) on caller-provided state.
void ref_sequential_tail(const void* gp, std::uint32_t* est, std::uint8_t* active, int ext,
                         RefStats* st) {
  const auto* g = static_cast<const kcore::Graph*>(gp);
  const std::uint32_t n = g->node_count();
  std::vector<std::uint32_t> e(est, est + n);
  kcore::ActiveFlags flags(n);
  for (std::uint32_t i = 0; i < n; ++i) flags[i].store(active[i]);
  kcore::RunReport rep;
  kcore::sequential_tail(*g, e, flags, ext != 0, rep);
  std::memcpy(est, e.data(), n * sizeof(std::uint32_t));
  for (std::uint32_t i = 0; i < n; ++i) active[i] = flags[i].load();
  st->iterations = rep.iterations;
  st->messages_sent = rep.messages_sent;
  st->messages_drained = rep.messages_drained;
  st->tail_pops = rep.tail_pops;
}

}  // extern "C"
