// test_dropin.cpp — the C++ drop-in kcore::gpu::fastk_run (B200) against the
// reference library itself: kcore::peel_coreness (src/oracle.cpp:21-66) and
// the reference CPU kcore::fastk_run (src/fastk.cpp:57-187), through the
// reference's own types.  Cases follow tests/test_fastk.cpp of the reference
// (written fresh; no doctest in this image, so a minimal CHECK harness).
// Exit code 0 = all checks passed.  Needs a B200 (run by tests/test_dropin.py).
#include <cstdint>
#include <cstdio>
#include <functional>
#include <random>
#include <stdexcept>
#include <vector>

#include "kcore/fastk.hpp"
#include "kcore/graph.hpp"
#include "kcore/oracle.hpp"
#include "kcore/report.hpp"
#include "kcore_gpu.hpp"

using namespace kcore;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                             \
  do {                                                                          \
    ++g_checks;                                                                 \
    if (!(cond)) {                                                              \
      ++g_fail;                                                                 \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                           \
  } while (0)

static Graph make(uint32_t n, std::vector<std::pair<NodeId, NodeId>> e) {
  return Graph::from_edges(n, e);
}

static Graph gnp(std::mt19937_64& rng, uint32_t n, double p) {
  std::bernoulli_distribution coin(p);
  std::vector<std::pair<NodeId, NodeId>> e;
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t j = i + 1; j < n; ++j)
      if (coin(rng)) e.push_back({i, j});
  return make(n, e);
}

static FastKOptions opts(unsigned t, uint32_t b, bool ext = true, bool hybrid = true) {
  FastKOptions o;
  o.threads = t;
  o.batch = b;
  o.extended_notify = ext;
  o.hybrid_tail = hybrid;
  return o;
}

int main() {
  const gpu::Rule R = gpu::Rule::Reference, C = gpu::Rule::Counting;

  {  // triangle (test_fastk.cpp:147-154)
    Graph t = make(3, {{0, 1}, {1, 2}, {0, 2}});
    EngineResult r = gpu::fastk_run(t, opts(4, 1, true, false), nullptr, R);
    CHECK((r.result.coreness == std::vector<uint32_t>{2, 2, 2}));
    CHECK(r.report.iterations == 1);
    CHECK(r.report.messages_sent == 0);
    CHECK(r.report.messages_drained == 3);
    CHECK(r.report.tail_pops == 0);
    CHECK(r.result.k_max == 2);
  }
  {  // invalid arguments (test_fastk.cpp:142-145)
    Graph t = make(3, {{0, 1}, {1, 2}, {0, 2}});
    bool threw = false;
    try { gpu::fastk_run(t, opts(0, 256)); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    threw = false;
    try { gpu::fastk_run(t, opts(4, 0)); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
  }
  {  // empty and edgeless (test_fastk.cpp:156-164)
    EngineResult e = gpu::fastk_run(Graph(), opts(3, 8));
    CHECK(e.result.coreness.empty());
    CHECK(e.report.iterations == 1);
    EngineResult l = gpu::fastk_run(make(4, {}), opts(2, 2));
    CHECK((l.result.coreness == std::vector<uint32_t>(4, 0)));
    CHECK(l.report.messages_sent == 0);
  }
  {  // every labeled graph up to 5 nodes (test_fastk.cpp:181-188)
    for (uint32_t n = 1; n <= 5; ++n) {
      std::vector<std::pair<NodeId, NodeId>> pairs;
      for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = i + 1; j < n; ++j) pairs.push_back({i, j});
      for (uint64_t mask = 0; mask < (1ull << pairs.size()); mask += (n == 5 ? 3 : 1)) {
        std::vector<std::pair<NodeId, NodeId>> e;
        for (size_t b = 0; b < pairs.size(); ++b)
          if (mask >> b & 1) e.push_back(pairs[b]);
        Graph g = make(n, e);
        CHECK(gpu::fastk_run(g, opts(2, 1), nullptr, C).result.coreness ==
              peel_coreness(g).coreness);
      }
    }
  }
  {  // random graphs x options; counters equal the reference CPU engine
    std::mt19937_64 rng(403);
    for (int rep = 0; rep < 8; ++rep) {
      Graph g = gnp(rng, 64 + 16 * rep, 0.09);
      CorenessResult truth = peel_coreness(g);
      for (bool ext : {false, true}) {
        for (gpu::Rule rule : {R, C}) {
          EngineResult r = gpu::fastk_run(g, opts(3, 4, ext, true), nullptr, rule);
          CHECK(verify(r.result, truth).empty());
          CHECK(r.result.k_max == truth.k_max);
        }
        EngineResult mine = gpu::fastk_run(g, opts(3, 4, ext, false), nullptr, R);
        EngineResult cpu = kcore::fastk_run(g, opts(3, 4, ext, false));
        CHECK(mine.report.iterations == cpu.report.iterations);
        CHECK(mine.report.messages_sent == cpu.report.messages_sent);
        CHECK(mine.report.messages_drained == cpu.report.messages_drained);
      }
    }
  }
  {  // no lost updates: inspector snapshots equal the reference engine's
    std::mt19937_64 rng(407);
    for (int rep = 0; rep < 4; ++rep) {
      Graph g = gnp(rng, 60 + rep * 20, 0.08);
      for (bool ext : {false, true}) {
        std::vector<std::vector<uint32_t>> sg, sc;
        std::vector<uint64_t> ag, ac;
        Instrumentation ig, ic;
        ig.inspector = [&](uint64_t, std::span<const uint32_t> e, uint64_t a) {
          sg.emplace_back(e.begin(), e.end());
          ag.push_back(a);
        };
        ic.inspector = [&](uint64_t, std::span<const uint32_t> e, uint64_t a) {
          sc.emplace_back(e.begin(), e.end());
          ac.push_back(a);
        };
        gpu::fastk_run(g, opts(3, 8, ext, false), &ig, R);
        kcore::fastk_run(g, opts(3, 8, ext, false), &ic);
        CHECK(sg == sc);
        CHECK(ag == ac);
      }
    }
  }
  {  // convergence trace through the reference's record_iteration
    Graph star = make(5, {{0, 1}, {0, 2}, {0, 3}, {0, 4}});
    CorenessResult truth = peel_coreness(star);
    Instrumentation it;
    it.truth = &truth;
    it.trace_convergence = true;
    EngineResult g = gpu::fastk_run(star, opts(4, 256), &it);
    EngineResult c = kcore::fastk_run(star, opts(4, 256), &it);
    CHECK(g.report.trace.size() == c.report.trace.size());
    for (size_t i = 0; i < g.report.trace.size() && i < c.report.trace.size(); ++i) {
      CHECK(g.report.trace[i].mean_error == c.report.trace[i].mean_error);
      CHECK(g.report.trace[i].active_fraction == c.report.trace[i].active_fraction);
    }
  }
  {  // bit-identical across threads, batches, repetitions (test_fastk.cpp:205-230)
    std::mt19937_64 rng(405);
    Graph g = gnp(rng, 150, 0.05);
    EngineResult base = gpu::fastk_run(g, opts(1, 64));
    CHECK(base.result.coreness == peel_coreness(g).coreness);
    for (unsigned t : {1u, 2u, 4u, 8u, 16u})
      for (uint32_t b : {1u, 64u, 256u, 4096u})
        CHECK(gpu::fastk_run(g, opts(t, b)).result.coreness == base.result.coreness);
  }
  {  // the independent device peel and device verify vs the reference peel
    std::mt19937_64 rng(77);
    for (int i = 0; i < 40; ++i) {
      Graph g = gnp(rng, 20 + 7 * i, 0.02 + 0.01 * (i % 9));
      const CorenessResult want = peel_coreness(g);
      const CorenessResult got = gpu::peel_coreness(g);
      CHECK(got.coreness == want.coreness);
      CHECK(got.k_max == want.k_max && got.k_avg == want.k_avg);
      CHECK(gpu::verify_fastk(g).empty());
      CHECK(gpu::verify_fastk(g, opts(4, 8), R).empty());
    }
    CHECK(gpu::peel_coreness(Graph()).coreness.empty());
  }
  {  // sequential_tail (tests/test_fastk.cpp:318-370): the B200 tail vs the reference's
    auto flags = [](std::vector<uint8_t> v) {
      ActiveFlags f(v.size());
      for (size_t i = 0; i < v.size(); ++i) f[i].store(v[i]);
      return f;
    };
    auto run_both = [&](const Graph& g, std::vector<uint32_t> est, std::vector<uint8_t> act,
                        bool ext) {
      std::vector<uint32_t> e1 = est, e2 = est;
      ActiveFlags a1 = flags(act), a2 = flags(act);
      RunReport r1, r2;
      sequential_tail(g, e1, a1, ext, r1);
      gpu::sequential_tail(g, e2, a2, ext, r2);
      CHECK(e1 == e2);
      CHECK(r1.tail_pops == r2.tail_pops);
      CHECK(r1.messages_drained == r2.messages_drained);
      CHECK(r1.messages_sent == r2.messages_sent);
      for (size_t u = 0; u < act.size(); ++u) CHECK(a2[u].load() == 0);
    };
    Graph k4p = make(5, {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}, {3, 4}});
    run_both(k4p, {3, 3, 3, 3, 1}, {1, 1, 1, 1, 1}, true);  // settled: 5 pops, nothing re-entered
    run_both(k4p, {9, 9, 9, 9, 9}, {0, 0, 0, 0, 0}, true);  // no active node: no-op
    run_both(make(3, {{0, 1}, {1, 2}}), {1, 2, 2}, {0, 1, 1}, true);  // re-push + stale pop
    std::mt19937_64 rng(417);
    for (int rep = 0; rep < 30; ++rep) {
      Graph g = gnp(rng, 40 + 5 * rep, 0.08);
      std::vector<uint32_t> est(g.node_count());
      std::vector<uint8_t> act(g.node_count());
      std::uniform_int_distribution<uint32_t> big(0, 200000);
      for (NodeId u = 0; u < g.node_count(); ++u) {
        est[u] = rep % 3 == 0 ? g.degree(u) : (rep % 3 == 1 ? big(rng) : g.degree(u) / 2);
        act[u] = (rng() & 3) != 0;
      }
      run_both(g, est, act, rep % 2 == 0);
    }
  }
  std::printf("test_dropin: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
