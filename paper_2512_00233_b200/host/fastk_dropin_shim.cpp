// fastk_dropin_shim.cpp — link-time drop-in: compile this INSTEAD of the
// reference's src/fastk.cpp and every existing caller of kcore::fastk_run
// (src/bench.cpp:138-144, tests, acceptance) and of kcore::sequential_tail
// (tests/test_fastk.cpp:318-370) runs on the B200.  These are the two
// out-of-line functions fastk.hpp declares (46-47, 38-39); should_notify and
// switch_condition are inline in the header.
//
// Which GPU rule the drop-in uses is a build-time choice, because it decides
// what the RunReport counters mean (report.hpp:17-23):
//   default                            Rule::Reference — the reference's own
//       activation rule and hybrid sequential tail: coreness AND every counter
//       (iterations, messages_sent, messages_drained, tail_pops) equal
//       kcore::fastk_run's, so the reference's own tests pass unchanged
//       (tests/cpp/test_shim.cpp re-expresses test_fastk.cpp against it).
//   -DKCORE_GPU_DROPIN_COUNTING        Rule::Counting — the fast support-counter
//       rule: the same coreness, but `batch` / `hybrid_tail` are ignored,
//       tail_pops is 0, messages_sent counts support decrements and
//       messages_drained counts only evaluations of vertices that drop
//       (INTEGRATION.md §1).
#include "kcore_gpu.hpp"

namespace kcore {
namespace {
#ifdef KCORE_GPU_DROPIN_COUNTING
constexpr gpu::Rule kDropinRule = gpu::Rule::Counting;
#else
constexpr gpu::Rule kDropinRule = gpu::Rule::Reference;
#endif
}  // namespace

EngineResult fastk_run(const Graph& g, const FastKOptions& options, const Instrumentation* instr) {
  return gpu::fastk_run(g, options, instr, kDropinRule);
}

void sequential_tail(const Graph& g, std::vector<std::uint32_t>& est, ActiveFlags& active,
                     bool extended_notify, RunReport& report) {
  gpu::sequential_tail(g, est, active, extended_notify, report);
}
}  // namespace kcore
