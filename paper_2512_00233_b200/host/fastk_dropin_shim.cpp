// fastk_dropin_shim.cpp — link-time drop-in: compile this INSTEAD of the
// reference's src/fastk.cpp and every existing caller of kcore::fastk_run
// (src/bench.cpp:138-144, tests, acceptance) and of kcore::sequential_tail
// (tests/test_fastk.cpp:318-370) runs on the B200.  These are the two
// out-of-line functions fastk.hpp declares (46-47, 38-39); should_notify and
// switch_condition are inline in the header.
#include "kcore_gpu.hpp"

namespace kcore {
EngineResult fastk_run(const Graph& g, const FastKOptions& options, const Instrumentation* instr) {
  return gpu::fastk_run(g, options, instr);
}

void sequential_tail(const Graph& g, std::vector<std::uint32_t>& est, ActiveFlags& active,
                     bool extended_notify, RunReport& report) {
  gpu::sequential_tail(g, est, active, extended_notify, report);
}
}  // namespace kcore
