// fastk_dropin_shim.cpp — link-time drop-in: compile this INSTEAD of the
// reference's src/fastk.cpp and every existing caller of kcore::fastk_run
// (src/bench.cpp:138-144, tests, acceptance) runs on the B200.
// (sequential_tail, fastk.cpp:28-55, is a CPU helper of the reference engine
// and has no GPU counterpart; builds that need it keep fastk.cpp and call
// kcore::gpu::fastk_run directly.)
#include "kcore_gpu.hpp"

namespace kcore {
EngineResult fastk_run(const Graph& g, const FastKOptions& options, const Instrumentation* instr) {
  return gpu::fastk_run(g, options, instr);
}
}  // namespace kcore
