// kcore_gpu.hpp — C++ drop-in for the reference's FastK entry point.
//
//   kcore::EngineResult kcore::gpu::fastk_run(const kcore::Graph&,
//                                             const kcore::FastKOptions&,
//                                             const kcore::Instrumentation*);
//
// Same signature, argument meaning and error behaviour as kcore::fastk_run
// (/root/reference/proj/include/kcore/fastk.hpp:46-47, src/fastk.cpp:57-187):
// std::invalid_argument for zero threads or batch before any work
// (fastk.cpp:58-59), Instrumentation hooks at every iteration boundary
// (report.hpp:33-39).  The work runs on the B200 through the C-ABI in
// include/kcore_b200.h; C-ABI failures surface as std::runtime_error
// (std::bad_alloc for device OOM).  Compiles against the reference's own
// headers — it is the file a maintainer adds to the reference build.
#pragma once

#include <vector>

#include "kcore/fastk.hpp"
#include "kcore/graph.hpp"
#include "kcore/oracle.hpp"
#include "kcore/report.hpp"

namespace kcore::gpu {

// Which re-evaluation rule the GPU uses (kc_rule): the reference's own
// (exact RunReport counters when hybrid_tail is off) or support counters.
enum class Rule { Reference = 0, Counting = 1, Auto = 2 };

EngineResult fastk_run(const Graph& g, const FastKOptions& options = {},
                       const Instrumentation* instr = nullptr, Rule rule = Rule::Auto);

// kcore::sequential_tail (include/kcore/fastk.hpp:38-39) on the B200: same
// signature and effect (estimates lowered, flags cleared, pops / drained /
// sent added to the report).
void sequential_tail(const Graph& g, std::vector<std::uint32_t>& est, ActiveFlags& active,
                     bool extended_notify, RunReport& report);

// kcore::peel_coreness (include/kcore/oracle.hpp:19-22) computed on the B200
// by an independent algorithm (kc_peel: level-synchronous parallel peel).
CorenessResult peel_coreness(const Graph& g);

// kcore::verify(fastk_run(g, options), peel_coreness(g)) (oracle.hpp:29-31)
// with both results and the comparison on the device: only mismatches
// (ascending node id) come back.
std::vector<Mismatch> verify_fastk(const Graph& g, const FastKOptions& options = {},
                                   Rule rule = Rule::Auto);

}  // namespace kcore::gpu
