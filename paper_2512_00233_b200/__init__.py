"""B200-native FastK coreness (arXiv 2512.00233 path) behind the reference API.

Host-side mirror of the reference's C++ interface for this path
(/root/reference/proj/include/kcore/{graph,fastk,oracle,report}.hpp) over the
C-ABI in include/kcore_b200.h (libkcore_b200.so, sm_100a):

    Graph.from_edges(n, edges)          graph.hpp:43-44 / graph.cpp:85-137
    FastKOptions(threads, batch, extended_notify, hybrid_tail)   fastk.hpp:12-22
    fastk_run(g, options, instr) -> EngineResult                 fastk.hpp:46-47
    EngineResult.result: CorenessResult(coreness, k_max, k_avg)  oracle.hpp:10-14
    EngineResult.report: RunReport(iterations, messages_sent,
                         messages_drained, tail_pops, trace)     report.hpp:17-28
    Instrumentation(truth, trace_convergence, inspector)         report.hpp:33-39
    should_notify / switch_condition                             fastk.hpp:25-31

Error behaviour follows the reference: zero threads or batch raise ValueError
(std::invalid_argument, fastk.cpp:58-59) before any work.  There is no CPU
fallback: without the built library or an sm_100 device every solve raises.
"""
from .api import (  # noqa: F401
    CorenessResult,
    DeviceCSR,
    EngineResult,
    FastKOptions,
    GpuGraph,
    Graph,
    Instrumentation,
    IterationStat,
    KCError,
    RunReport,
    Rule,
    fastk_run,
    fastk_run_abi,
    IoError,
    ParseError,
    gen_config,
    load_edge_list,
    load_edge_list_file,
    library_path,
    load_library,
    make_coreness_result,
    should_notify,
    switch_condition,
    trim_memory,
)
