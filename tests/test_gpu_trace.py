"""Convergence traces reduced on the device (kc_solve_traced) vs the
reference's record_iteration (src/report.cpp:7-18) over its own snapshots."""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def rows_from_snapshots(snaps, acts, truth):
    """record_iteration restated over the reference's per-boundary estimates."""
    n = len(truth)
    t = np.asarray(truth, dtype=np.float64)
    out = []
    for s, a in zip(snaps, acts):
        gap = float((np.asarray(s, dtype=np.float64) - t).sum()) if n else 0.0
        out.append((gap / n if n else 0.0, a / n if n else 0.0))
    return out


def test_device_trace_equals_reference_trajectory(gpu):
    checked = 0
    for g in golden("random_graphs.json"):
        if "observed" not in g:
            continue
        G = gpu.Graph.from_edges(g["n"], g["edges"])
        truth = gpu.make_coreness_result(g["coreness"])
        for ext in (1, 0):
            want = g["observed"][f"ext{ext}"]
            r = gpu.fastk_run(G, gpu.FastKOptions(rule=gpu.Rule.REFERENCE, extended_notify=bool(ext),
                                                  hybrid_tail=False),
                              gpu.Instrumentation(truth=truth, trace_convergence=True))
            got = [(t.mean_error, t.active_fraction) for t in r.report.trace]
            assert got == rows_from_snapshots(want["snapshots"], want["active"], g["coreness"])
            checked += 1
    assert checked >= 8


@pytest.mark.parametrize("rule", ["REFERENCE", "COUNTING"])
@pytest.mark.parametrize("hybrid", [False, True])
def test_device_trace_equals_host_hook_trace(gpu, oracle, rule, hybrid):
    """Same rows whether the boundary estimates cross PCIe (inspector) or only
    their sum does (device trace)."""
    g = oracle.build_csr(1 << 14, oracle.gen_rmat(14, 16, 5))
    G = gpu.Graph(g.off, g.nbr)
    truth = gpu.make_coreness_result(oracle.peel(g))
    opts = gpu.FastKOptions(rule=gpu.Rule[rule], hybrid_tail=hybrid)
    dev = gpu.fastk_run(G, opts, gpu.Instrumentation(truth=truth, trace_convergence=True))
    seen = []
    host = gpu.fastk_run(G, opts, gpu.Instrumentation(truth=truth, trace_convergence=True,
                                                      inspector=lambda it, e, a: seen.append(it)))
    assert [(t.mean_error, t.active_fraction) for t in dev.report.trace] == \
        [(t.mean_error, t.active_fraction) for t in host.report.trace]
    assert len(dev.report.trace) == len(seen)
    assert dev.report.trace[-1].mean_error == 0.0 and dev.report.trace[-1].active_fraction == 0.0
    assert np.array_equal(dev.result.coreness, truth.coreness)
    assert dev.report.iterations == host.report.iterations
    assert dev.report.tail_pops == host.report.tail_pops
