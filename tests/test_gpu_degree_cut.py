"""Degree cut table (kc_count.cu DegCut, sorted layouts only): round 0
evaluated from row ids and the cut table without gathers, windowed
evaluations that skip and stop at ids below their floor.  Graphs chosen for
the cases the cut logic has to get right: a hub above the warp scan limit
(8,192) evaluated by one warp in round 0, degrees above H (clamped start),
long runs of equal degrees (ties), rows whose prefix is the whole row.  The
coreness must equal the oracle's peel and every RunReport counter must equal
the unsorted layout's (same Jacobi trajectory, same notifications)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KEYS = ("iterations", "messages_sent", "messages_drained", "e_scan")


def _graphs(oracle):
    rng = np.random.default_rng(2024)
    # star with 20,000 leaves, a 60-clique on some leaves, random chords
    n = 20001
    e = [(0, i) for i in range(1, n)]
    cl = rng.choice(np.arange(1, n), 60, replace=False)
    e += [(int(a), int(b)) for i, a in enumerate(cl) for b in cl[i + 1:]]
    e += [(int(a), int(b)) for a, b in rng.integers(1, n, (30000, 2)) if a != b]
    yield "star_clique", n, np.array(e, np.uint32).reshape(-1)
    yield "grid_ties", 200 * 200, oracle.gen_grid(200, 5)
    yield "chunglu_hubs", 60000, oracle.gen_chunglu(60000, 6, cliques=20, csize=80, wmax=3e4)
    yield "rmat15", 1 << 15, oracle.gen_rmat(15, 24, 8)
    # two hubs sharing all leaves: every leaf's row is all-hub (prefix = row)
    m = 12000
    e = [(0, i) for i in range(2, m)] + [(1, i) for i in range(2, m)] + [(0, 1)]
    yield "twin_hubs", m, np.array(e, np.uint32).reshape(-1)


@pytest.mark.parametrize("rule", ["COUNTING", "REFERENCE"])
def test_sorted_equals_unsorted_and_peel(gpu, oracle, rule):
    for name, n, pairs in _graphs(oracle):
        g = oracle.build_csr(n, pairs)
        truth = oracle.peel(g)
        G = gpu.Graph(g.off, g.nbr)
        o = gpu.FastKOptions(rule=gpu.Rule[rule], hybrid_tail=False)
        reports = []
        for flags in (0, gpu.api.KC_UPLOAD_UNSORTED_ROWS, gpu.api.KC_UPLOAD_FORCE_EST32):
            core, st = gpu.GpuGraph(G, flags=flags).solve(o)
            assert np.array_equal(core, truth), (name, flags)
            reports.append({k: st[k] for k in KEYS})
        assert reports[0] == reports[1] == reports[2], name


def test_clamped_start_hub_round_zero(gpu, oracle):
    """Max degree far above H: the round-0 prefix rule must treat positions
    beyond cap = min(deg, H) as failing; iterations equal the reference
    rule's (round 0 counts as changed)."""
    n = 30001
    e = [(0, i) for i in range(1, n)] + [(i, i + 1) for i in range(1, n - 1)]
    g = oracle.build_csr(n, np.array(e, np.uint32).reshape(-1))
    G = gpu.Graph(g.off, g.nbr)
    core_c, st_c = gpu.GpuGraph(G).solve(gpu.FastKOptions(rule=gpu.Rule.COUNTING))
    core_r, st_r = gpu.GpuGraph(G).solve(gpu.FastKOptions(rule=gpu.Rule.REFERENCE,
                                                          hybrid_tail=False))
    assert np.array_equal(core_c, oracle.peel(g)) and np.array_equal(core_r, core_c)
    assert st_c["iterations"] == st_r["iterations"]
    assert st_c["h_graph"] < 30000


def test_reference_rule_counters_exact_and_repeatable(gpu, oracle):
    """Hub notify (kc_solve.cu notify_huge) applies E[u] = t only after a CTA
    barrier: with the degree cut a warp can finish its share of a hub row early,
    and before the barrier its store could reach a lagging warp's cap = E[u]
    load, which then skipped its notifications (a rare, timing-dependent
    messages_sent deficit).  Every solve's RunReport must equal the CPU
    Jacobi replay of the reference rule exactly (not just repeat itself): on
    hub-heavy graphs whose hubs (degree > 8,192) take the CTA-wide notify
    path with the degree cut active (sorted rows)."""
    graphs = [(name, n, pairs) for name, n, pairs in _graphs(oracle)
              if name in ("star_clique", "chunglu_hubs", "rmat15")]
    graphs.append(("rmat18_hubs", 1 << 18, oracle.gen_rmat(18, 16, 21)))
    for name, n, pairs in graphs:
        g = oracle.build_csr(n, pairs)
        if name == "rmat18_hubs":
            assert int(np.diff(g.off).max()) > 8192  # the CTA-wide hub path
        want = oracle.jacobi(g, "ref_ext")["stats"]
        gg = gpu.GpuGraph(gpu.Graph(g.off, g.nbr))
        o = gpu.FastKOptions(rule=gpu.Rule.REFERENCE, hybrid_tail=False)
        for _ in range(25):
            _, st = gg.solve(o)
            assert {k: st[k] for k in KEYS} == {k: want[k] for k in KEYS}, name
