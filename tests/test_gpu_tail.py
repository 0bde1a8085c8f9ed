"""FastK's hybrid sequential tail on the device (kc_tail.cu) vs the reference.

The reference (src/fastk.cpp:28-55, 102-118) stops its rounds once a round
changed something but fewer than `batch` vertices are active and finishes on
one thread with a min-priority queue.  With rule REFERENCE and hybrid_tail on
(the reference's default), the GPU must report the same RunReport —
iterations, messages_sent, messages_drained and tail_pops — as the reference
compiled from /root/reference (golden fixtures) and as the oracle's
restatement (larger graphs).
"""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

KEYS = ("iterations", "messages_sent", "messages_drained", "tail_pops")


def report(r):
    return {k: getattr(r.report, k) for k in KEYS}


def run(gpu, G, ext, batch, hybrid=True):
    return gpu.fastk_run(G, gpu.FastKOptions(rule=gpu.Rule.REFERENCE, extended_notify=ext,
                                             batch=batch, hybrid_tail=hybrid))


def test_named_graphs_all_option_combinations(gpu):
    for name, g in golden("named_graphs.json").items():
        G = gpu.Graph(np.array(g["offsets"], np.uint64), np.array(g["neighbors"], np.uint32))
        for key, want in g["fastk"].items():
            ext, tail, batch = key.split("_")
            r = run(gpu, G, ext == "ext1", int(batch[1:]), tail == "tail1")
            assert r.result.coreness.tolist() == g["coreness"], (name, key)
            assert report(r) == want, (name, key)


def test_random_graphs_all_option_combinations(gpu):
    n_tail = 0
    for g in golden("random_graphs.json"):
        G = gpu.Graph.from_edges(g["n"], g["edges"])
        for key, want in g["fastk"].items():
            ext, tail, batch = key.split("_")
            r = run(gpu, G, ext == "ext1", int(batch[1:]), tail == "tail1")
            assert r.result.coreness.tolist() == g["coreness"], key
            assert report(r) == want, (g["n"], key)
            n_tail += want["tail_pops"] > 0
    assert n_tail >= 10  # the fixtures exercise the tail


@pytest.mark.parametrize("batch", [1, 16, 256, 4096])
def test_larger_graphs_vs_oracle_restatement(gpu, oracle, batch):
    """Skewed and long-diameter graphs where the tail runs hubs and long
    chains: counters equal oracle.fastk (fastk_run restated, pinned to the
    reference in test_oracle.py)."""
    graphs = [("rmat14", 1 << 14, oracle.gen_rmat(14, 16, 3)),
              ("grid96", 96 * 96, oracle.gen_grid(96, 2)),
              ("chunglu", 30000, oracle.gen_chunglu(30000, 4, cliques=3, csize=60))]
    for name, n, pairs in graphs:
        g = oracle.build_csr(n, pairs)
        G = gpu.Graph(g.off, g.nbr)
        for ext in (True, False):
            core, st = oracle.fastk(g, batch=batch, ext=ext, hybrid=True)
            r = run(gpu, G, ext, batch)
            assert np.array_equal(r.result.coreness, core), (name, ext)
            assert report(r) == {k: st[k] for k in KEYS}, (name, ext, batch)


def test_observed_mode_reports_the_tail_boundary(gpu, oracle):
    """Instrumented run (one round per launch): the switch boundary, then one
    more boundary with nothing active after the tail (fastk.cpp:180-183)."""
    g = oracle.build_csr(1 << 12, oracle.gen_rmat(12, 16, 3))
    G = gpu.Graph(g.off, g.nbr)
    core, st = oracle.fastk(g, batch=256, ext=True, hybrid=True)
    assert st["tail_pops"] > 0
    seen = []
    r = gpu.fastk_run(G, gpu.FastKOptions(rule=gpu.Rule.REFERENCE, batch=256),
                      gpu.Instrumentation(inspector=lambda it, e, a: seen.append((it, a, e.copy()))))
    assert report(r) == {k: st[k] for k in KEYS}
    its = [s[0] for s in seen]
    assert its == list(range(st["iterations"] + 2))
    assert seen[-2][1] < 256 and seen[-1][1] == 0
    assert np.array_equal(seen[-1][2], core)
    # and the same counters as the one-launch path
    assert report(run(gpu, G, True, 256)) == report(r)


def test_tail_is_invisible_to_the_counting_rule(gpu, oracle):
    g = oracle.build_csr(1 << 13, oracle.gen_rmat(13, 16, 4))
    G = gpu.Graph(g.off, g.nbr)
    a = gpu.fastk_run(G, gpu.FastKOptions(rule=gpu.Rule.COUNTING, hybrid_tail=True))
    b = gpu.fastk_run(G, gpu.FastKOptions(rule=gpu.Rule.COUNTING, hybrid_tail=False))
    assert np.array_equal(a.result.coreness, b.result.coreness)
    assert a.report.tail_pops == 0 and report(a) == report(b)


# ---------------------------------------------------- standalone sequential_tail
def test_standalone_tail_reference_cases(gpu):
    """tests/test_fastk.cpp:318-357 of the reference, through
    kc_sequential_tail (fastk.hpp:38-39)."""
    k4p = gpu.GpuGraph(gpu.Graph.from_edges(5, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3),
                                                (2, 3), (3, 4)]))
    e, a, st = k4p.sequential_tail([3, 3, 3, 3, 1], [1, 1, 1, 1, 1])
    assert e.tolist() == [3, 3, 3, 3, 1] and a.tolist() == [0] * 5
    assert (st["tail_pops"], st["messages_drained"], st["messages_sent"]) == (5, 5, 0)
    e, a, st = k4p.sequential_tail([9] * 5, [0] * 5)
    assert e.tolist() == [9] * 5 and st["tail_pops"] == 0 and st["messages_drained"] == 0
    path = gpu.GpuGraph(gpu.Graph.from_edges(3, [(0, 1), (1, 2)]))
    e, a, st = path.sequential_tail([1, 2, 2], [0, 1, 1])
    assert e.tolist() == [1, 1, 1]
    assert (st["tail_pops"], st["messages_drained"], st["messages_sent"]) == (3, 2, 1)


def test_standalone_tail_from_degrees_solves(gpu, oracle):
    # test_fastk.cpp:359-370: the tail alone reaches the coreness from degrees
    rng = np.random.default_rng(417)
    for _ in range(10):
        n = 70
        iu = np.triu_indices(n, 1)
        keep = rng.random(iu[0].size) < 0.1
        g = oracle.build_csr(n, np.stack([iu[0][keep], iu[1][keep]], 1).astype(np.uint32).reshape(-1))
        gg = gpu.GpuGraph(gpu.Graph(g.off, g.nbr))
        e, a, _ = gg.sequential_tail(np.diff(g.off).astype(np.uint32), np.ones(n, np.uint8))
        assert np.array_equal(e, oracle.peel(g)) and not a.any()


@pytest.mark.parametrize("ext", [True, False])
def test_standalone_tail_vs_oracle_and_reference(gpu, oracle, ext):
    """Arbitrary estimates (above 2^16 too, on a 16-bit handle), random active
    sets, isolated vertices: estimates and counters equal the C restatement
    and, where built, the reference's own sequential_tail."""
    rng = np.random.default_rng(9 + ext)
    for scale, pairs_fn in ((12, lambda: oracle.gen_rmat(12, 8, 5)),
                            (0, lambda: oracle.gen_er(3000, 9000, 6))):
        n = (1 << scale) if scale else 3000
        g = oracle.build_csr(n, pairs_fn())
        gg = gpu.GpuGraph(gpu.Graph(g.off, g.nbr))
        deg = np.diff(g.off).astype(np.uint32)
        for est in (deg, rng.integers(0, 200000, n).astype(np.uint32), deg // 2):
            act = (rng.random(n) < 0.6).astype(np.uint8)
            e, a, st = gg.sequential_tail(est, act, ext)
            e0, a0, st0 = oracle.sequential_tail(g, est, act, ext)
            assert np.array_equal(e, e0) and not a.any()
            for k in ("tail_pops", "messages_drained", "messages_sent"):
                assert st[k] == st0[k], k
            if oracle.ref_available():
                e1, _, st1 = oracle.RefGraph(g).sequential_tail(est, act, ext)
                assert np.array_equal(e, e1)
                assert st["tail_pops"] == st1["tail_pops"]
