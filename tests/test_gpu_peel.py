"""Independent device checker (kc_peel.cu): kcore::peel_coreness
(src/oracle.cpp:21-66) as a level-synchronous parallel peel, and
kcore::verify (oracle.cpp:68-75) on the device."""
import hashlib

import numpy as np
import pytest

from conftest import golden
from test_gpu_parity import CFG, _digests, labeled_union, union_csr

pytestmark = pytest.mark.gpu


def test_named_and_random_graphs(gpu):
    for name, g in golden("named_graphs.json").items():
        G = gpu.Graph(np.array(g["offsets"], np.uint64), np.array(g["neighbors"], np.uint32))
        core, st = gpu.GpuGraph(G).peel()
        assert core.tolist() == g["coreness"], name
        assert st["k_max"] == g["k_max"] and abs(st["k_avg"] - g["k_avg"]) < 1e-9
    for g in golden("random_graphs.json"):
        G = gpu.Graph.from_edges(g["n"], g["edges"])
        core, _ = gpu.GpuGraph(G).peel()
        assert core.tolist() == g["coreness"]


def test_every_labeled_graph_on_6_nodes(gpu, oracle):
    g = union_csr(oracle, labeled_union(6))
    core, _ = gpu.GpuGraph(gpu.Graph(g.off, g.nbr)).peel()
    assert np.array_equal(core, oracle.peel(g))


@pytest.mark.parametrize("flags", [0, 1, 4])
def test_skewed_and_long_graphs(gpu, oracle, flags):
    """Hubs (grid-wide frontier rows), long chains (many frontier passes)."""
    graphs = [(1 << 16, oracle.gen_rmat(16, 16, 3)), (300 * 300, oracle.gen_grid(300, 2)),
              (200000, oracle.gen_chunglu(200000, 4, cliques=10, csize=100)),
              (5001, np.array([[i, i + 1] for i in range(5000)], np.uint32).reshape(-1))]
    for n, pairs in graphs:
        g = oracle.build_csr(n, pairs)
        core, st = gpu.GpuGraph(gpu.Graph(g.off, g.nbr), flags=flags).peel()
        truth = oracle.peel(g)
        assert np.array_equal(core, truth)
        assert st["iterations"] == int(truth.max()) + 1  # one level per k


def test_verify_clean_and_perturbed(gpu, oracle):
    g = oracle.build_csr(1 << 15, oracle.gen_rmat(15, 16, 8))
    gg = gpu.GpuGraph(gpu.Graph(g.off, g.nbr))
    for rule in ("COUNTING", "REFERENCE"):
        count, bad = gg.verify(gpu.FastKOptions(rule=gpu.Rule[rule]))
        assert count == 0 and bad == []
    # self-test of the mismatch path: candidate[u] += 1 for u % 997 == 0
    count, bad = gg.verify(gpu.FastKOptions(debug_flags=gpu.api.KC_DEBUG_VERIFY_PERTURB), cap=5)
    want = [u for u in range(g.n) if u % 997 == 0]
    truth = oracle.peel(g)
    assert count == len(want)
    assert bad == [(u, int(truth[u]) + 1, int(truth[u])) for u in want[:5]]


def test_empty_and_edgeless(gpu):
    core, st = gpu.GpuGraph(gpu.Graph()).peel()
    assert core.size == 0
    core, _ = gpu.GpuGraph(gpu.Graph.from_edges(5, [])).peel()
    assert core.tolist() == [0] * 5
    assert gpu.GpuGraph(gpu.Graph.from_edges(5, [])).verify() == (0, [])


@pytest.mark.parametrize("cfg", [1, 2, 3, pytest.param(4, marks=pytest.mark.slow),
                                 pytest.param(5, marks=pytest.mark.slow)])
def test_full_size_configs(gpu, cfg):
    """The device peel reproduces the reference peel's coreness digest on the
    full BASELINE.json configs, and FastK verifies clean against it."""
    d = _digests().get(str(cfg))
    if d is None:
        pytest.skip(f"golden digest for config {cfg} not generated")
    p0, p1, p2, seed = CFG[cfg]
    gg = gpu.GpuGraph(gpu.gen_config(cfg, p0, p1, p2, seed=seed))
    core, st = gg.peel()
    assert hashlib.sha256(core.astype(np.uint32).tobytes()).hexdigest() == d["coreness_sha256"]
    assert st["k_max"] == d["k_max"]
    assert gg.verify() == (0, [])
