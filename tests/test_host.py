"""Host-side mirror of the reference API (paper_2512_00233_b200.api) on CPU:
graph construction, result aggregates, rules — against the oracle, the
reference and the golden fixtures."""
import numpy as np

from conftest import golden


def test_graph_from_edges_matches_reference_builder(kc, ref):
    rng = np.random.default_rng(3)
    for _ in range(15):
        n = int(rng.integers(1, 200))
        pairs = rng.integers(0, n, (int(rng.integers(0, 800)), 2))
        g = kc.Graph.from_edges(n, pairs.tolist())
        r = ref.RefGraph(n=n, pairs=pairs.astype(np.uint32).reshape(-1)).csr()
        assert np.array_equal(g.offsets(), r.off)
        assert np.array_equal(g.neighbor_array(), r.nbr)
        assert g.node_count() == n
        assert g.edge_count() == r.nbr.size // 2


def test_graph_accessors():
    import paper_2512_00233_b200 as K
    g = K.Graph.from_edges(5, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (3, 4), (4, 4)])
    assert g.degree(3) == 4 and list(g.neighbors(3)) == [0, 1, 2, 4]
    assert g.edge_count() == 7
    e = K.Graph()
    assert e.node_count() == 0 and e.edge_count() == 0


def test_make_coreness_result():
    import paper_2512_00233_b200 as K
    # tests/test_oracle.cpp:79-87
    r = K.make_coreness_result([3, 1, 2])
    assert r.k_max == 3 and abs(r.k_avg - 2.0) < 1e-12
    e = K.make_coreness_result([])
    assert e.k_max == 0 and e.k_avg == 0.0


def test_rule_helpers_match_reference():
    import paper_2512_00233_b200 as K
    g = golden("rules.json")
    for c in g["should_notify"]:
        assert int(K.should_notify(*c["args"])) == c["value"]
    for c in g["switch_condition"]:
        assert int(K.switch_condition(*c["args"])) == c["value"]


def test_named_graph_fixtures_roundtrip():
    import paper_2512_00233_b200 as K
    for name, g in golden("named_graphs.json").items():
        G = K.Graph.from_edges(g["n"], g["edges"])
        assert G.offsets().tolist() == g["offsets"], name
        assert G.neighbor_array().tolist() == g["neighbors"], name


def test_graph_rejects_malformed_csr():
    """The reference's Graph cannot be built in an invalid state
    (graph.hpp:37-75): the Python mirror rejects what the device would
    otherwise index out of bounds with."""
    import pytest
    import paper_2512_00233_b200 as K
    with pytest.raises(ValueError):
        K.Graph(np.array([0, 2, 1, 3], np.uint64), np.array([1, 2, 0], np.uint32))  # decreasing
    with pytest.raises(ValueError):
        K.Graph(np.array([0, 1, 2], np.uint64), np.array([1, 5], np.uint32))  # id >= n
    with pytest.raises(ValueError):
        K.Graph(np.array([1, 2], np.uint64), np.array([0], np.uint32))  # offsets[0] != 0


def test_host_copy_every_alignment(kc):
    """kc_hostcopy.cpp (the pageable staging path's host copy: non-temporal
    stores behind a run-time AVX2 check, memcpy otherwise): byte-exact for
    every destination / source misalignment and for sizes around the 64 KB
    switch and the 128-byte inner step; bytes outside the range untouched."""
    import numpy as np
    L = kc.load_library()
    rng = np.random.default_rng(7)
    src = rng.integers(0, 256, 1 << 20, dtype=np.uint8)
    sizes = [0, 1, 31, 32, 33, 127, 128, 129, 4095, 65535, 65536, 65537, 65536 + 127, 200001, 524288 + 77]
    for n in sizes:
        for da in (0, 1, 7, 31, 33):
            for sa in (0, 3, 32, 63):
                dst = np.full(n + 256, 0xA5, dtype=np.uint8)
                L.kc_debug_host_copy(dst.ctypes.data + 64 + da, src.ctypes.data + sa, n)
                assert np.array_equal(dst[64 + da: 64 + da + n], src[sa: sa + n]), (n, da, sa)
                assert np.all(dst[: 64 + da] == 0xA5) and np.all(dst[64 + da + n:] == 0xA5), (n, da, sa)
