"""The on-device layout (kc_prep.cu): relabel by descending degree with every
row sorted on chip while it is rewritten (8-lane bitonic tiles for rows <=
64, block radix sorts in seven capacities up to 8,192, a segmented radix sort
for the hubs).  Checked directly on the laid-out CSR (kc_debug_layout): ids
in non-increasing degree order, every row ascending, and every row equal — as
a multiset, mapped back through perm — to the caller's row.  Graphs with rows
in every tier, from host memory (chunked, pipelined upload) and from device
memory (one part)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check_layout(gpu, G, flags=0, expect_sorted=True):
    H = gpu.GpuGraph(G, flags=flags)
    off, adj, perm, srt = H.layout()
    assert srt == expect_sorted
    o_off = np.asarray(G.offsets(), dtype=np.uint64)
    o_adj = np.asarray(G.neighbor_array(), dtype=np.uint32)
    n = len(o_off) - 1
    n_nz = len(off) - 1
    deg_old = np.diff(o_off).astype(np.int64)
    assert len(np.unique(perm)) == n and int(perm.max()) == n - 1
    # non-increasing degrees, isolated vertices last
    deg_new = np.diff(off).astype(np.int64)
    assert np.array_equal(deg_new, deg_old[perm[:n_nz]])
    assert np.all(deg_new[:-1] >= deg_new[1:]) and (n_nz == 0 or deg_new[-1] > 0)
    assert np.all(deg_old[perm[n_nz:]] == 0)
    # rows: sorted ascending, and the caller's row under the relabelling
    inv = np.empty(n, dtype=np.uint32)
    inv[perm] = np.arange(n, dtype=np.uint32)
    row = np.repeat(np.arange(n_nz, dtype=np.int64), deg_new)
    if expect_sorted and len(adj) > 1:
        same = row[1:] == row[:-1]
        assert np.all(adj[1:][same] >= adj[:-1][same]), "a row is not ascending"
    # expected: caller rows in new-id order, mapped through inv, each sorted
    starts = o_off[perm[:n_nz]].astype(np.int64)
    idx = np.repeat(starts - np.concatenate(([0], np.cumsum(deg_new)[:-1])), deg_new) + np.arange(len(adj))
    want = inv[o_adj[idx]]
    key_w = row * n + want.astype(np.int64)
    key_g = row * n + adj.astype(np.int64)
    assert np.array_equal(np.sort(key_w), np.sort(key_g))
    if expect_sorted:
        assert np.array_equal(np.sort(key_w), key_g)
    return H


def _tier_graph(oracle, seed=7):
    """Rows in every sort tier: degrees 1 .. ~20,000 (a few hubs above 8,192),
    duplicates of tier-boundary degrees."""
    rng = np.random.default_rng(seed)
    n = 60000
    targets = [1, 2, 7, 8, 9, 16, 17, 33, 63, 64, 65, 100, 128, 129, 255, 256, 257, 511, 512, 513,
               1000, 1020, 1021, 1024, 1025, 2047, 2048, 2049, 4096, 4097, 8191, 8192, 8193, 12000,
               20000]
    e = []
    v = 0
    for d in targets:
        for _ in range(2):
            nb = rng.choice(n - 100, d, replace=False) + 100
            e.append(np.stack([np.full(d, v, dtype=np.uint32), nb.astype(np.uint32)], 1))
            v += 1
    e.append(rng.integers(100, n, (150000, 2)).astype(np.uint32))
    pairs = np.concatenate(e).reshape(-1)
    return n, pairs


def test_layout_every_tier(gpu, oracle):
    n, pairs = _tier_graph(oracle)
    g = oracle.build_csr(n, pairs)
    G = gpu.Graph(g.off, g.nbr)
    for flags in (0, gpu.api.KC_UPLOAD_FORCE_OFF64):
        H = _check_layout(gpu, G, flags)
        core, _ = H.solve(gpu.FastKOptions())
        assert np.array_equal(core, oracle.peel(g))
    _check_layout(gpu, G, gpu.api.KC_UPLOAD_UNSORTED_ROWS, expect_sorted=False)


def test_layout_small_graphs(gpu, oracle):
    for name, n, pairs in (("grid", 150 * 150, oracle.gen_grid(150, 3)),
                           ("rmat14", 1 << 14, oracle.gen_rmat(14, 16, 5)),
                           ("star", 9001, np.array([(0, i) for i in range(1, 9001)], np.uint32).reshape(-1))):
        g = oracle.build_csr(n, pairs)
        _check_layout(gpu, gpu.Graph(g.off, g.nbr))


def test_layout_chunked_upload(gpu, oracle):
    """More than 64 MB of neighbours: the host upload is cut into chunks and
    every chunk's rows are relabelled and sorted as they land."""
    K = gpu
    d = K.gen_config(3, 20, 16, 0, seed=11)          # R-MAT 20: 30 M entries, ~120 MB
    G = d.download()
    d.free()
    H = _check_layout(gpu, G)
    Hd = K.GpuGraph(K.gen_config(3, 20, 16, 0, seed=11))   # device input: one part
    a = H.layout()
    b = Hd.layout()
    assert all(np.array_equal(x, y) for x, y in zip(a[:3], b[:3])) and a[3] and b[3]


def test_one_shot_alternating_sizes(gpu, oracle):
    """kc_fastk_run recycles its large device blocks by exact size between
    calls (kc_api.cu block cache) and releases the sizes of a graph it has not
    seen for two uploads: alternate graphs of different sizes (blocks >= 1 MB)
    and repeat one of them — every result must equal the oracle's peel."""
    cases = []
    for scale, ef, seed in ((17, 16, 1), (16, 24, 2), (18, 8, 3)):
        g = oracle.build_csr(1 << scale, oracle.gen_rmat(scale, ef, seed))
        cases.append((gpu.Graph(g.off, g.nbr), oracle.peel(g)))
    order = [0, 1, 0, 2, 2, 1, 0, 0, 2, 1]
    for step, i in enumerate(order):
        G, truth = cases[i]
        core, st = gpu.fastk_run_abi(G)
        assert np.array_equal(core, truth), i
        if step == 5:
            gpu.trim_memory()  # kc_trim_memory: everything kept between calls goes back
