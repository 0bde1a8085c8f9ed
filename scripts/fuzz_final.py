"""Randomised end-to-end check of the round's new code paths on the GPU: random
graphs from several families and sizes (rows in every sort tier, odd array
sizes for the block cache), uploaded with every layout flag, solved through the
resident handle (both rules) and through the one-shot kc_fastk_run, each result
compared with the oracle's peel; the laid-out CSR checked for sortedness.
KC_SPLIT_ROUNDS in the environment forces the per-phase kernels on.
usage: python scripts/fuzz_final.py --seconds 240"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_00233_b200 as K
from oracle import pyoracle as O

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=240)
ap.add_argument("--seed", type=int, default=12345)
a = ap.parse_args()
rng = np.random.default_rng(a.seed)
t_end = time.time() + a.seconds
n_graphs = n_checks = 0
FLAGS = (0, K.api.KC_UPLOAD_UNSORTED_ROWS, K.api.KC_UPLOAD_FORCE_OFF64, K.api.KC_UPLOAD_FORCE_EST32,
         K.api.KC_UPLOAD_FORCE_OFF64 | K.api.KC_UPLOAD_FORCE_EST32)


def make(rng):
    kind = rng.integers(0, 6)
    if kind == 0:
        n = int(rng.integers(50, 200000)); m = int(rng.integers(n, 12 * n))
        return "er", n, O.gen_er(n, m, int(rng.integers(1, 1 << 30)))
    if kind == 1:
        sc = int(rng.integers(8, 18)); ef = int(rng.integers(2, 40))
        return f"rmat{sc}x{ef}", 1 << sc, O.gen_rmat(sc, ef, int(rng.integers(1, 1 << 30)))
    if kind == 2:
        n = int(rng.integers(2000, 150000))
        return "chunglu", n, O.gen_chunglu(n, int(rng.integers(1, 1 << 30)), cliques=int(rng.integers(0, 30)),
                                           csize=int(rng.integers(5, 120)), wmax=float(rng.integers(50, 40000)))
    if kind == 3:
        side = int(rng.integers(10, 400))
        return "grid", side * side, O.gen_grid(side, int(rng.integers(1, 1 << 30)))
    if kind == 4:  # hubs of chosen degrees (tier boundaries) over a random background
        n = int(rng.integers(20000, 120000))
        e = [rng.integers(0, n, (int(rng.integers(n, 4 * n)), 2)).astype(np.uint32)]
        for v, d in enumerate(rng.choice([63, 64, 65, 127, 128, 129, 255, 257, 511, 513, 1019, 1020, 1021, 1024, 1025,
                                          2047, 2049, 4095, 4097, 8191, 8192, 8193, 9000, 15000], 12)):
            nb = rng.choice(n - 20, int(min(d, n - 21)), replace=False) + 20
            e.append(np.stack([np.full(len(nb), v, np.uint32), nb.astype(np.uint32)], 1))
        return "tiers", n, np.concatenate(e).reshape(-1)
    n = int(rng.integers(2, 3000))  # tiny / degenerate
    m = int(rng.integers(0, 3 * n))
    return "tiny", n, rng.integers(0, n, (m, 2)).astype(np.uint32).reshape(-1)


while time.time() < t_end:
    name, n, pairs = make(rng)
    g = O.build_csr(n, pairs)
    truth = O.peel(g)
    G = K.Graph(g.off, g.nbr)
    n_graphs += 1
    for flags in FLAGS:
        H = K.GpuGraph(G, flags=flags)
        off, adj, perm, srt = H.layout()
        if srt and len(adj) > 1:
            row = np.repeat(np.arange(len(off) - 1), np.diff(off).astype(np.int64))
            same = row[1:] == row[:-1]
            assert np.all(adj[1:][same] >= adj[:-1][same]), (name, n, flags, "row not ascending")
        for rule, hyb in ((K.Rule.COUNTING, False), (K.Rule.REFERENCE, False), (K.Rule.REFERENCE, True)):
            core, st = H.solve(K.FastKOptions(rule=rule, hybrid_tail=hyb))
            assert np.array_equal(core, truth), (name, n, g.nnz, flags, rule, hyb)
            n_checks += 1
        H.free()
    core, st = K.fastk_run_abi(G)
    assert np.array_equal(core, truth), (name, n, "one-shot")
    n_checks += 1
    if n_graphs % 7 == 0:
        K.trim_memory()
print(f"fuzz: {n_graphs} graphs, {n_checks} solves, all equal to the oracle's peel "
      f"(KC_SPLIT_ROUNDS={os.environ.get('KC_SPLIT_ROUNDS', 'default')})")
