"""Randomised parity sweep (development aid): sorted / unsorted / 32-bit
layouts, both rules, against the oracle's peel on many small graphs of mixed
shapes (hubs above H, cliques, stars, paths, power laws, grids)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import pyoracle as O
import paper_2512_00233_b200 as K

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
FLAGS = (0, K.api.KC_UPLOAD_UNSORTED_ROWS, K.api.KC_UPLOAD_FORCE_EST32,
         K.api.KC_UPLOAD_FORCE_OFF64 | K.api.KC_UPLOAD_UNSORTED_ROWS)


def graph(kind):
    if kind == 0:
        n = int(rng.integers(2, 3000)); m = int(rng.integers(1, 20 * n))
        return n, O.gen_er(n, m, int(rng.integers(1 << 30)))
    if kind == 1:
        s = int(rng.integers(6, 14)); return 1 << s, O.gen_rmat(s, int(rng.integers(2, 40)), int(rng.integers(1 << 30)))
    if kind == 2:
        side = int(rng.integers(2, 120)); return side * side, O.gen_grid(side, int(rng.integers(1 << 30)))
    if kind == 3:
        n = int(rng.integers(100, 20000))
        return n, O.gen_chunglu(n, int(rng.integers(1 << 30)), cliques=int(rng.integers(0, 6)),
                                csize=int(rng.integers(3, 90)), wmax=float(rng.integers(10, 20000)))
    # stars, cliques, paths glued together
    n = int(rng.integers(10, 15000)); e = []
    for _ in range(int(rng.integers(1, 6))):
        c = int(rng.integers(0, n)); k = int(rng.integers(1, n))
        e += [(c, int(x)) for x in rng.integers(0, n, k) if x != c]
    cl = rng.choice(n, int(rng.integers(2, min(n, 80))), replace=False)
    e += [(int(a), int(b)) for i, a in enumerate(cl) for b in cl[i + 1:]]
    e += [(i, i + 1) for i in range(0, n - 1, 3)]
    return n, np.array(e, np.uint32).reshape(-1)


bad = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 120):
    kind = it % 5
    n, pairs = graph(kind)
    g = O.build_csr(n, pairs)
    truth = O.peel(g)
    G = K.Graph(g.off, g.nbr)
    reps = {}
    for flags in FLAGS:
        gg = K.GpuGraph(G, flags=flags)
        for rule in (K.Rule.COUNTING, K.Rule.REFERENCE):
            core, st = gg.solve(K.FastKOptions(rule=rule, hybrid_tail=False))
            if not np.array_equal(core, truth):
                bad += 1
                print("MISMATCH", it, kind, n, flags, int(rule), flush=True)
            key = (int(rule),)
            r = (st["iterations"], st["messages_sent"], st["e_scan"])
            if key in reps and reps[key] != r:
                bad += 1
                print("COUNTERS", it, kind, n, flags, int(rule), reps[key], r, flush=True)
            reps.setdefault(key, r)
        gg.free()
print("graphs", it + 1, "failures", bad)
