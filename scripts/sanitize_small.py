"""Small end-to-end exercise of every device path, for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_00233_b200 as K
from oracle import pyoracle as O
g = O.build_csr(1 << 11, O.gen_rmat(11, 8, 3))
truth = O.peel(g)
G = K.Graph(g.off, g.nbr)
for flags in (0, K.api.KC_UPLOAD_UNSORTED_ROWS, 3):
    gg = K.GpuGraph(G, flags=flags)
    for rule in (K.Rule.COUNTING, K.Rule.REFERENCE):
        for hyb in (True, False):
            core, st = gg.solve(K.FastKOptions(rule=rule, hybrid_tail=hyb, batch=64))
            assert np.array_equal(core, truth), (flags, rule, hyb)
    core, _ = gg.peel()
    assert np.array_equal(core, truth)
    assert gg.verify() == (0, [])
    e, a, _ = gg.sequential_tail(np.diff(g.off).astype(np.uint32), np.ones(g.n, np.uint8))
    assert np.array_equal(e, truth)
    gg.free()
r = K.fastk_run(G, K.FastKOptions(), K.Instrumentation(truth=K.make_coreness_result(truth),
                                                       trace_convergence=True))
assert np.array_equal(r.result.coreness, truth)
d = K.load_edge_list("# x\n1 2\n2 3\n3 1\n3 4\n")
assert d.n == 4
print("sanitize_small ok")
