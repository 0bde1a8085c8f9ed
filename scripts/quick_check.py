"""Quick GPU-vs-oracle parity sweep (development aid; tests/ hold the gate)."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
from oracle import pyoracle as O
import paper_2512_00233_b200 as K

def check(name, n, pairs, rules=(K.Rule.COUNTING, K.Rule.REFERENCE)):
    g = O.build_csr(n, pairs)
    truth = O.peel(g)
    G = K.Graph(g.off, g.nbr)
    gg = K.GpuGraph(G)
    for rule in rules:
        for ext in (True, False):
            t = time.time()
            core, st = gg.solve(K.FastKOptions(rule=rule, extended_notify=ext, hybrid_tail=False))
            ok = np.array_equal(core, truth)
            j = O.jacobi(g, "ref_ext" if ext else "ref_plain")
            extra = ""
            if rule == K.Rule.REFERENCE:
                extra = " ref-counters %s" % (
                    (st["iterations"], st["messages_sent"], st["messages_drained"]) ==
                    (j["stats"]["iterations"], j["stats"]["messages_sent"], j["stats"]["messages_drained"]))
            print(f"{name:10s} rule={int(rule)} ext={int(ext)} ok={ok} it={st['iterations']} "
                  f"solve={st['t_solve_ms']:.3f}ms escan={st['e_scan']} kmax={st['k_max']}{extra}",
                  flush=True)
            if not ok:
                bad = np.nonzero(core != truth)[0]
                print("   mismatches", bad.size, bad[:10], core[bad[:10]], truth[bad[:10]])
    gg.free()

check("tri", 3, np.array([0,1,1,2,0,2], np.uint32))
check("er10k", 10000, O.gen_er(10000, 100000, 1))
check("grid64", 64*64, O.gen_grid(64, 2))
check("rmat12", 1<<12, O.gen_rmat(12, 16, 3))
check("rmat16", 1<<16, O.gen_rmat(16, 16, 3))
check("cl1e5", 100000, O.gen_chunglu(100000, 4, cliques=5, csize=100))
check("er100k", 100000, O.gen_er(100000, 1000000, 1))
check("rmat20", 1<<20, O.gen_rmat(20, 16, 3), rules=(K.Rule.COUNTING,))
