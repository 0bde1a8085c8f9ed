"""Hunt the rare reference-rule counter deviation (DESIGN.md §3.2 open item):
many solves of one config alternating hybrid_tail off / on; on a deviation,
print the first round whose per-round counters differ from the majority run.
Development aid."""
import argparse, sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_00233_b200 as K
from bench import CONFIGS
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=100)
a = ap.parse_args()
desc, (p0, p1, p2), seed = CONFIGS[a.config]
g = K.GpuGraph(K.gen_config(a.config, p0, p1, p2, seed=seed))
ref = {}
dev = 0
for i in range(a.reps):
    hyb = bool(i & 1)
    core, st = g.solve(K.FastKOptions(rule=K.Rule.REFERENCE, hybrid_tail=hyb))
    rs = g.round_stats(st["iterations"]).astype(np.int64)
    key = (st["messages_sent"], st["messages_drained"])
    if hyb not in ref:
        ref[hyb] = (key, rs)
        continue
    if key != ref[hyb][0]:
        dev += 1
        r0 = ref[hyb][1]
        n = min(len(r0), len(rs))
        diff = np.nonzero((r0[:n] != rs[:n]).any(axis=1))[0]
        first = int(diff[0]) if diff.size else -1
        print("DEVIATION solve", i, "hybrid", hyb, key, "vs", ref[hyb][0], "first round", first, flush=True)
        if first >= 0:
            print("  ref ", r0[first].tolist(), "\n  this", rs[first].tolist(), flush=True)
print("solves", a.reps, "deviations", dev)
