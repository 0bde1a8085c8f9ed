"""Repeat the reference-rule solve on one config and print the distinct
RunReport counters seen (determinism check; development aid)."""
import argparse, sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_00233_b200 as K
from bench import CONFIGS
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--hybrid", type=int, default=1)
ap.add_argument("--alternate", action="store_true", help="alternate hybrid_tail off / on")
a = ap.parse_args()
desc, (p0, p1, p2), seed = CONFIGS[a.config]
g = K.GpuGraph(K.gen_config(a.config, p0, p1, p2, seed=seed))
seen = collections.Counter()
for i in range(a.reps):
    hyb = bool(i & 1) if a.alternate else bool(a.hybrid)
    core, st = g.solve(K.FastKOptions(rule=K.Rule.REFERENCE, hybrid_tail=hyb))
    seen[(hyb, st["iterations"], st["messages_sent"], st["messages_drained"], st["tail_pops"])] += 1
for k, v in seen.items():
    print("cfg", a.config, "counters", k, "x", v)
