"""Reference rule with and without the hybrid tail on one config (timing + counters)."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_00233_b200 as K
from bench import CONFIGS
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--scale", type=int, default=0)
a = ap.parse_args()
desc, (p0, p1, p2), seed = CONFIGS[a.config]
if a.scale: p0 = a.scale
g = K.GpuGraph(K.gen_config(a.config, p0, p1, p2, seed=seed))
for hyb in (False, True, True):
    core, st = g.solve(K.FastKOptions(rule=K.Rule.REFERENCE, hybrid_tail=hyb))
    print("hybrid", hyb, {k: st[k] for k in ("iterations", "messages_sent", "messages_drained",
                                               "tail_pops", "t_solve_ms")}, flush=True)
