"""Per-round phase imbalance: for each phase, the max and the mean over CTAs of
the time a CTA spent in it (debug phase timestamps).  The gap between them is
time CTAs wait at the next grid barrier."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_00233_b200 as K
from paper_2512_00233_b200.api import KC_DEBUG_PHASE_TIMES
from bench import CONFIGS
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
a = ap.parse_args()
desc, (p0, p1, p2), seed = CONFIGS[a.config]
g = K.GpuGraph(K.gen_config(a.config, p0, p1, p2, seed=seed))
o = K.FastKOptions()
g.solve(o)
o.debug_flags = KC_DEBUG_PHASE_TIMES
core, st = g.solve(o)
pt = g.phase_times().astype(np.int64)
R = min(st["iterations"], 256)
# phases: [1]-[0] round start+cache, [4]-[1] evaluate, [5]-[4] sync1, [7]-[6] notify+sync2
ev = (pt[:R, :, 4] - pt[:R, :, 1]) / 1e3
no = (pt[:R, :, 7] - pt[:R, :, 6]) / 1e3
print("round  eval_max eval_mean   notify_max notify_mean   (us; notify includes the closing barrier)")
for r in range(R):
    print(f"{r:5d} {ev[r].max():9.1f} {ev[r].mean():9.1f}   {no[r].max():10.1f} {no[r].mean():10.1f}")
print("sum: eval max %.0f mean %.0f | notify max %.0f mean %.0f | solve %.0f us" % (
    ev.max(1).sum(), ev.mean(1).sum(), no.max(1).sum(), no.mean(1).sum(), st["t_solve_ms"] * 1e3))
