"""Per-round phase timing of the persistent solver (debug instrumentation)."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_00233_b200 as K
from paper_2512_00233_b200.api import KC_DEBUG_PHASE_TIMES
from bench import CONFIGS
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--scale", type=int, default=0)
ap.add_argument("--rule", type=int, default=2)
ap.add_argument("--cache", type=int, default=0)
ap.add_argument("--debug-flags", type=int, default=0, help="extra KC_DEBUG_* bits (e.g. 8: no pull)")
a = ap.parse_args()
desc, (p0, p1, p2), seed = CONFIGS[a.config]
if a.scale: p0 = a.scale
d = K.gen_config(a.config, p0, p1, p2, seed=seed)
g = K.GpuGraph(d)
o = K.FastKOptions(rule=K.Rule(a.rule), smem_cache=a.cache)
o.debug_flags = a.debug_flags
g.solve(o)
core, st = g.solve(o)
print("plain solve ms", st["t_solve_ms"], "iters", st["iterations"])
o.debug_flags = KC_DEBUG_PHASE_TIMES | a.debug_flags
core, st = g.solve(o)
print("instrumented solve ms", st["t_solve_ms"])
pt = g.phase_times().astype(np.int64)
R = min(st["iterations"], 256)
names = ["compact", "ev_huge", "ev_bigwarp", "ev_small", "sync1", "fillN", "notify+s2"]
rs = g.round_stats(R).astype(np.int64)
t0 = pt[0, :, 0].min()
print("round  start_us  " + " ".join(f"{n:>10s}" for n in names) +
      "   |  evals   escan(M) ascan(M) nscan(M) fires(M)  q:huge big warp sub thread  (max over CTAs, us)")
tot = np.zeros(7)
for r in range(R):
    d = np.diff(pt[r], axis=1) / 1e3  # per CTA per phase
    mx = d.max(axis=0); tot += mx
    q = rs[r]
    qs = [q[6] & 0xffffffff, q[6] >> 32, q[7] & 0xffffffff, q[7] >> 32, q[8]]
    print(f"{r:5d} {(pt[r,:,0].min()-t0)/1e3:9.1f}  " + " ".join(f"{x:10.1f}" for x in mx) +
          f"   | {q[0]:8d} {q[1]/1e6:8.2f} {q[5]/1e6:8.2f} {q[4]/1e6:8.2f} {q[3]/1e6:8.2f}  " + " ".join(str(int(v)) for v in qs))
pr = pt[255]
if pr[:, 1].max() > 0:  # PULL's phases (kc_count.cu pull_phase)
    d = np.diff(pr[:, 1:5], axis=1) / 1e3
    mx = d.max(axis=0)
    print("PULL phases (max over CTAs, us): huge %.1f  big+warp %.1f  sub+thread+long %.1f" % tuple(mx))
print("totals: escan %.1fM ascan %.1fM nscan %.1fM" % (rs[:,1].sum()/1e6, rs[:,5].sum()/1e6, rs[:,4].sum()/1e6))
print("sum of max:", " ".join(f"{n}={x:.0f}" for n, x in zip(names, tot)))
