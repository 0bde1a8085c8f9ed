"""Fixed cost of a round: graphs whose rounds hold a handful of vertices.
A path of n vertices converges in ~n/2 Jacobi rounds with 2 droppers each."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_00233_b200 as K
from oracle import pyoracle as O

for n in (1001, 3001):
    e = np.array([(i, i + 1) for i in range(n - 1)], np.uint32).reshape(-1)
    g = O.build_csr(n, e)
    gg = K.GpuGraph(K.Graph(g.off, g.nbr))
    for rule in (K.Rule.COUNTING, K.Rule.REFERENCE):
        o = K.FastKOptions(rule=rule, hybrid_tail=False)
        gg.solve(o)
        _, st = gg.solve(o)
        print(f"path n={n} rule={rule.name}: {st['iterations']} rounds, {st['t_solve_ms']:.3f} ms, "
              f"{st['t_solve_ms'] * 1e3 / st['iterations']:.2f} us/round", flush=True)

# per-phase breakdown (max over CTAs) of the counting solver's rounds on the path
from paper_2512_00233_b200.api import KC_DEBUG_PHASE_TIMES
n = 1001
e = np.array([(i, i + 1) for i in range(n - 1)], np.uint32).reshape(-1)
g = O.build_csr(n, e)
gg = K.GpuGraph(K.Graph(g.off, g.nbr))
o = K.FastKOptions(rule=K.Rule.COUNTING)
o.debug_flags = KC_DEBUG_PHASE_TIMES
gg.solve(o)
_, st = gg.solve(o)
pt = gg.phase_times().astype(np.int64)
names = ["start", "ev_huge", "ev_bigwarp", "ev_small", "sync1", "fillN", "notify+s2"]
acc = np.zeros(7)
rows = range(10, 200)
for r in rows:
    d = np.diff(pt[r], axis=1) / 1e3
    acc += d.max(axis=0)
print("path n=1001 counting, rounds 10-199, mean per round (max over CTAs, us):",
      " ".join(f"{nm}={x / len(rows):.2f}" for nm, x in zip(names, acc)))
# the CTA that did the work vs the others in one round
r = 50
d = np.diff(pt[r], axis=1) / 1e3
busy = np.argmax(d[:, 2] + d[:, 3])
print("round 50, busiest CTA", busy, " ".join(f"{nm}={x:.2f}" for nm, x in zip(names, d[busy])))
print("round 50, CTA 0      ", " ".join(f"{nm}={x:.2f}" for nm, x in zip(names, d[0])))
print("round-start spread (us):", (pt[r, :, 0].max() - pt[r, :, 0].min()) / 1e3)
