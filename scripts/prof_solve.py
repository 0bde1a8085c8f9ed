"""Profiling driver: build a config on the GPU, lay it out, solve it `--reps`
times (the first is warm-up).  Used under ncu with -k regex:rounds_kernel."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_00233_b200 as K
from bench import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--scale", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--rule", type=int, default=2)
ap.add_argument("--cache", type=int, default=0)
ap.add_argument("--legacy", action="store_true", help="counting rule on the flag-frontier solver")
ap.add_argument("--probe", type=int, default=0, help="then N passes of kc_debug_gather_probe")
a = ap.parse_args()
desc, (p0, p1, p2), seed = CONFIGS[a.config]
if a.scale: p0 = a.scale
d = K.gen_config(a.config, p0, p1, p2, seed=seed)
g = K.GpuGraph(d)
print("upload/prep ms", g.timings(), flush=True)
for i in range(a.reps):
    o = K.FastKOptions(rule=K.Rule(a.rule), smem_cache=a.cache)
    if a.legacy:
        o.debug_flags = K.api.KC_DEBUG_LEGACY_COUNT
    core, st = g.solve(o)
    print(i, {k: st[k] for k in ("iterations", "e_scan", "v_eval", "t_solve_ms", "k_max")}, flush=True)
if a.probe:
    ms = g.gather_probe(a.probe)
    print(f"gather probe: {ms:.3f} ms per pass over {g.nnz} entries = "
          f"{g.nnz / ms / 1e6:.1f} G gathers/s", flush=True)
