"""Repeat solves (both rules) on full-size configs and compare coreness
digests — catches nondeterministic races that a single run would miss."""
import argparse, hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_00233_b200 as K
from bench import CONFIGS
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
want = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "tests", "golden", "configs.json")))[str(a.config)]["coreness_sha256"]
desc, (p0, p1, p2), seed = CONFIGS[a.config]
d = K.gen_config(a.config, p0, p1, p2, seed=seed)
bad = 0
for flags in (0, K.api.KC_UPLOAD_UNSORTED_ROWS):
    g = K.GpuGraph(d, flags=flags)
    for r in range(a.reps):
        rule = K.Rule.COUNTING if r % 4 else K.Rule.REFERENCE
        core, st = g.solve(K.FastKOptions(rule=rule))
        h = hashlib.sha256(core.astype(np.uint32).tobytes()).hexdigest()
        bad += h != want
    g.free()
print(f"config {a.config}: {2 * a.reps} solves, {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
