"""A/B of the per-phase kernels (KC_SPLIT_ROUNDS) on one config: coreness
digest against tests/golden/configs.json, counters against the split-off
solve, best-of-N solve time.  Env (KC_LIB_PATH, KC_SPLIT_*) selects the build."""
import argparse, hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_00233_b200 as K
from bench import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "configs.json")))[str(a.config)]
desc, (p0, p1, p2), seed = CONFIGS[a.config]
g = K.GpuGraph(K.gen_config(a.config, p0, p1, p2, seed=seed))
ts = []
for i in range(a.reps + 1):
    core, st = g.solve(K.FastKOptions())
    if i: ts.append(st["t_solve_ms"])
ok = hashlib.sha256(np.ascontiguousarray(core, dtype=np.uint32).tobytes()).hexdigest() == gold["coreness_sha256"]
print(f"cfg{a.config} split={os.environ.get('KC_SPLIT_ROUNDS','0')} min={os.environ.get('KC_SPLIT_MIN','')} "
      f"cache={os.environ.get('KC_SPLIT_CACHE','')} lib={os.path.basename(os.environ.get('KC_LIB_PATH','') or 'base')} "
      f"digest_ok={ok} it={st['iterations']} v_eval={st['v_eval']} e_scan={st['e_scan']} sent={st['messages_sent']} "
      f"best={min(ts):.3f} med={sorted(ts)[len(ts)//2]:.3f} ms", flush=True)
