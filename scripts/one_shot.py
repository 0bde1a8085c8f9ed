"""One kc_fastk_run call (host CSR) on a config, for launch lists under ncu."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_00233_b200 as K
from bench import CONFIGS
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
desc, (p0, p1, p2), seed = CONFIGS[a.config]
host = K.gen_config(a.config, p0, p1, p2, seed=seed).download()
G = K.Graph(host.offsets(), host.neighbor_array())
import time
for _ in range(a.reps):
    t0 = time.perf_counter()
    core, st = K.fastk_run_abi(G)
    wall = (time.perf_counter() - t0) * 1e3
    print({k: round(st[k], 3) for k in ("t_upload_ms", "t_prep_ms", "t_solve_ms", "t_download_ms")},
          "wall_ms", round(wall, 3))
