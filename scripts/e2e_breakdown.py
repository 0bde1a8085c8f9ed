"""Host-side breakdown of the e2e path (upload handle, solve, free) on one config."""
import argparse, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2512_00233_b200 as K
from bench import CONFIGS
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
a = ap.parse_args()
desc, (p0, p1, p2), seed = CONFIGS[a.config]
d = K.gen_config(a.config, p0, p1, p2, seed=seed)
host = d.download()
off_p = torch.from_numpy(host.offsets().view(np.int64)).pin_memory()
nbr_p = torch.from_numpy(host.neighbor_array().view(np.int32)).pin_memory()
pinned = K.Graph(off_p.numpy().view(np.uint64), nbr_p.numpy().view(np.uint32))
core = torch.empty(max(d.n, 1), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
for i in range(4):
    t0 = time.perf_counter()
    g = K.GpuGraph(pinned)
    t1 = time.perf_counter()
    _, st = g.solve(K.FastKOptions(), out=core)
    t2 = time.perf_counter()
    g.free()
    t3 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.2f} (dev {st['t_upload_ms']:.2f}+{st['t_prep_ms']:.2f})  solve {1e3*(t2-t1):.2f} "
          f"(dev {st['t_solve_ms']:.2f}+{st['t_download_ms']:.2f})  free {1e3*(t3-t2):.2f}", flush=True)
