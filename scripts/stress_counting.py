"""Counting-rule stress on the big configs: many back-to-back solves of the
same device-resident graph, each coreness compared on the device against the
first one (whose sha256 must equal the committed golden digest, i.e. the
reference's kcore::peel_coreness result), and the counters (iterations,
e_scan, v_eval, messages_sent) compared too.  Races show up as deviations
(DESIGN.md §5).  Usage: python scripts/stress_counting.py --config 5 --solves 200
"""
import argparse, hashlib, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2512_00233_b200 as K
from bench import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--solves", type=int, default=200)
ap.add_argument("--rule", type=int, default=2)
a = ap.parse_args()
gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "configs.json")))[str(a.config)]
desc, (p0, p1, p2), seed = CONFIGS[a.config]
d = K.gen_config(a.config, p0, p1, p2, seed=seed)
keys = ("iterations", "e_scan", "v_eval", "messages_sent", "messages_drained")
total_dev = 0
for flags, name in ((0, "sorted rows"), (K.api.KC_UPLOAD_UNSORTED_ROWS, "unsorted rows")):
    g = K.GpuGraph(d, flags=flags)
    n = g.n
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    first = torch.empty_like(out)
    o = K.FastKOptions(rule=K.Rule(a.rule))
    st0 = g.solve_device(first.data_ptr(), o)
    torch.cuda.synchronize()
    sha = hashlib.sha256(first.cpu().numpy().view(np.uint32).tobytes()).hexdigest()
    ok_gold = sha == gold["coreness_sha256"]
    dev = 0
    t0 = time.time()
    ms = []
    for i in range(a.solves):
        st = g.solve_device(out.data_ptr(), o)
        ms.append(st["t_solve_ms"])
        same = bool(torch.equal(out, first))
        cnt_same = all(st[k] == st0[k] for k in keys)
        if not (same and cnt_same):
            dev += 1
            print(f"  deviation at solve {i}: coreness_equal={same} "
                  f"counters={ {k: (st[k], st0[k]) for k in keys if st[k] != st0[k]} }", flush=True)
    total_dev += dev + (0 if ok_gold else 1)
    print(f"cfg{a.config} {name} rule={K.Rule(a.rule).name}: first solve sha256 == golden: {ok_gold}; "
          f"{a.solves} solves, {dev} deviations (coreness or counters); "
          f"t_solve median {np.median(ms):.3f} ms; wall {time.time() - t0:.1f} s; "
          f"counters {({k: st0[k] for k in keys})}", flush=True)
    g.free()
print("TOTAL deviations:", total_dev)
sys.exit(1 if total_dev else 0)
