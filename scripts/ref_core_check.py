"""Reference-rule coreness of the full-size configs 4 and 5 against the golden digests (development aid)."""
import sys, os, json, hashlib
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2512_00233_b200 as K
from bench import CONFIGS
d = json.load(open("tests/golden/configs.json"))
for cfg in (5, 4):
    want = d[str(cfg)]["coreness_sha256"] if str(cfg) in d else d[f"cfg{cfg}"]["coreness_sha256"]
    desc, (p0, p1, p2), seed = CONFIGS[cfg]
    g = K.GpuGraph(K.gen_config(cfg, p0, p1, p2, seed=seed))
    for hyb in (False, True, True, True):
        core, st = g.solve(K.FastKOptions(rule=K.Rule.REFERENCE, hybrid_tail=hyb))
        ok = hashlib.sha256(core.astype(np.uint32).tobytes()).hexdigest() == want
        print(cfg, hyb, ok, st["messages_sent"], flush=True)
