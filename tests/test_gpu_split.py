"""The per-phase kernels of the counting solver (kc_count_split.cu): rounds
1 .. KC_SPLIT_ROUNDS run one kernel per phase, then the persistent kernel
resumes.  The switches are read once per process, so each case runs in a
subprocess: coreness (sha256) and every counter must equal the in-process
solve (persistent kernel only: the graphs are below the size that turns the
per-phase kernels on).  Cases: hand-off on a small round, the round limit
reached while rounds are still large, convergence inside the per-phase
kernels, with and without the shared-memory estimate cache."""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("iterations", "e_scan", "v_eval", "messages_sent", "messages_drained")

CHILD = r"""
import sys, json, hashlib
sys.path.insert(0, %r)
import numpy as np
import paper_2512_00233_b200 as K
from oracle import pyoracle as O
out = {}
for name, n, pairs in (("rmat16", 1 << 16, O.gen_rmat(16, 24, 3)),
                       ("chunglu", 80000, O.gen_chunglu(80000, 9, cliques=30, csize=60, wmax=2e4))):
    g = O.build_csr(n, pairs)
    for flags in (0, K.api.KC_UPLOAD_UNSORTED_ROWS):
        core, st = K.GpuGraph(K.Graph(g.off, g.nbr), flags=flags).solve(K.FastKOptions())
        out[f"{name}/{flags}"] = {"sha": hashlib.sha256(np.ascontiguousarray(core, dtype=np.uint32).tobytes()).hexdigest(),
                                  **{k: int(st[k]) for k in %r}}
print("RESULT " + json.dumps(out))
"""


def _run(env_extra):
    env = dict(os.environ)
    env.pop("KC_SPLIT_ROUNDS", None)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, KEYS)], capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")][-1]
    return json.loads(line[len("RESULT "):])


def test_split_kernels_equal_persistent(gpu, oracle):
    base = _run({})  # below the size criterion: the persistent kernel alone
    for name, n, pairs in (("rmat16", 1 << 16, oracle.gen_rmat(16, 24, 3)),):
        g = oracle.build_csr(n, pairs)
        truth = hashlib.sha256(np.ascontiguousarray(oracle.peel(g), dtype=np.uint32).tobytes()).hexdigest()
        assert base[f"{name}/0"]["sha"] == truth
    cases = [
        {"KC_SPLIT_ROUNDS": "16"},                                    # hand-off on a small round
        {"KC_SPLIT_ROUNDS": "3", "KC_SPLIT_MIN": "0"},                # round limit reached
        {"KC_SPLIT_ROUNDS": "4000", "KC_SPLIT_MIN": "0"},             # converges inside
        {"KC_SPLIT_ROUNDS": "1", "KC_SPLIT_MIN": "0"},
        {"KC_SPLIT_ROUNDS": "16", "KC_SPLIT_CACHE": "0"},
    ]
    for env in cases:
        got = _run(env)
        assert got == base, env
