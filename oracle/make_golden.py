#!/usr/bin/env python3
"""Generate tests/golden/* from the UNMODIFIED reference (oracle/_ref).

TEST INFRASTRUCTURE.  Run in the build container (needs /root/reference for
oracle/_ref/libkcore_ref.so):

    python oracle/make_golden.py            # small fixtures (seconds)
    python oracle/make_golden.py --configs  # + full-size config digests (slow)

Every fixture records what the reference computes on inputs defined here
(seeded numpy / kcgen v1), so the GPU tests can pin results without the
reference at run time.  The reference tests' own known-answer cases are
reproduced verbatim where they are literal (tests/test_kernel.cpp:30-44,
tests/test_fastk.cpp:118-179, tests/test_oracle.cpp:43-67,
tests/test_bench.cpp:166-176); their random suites (std::mt19937_64 +
libstdc++ distributions) are replaced by numpy-seeded inputs of the same
shapes, run through the same reference functions.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from oracle import pyoracle as O  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
UNKNOWN = 0xFFFFFFFF  # kUnknownEstimate, include/kcore/kernel.hpp:13-15


def named_graphs():
    """tests/test_support.hpp:31-67 named fixtures (+ families of test_oracle.cpp)."""
    g = {}
    g["triangle"] = (3, [(0, 1), (1, 2), (0, 2)])
    g["star4"] = (5, [(0, i) for i in range(1, 5)])
    g["star9"] = (10, [(0, i) for i in range(1, 10)])
    g["path5"] = (5, [(i, i + 1) for i in range(4)])
    g["path6"] = (6, [(i, i + 1) for i in range(5)])
    g["cycle7"] = (7, [(i, (i + 1) % 7) for i in range(7)])
    g["complete6"] = (6, [(i, j) for i in range(6) for j in range(i + 1, 6)])
    g["k4_pendant"] = (5, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (3, 4)])
    g["k4_pendant0"] = (5, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (0, 4)])
    g["barbell"] = (6, [(0, 1), (1, 2), (0, 2), (2, 3), (3, 4), (4, 5), (3, 5)])
    g["edgeless4"] = (4, [])
    g["single"] = (1, [])
    g["empty"] = (0, [])
    g["self_loops_dups"] = (4, [(0, 0), (0, 1), (1, 0), (0, 1), (2, 3), (3, 3)])
    return g


def gnp_edges(rng, n, p):
    iu = np.triu_indices(n, 1)
    keep = rng.random(iu[0].size) < p
    return np.stack([iu[0][keep], iu[1][keep]], 1).astype(np.uint32)


def fastk_matrix(rg):
    """Reference counters under the option matrix the tests use."""
    out = {}
    for ext in (True, False):
        for hybrid in (True, False):
            for batch in (1, 3, 256):
                core, st = rg.fastk(threads=4, batch=batch, ext=ext, hybrid=hybrid)
                out[f"ext{int(ext)}_tail{int(hybrid)}_b{batch}"] = st
    return out, core


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_small():
    os.makedirs(GOLDEN, exist_ok=True)
    # --- compute_index: literal KATs + numpy-seeded randoms through the reference
    kats = [([1, 2, 3], 3), ([5, 5, 5, 5], 4), ([2, 1, 1], 3), ([], 5), ([9, 9, 9], 0),
            ([0, 0, 0], 3), ([1], 1), ([UNKNOWN, UNKNOWN], 2), ([UNKNOWN, 1], 2)]
    rng = np.random.default_rng(201)
    for _ in range(400):
        ln = int(rng.integers(0, 51))
        vals = rng.integers(0, 60, ln).astype(np.int64)
        vals[rng.integers(0, 60, ln) == 59] = UNKNOWN
        kats.append((vals.tolist(), int(rng.integers(0, 51))))
    ci = [{"est": v, "cap": c, "index": O.ref_compute_index(np.array(v, np.uint32), c)}
          for v, c in kats]
    with open(os.path.join(GOLDEN, "compute_index.json"), "w") as f:
        json.dump(ci, f)

    # --- should_notify / switch_condition (fastk.hpp:25-31; test_fastk.cpp:118-140)
    R = O.ref()
    sn = [{"args": [a, b, c], "value": int(R.ref_should_notify(a, b, c))}
          for a in range(0, 7) for b in range(0, 7) for c in range(0, 7)]
    sw = [{"args": [a, b], "value": int(R.ref_switch_condition(a, b))}
          for a, b in [(255, 256), (256, 256), (0, 1), (0, 4096), (5, 3)]]
    with open(os.path.join(GOLDEN, "rules.json"), "w") as f:
        json.dump({"should_notify": sn, "switch_condition": sw}, f)

    # --- named graphs: reference CSR (from_edges), peel, fastk counters
    named = {}
    for name, (n, edges) in named_graphs().items():
        pairs = np.array(edges, np.uint32).reshape(-1)
        rg = O.RefGraph(n=n, pairs=pairs)
        csr = rg.csr()
        core, kmax, kavg = rg.peel()
        counters, fcore = fastk_matrix(rg)
        assert np.array_equal(core, fcore)
        named[name] = {"n": n, "edges": [list(map(int, e)) for e in edges],
                       "offsets": csr.off.tolist(), "neighbors": csr.nbr.tolist(),
                       "coreness": core.tolist(), "k_max": kmax, "k_avg": kavg,
                       "fastk": counters}
    with open(os.path.join(GOLDEN, "named_graphs.json"), "w") as f:
        json.dump(named, f)

    # --- random G(n, p) graphs: coreness + counters + observed trajectories
    rng = np.random.default_rng(909)
    rand = []
    for i in range(24):
        n = int(rng.integers(2, 65)) if i < 16 else int(rng.integers(100, 400))
        p = float(rng.uniform(0.01, 0.5)) if i < 16 else float(rng.uniform(0.005, 0.05))
        e = gnp_edges(rng, n, p)
        rg = O.RefGraph(n=n, pairs=e.reshape(-1))
        core, kmax, kavg = rg.peel()
        counters, _ = fastk_matrix(rg)
        entry = {"n": n, "edges": e.tolist(), "coreness": core.tolist(), "k_max": kmax,
                 "fastk": counters}
        if i % 3 == 0:
            obs = {}
            for ext in (True, False):
                oc, st, snaps, acts = rg.fastk_observed(threads=3, batch=8, ext=ext, hybrid=False)
                obs[f"ext{int(ext)}"] = {"snapshots": snaps.tolist(), "active": acts.tolist(),
                                         "report": st}
            entry["observed"] = obs
        rand.append(entry)
    with open(os.path.join(GOLDEN, "random_graphs.json"), "w") as f:
        json.dump(rand, f)

    # --- star-4 convergence trace (test_bench.cpp:166-176 expects
    #     0,0.6,1.0 / 1,0,0 / 2,0,0 for FastK with the queue tail)
    rg = O.RefGraph(n=5, pairs=np.array([0, 1, 0, 2, 0, 3, 0, 4], np.uint32))
    me, af = rg.fastk_trace(threads=4, batch=256, ext=True, hybrid=True)
    with open(os.path.join(GOLDEN, "trace_star4.json"), "w") as f:
        json.dump({"mean_error": me.tolist(), "active_fraction": af.tolist()}, f)
    print("small fixtures written to", GOLDEN)


CONFIGS = {  # must match bench.py CONFIGS (kcgen v1)
    1: ("er", (100000, 1000000), 1),
    2: ("grid", (4096,), 2),
    3: ("rmat", (22, 16), 3),
    4: ("chunglu", (20000000, 200, 300), 4),
    5: ("rmat", (26, 16), 5),
}


def gen(cfg, scale=None):
    kind, args, seed = CONFIGS[cfg]
    if kind == "er":
        n = args[0]
        return n, O.gen_er(n, args[1], seed)
    if kind == "grid":
        side = args[0] if scale is None else scale
        return side * side, O.gen_grid(side, seed)
    if kind == "rmat":
        sc = args[0] if scale is None else scale
        return 1 << sc, O.gen_rmat(sc, args[1], seed)
    n = args[0] if scale is None else scale
    return n, O.gen_chunglu(n, seed, cliques=args[1], csize=args[2])


def make_configs(which):
    path = os.path.join(GOLDEN, "configs.json")
    have = json.load(open(path)) if os.path.exists(path) else {}
    for cfg in which:
        n, pairs = gen(cfg)
        g = O.build_csr(n, pairs)
        del pairs
        core = O.peel(g)
        rec = {"n": g.n, "nnz": g.nnz, "offsets_sha256": sha(g.off), "neighbors_sha256": sha(g.nbr),
               "coreness_sha256": sha(core.astype(np.uint32)), "k_max": int(core.max()),
               "k_sum": int(core.astype(np.uint64).sum()), "h_graph": O.degree_hindex(g),
               "max_degree": int(np.diff(g.off).max()),
               "coreness_histogram": np.bincount(core).tolist()}
        # the reference rule's work for the ref-equivalent GTEPS (every config;
        # cfg 4 / 5 take minutes of single-threaded replay)
        j = O.jacobi(g, "ref_ext", clamp=True)
        rec["jacobi_ref_ext"] = j["stats"]
        have[str(cfg)] = rec
        print(cfg, {k: v for k, v in rec.items() if k != "coreness_histogram"}, flush=True)
        with open(path, "w") as f:
            json.dump(have, f, indent=1)


def edge_list_cases():
    """Texts exercising kcore::load_edge_list (graph.cpp:22-80, 141-199)."""
    rng = np.random.default_rng(2024)
    cases = {
        "basic": "# comment\n10 20\n20 30\n 30\t10 \r\n\n5 5\n",
        "crlf_no_final_newline": "1 2\r\n2 3\r\n3 1",
        "dups_loops_reversed": "4 4\n1 2\n2 1\n1 2\n2 3\n3 3\n",
        "sparse_large_ids": "18446744073709551615 0\n1099511627776 7\n7 18446744073709551615\n",
        "leading_zeros_tabs": "\t0001\t\t002\n002 \t 3\r\n",
        "empty": "",
        "only_comments": "# a\n   # b\n\n\t\r\n",
        "err_token": "1 2\n3 x4\n5 6\n",
        "err_negative": "-1 2\n",
        "err_plus": "1 2\n+3 4\n",
        "err_overflow": "18446744073709551616 1\n",
        "err_one_id": "1 2\n\n7\n",
        "err_three_ids": "1 2\n2 3 4\n",
        "err_trailing_comment": "1 2 # c\n",
        "err_last_line_no_newline": "1 2\n3",
        "err_first_of_two": "a b\n1\n",
        "err_vertical_tab": "1\v2\n",
    }
    lines = []
    for _ in range(3000):  # random spacing, comments, large and small ids
        r = rng.random()
        if r < 0.05:
            lines.append("# " + "x" * int(rng.integers(0, 10)))
        elif r < 0.08:
            lines.append(" \t" * int(rng.integers(0, 3)))
        else:
            a = int(rng.integers(0, 500)) if rng.random() < 0.7 else int(rng.integers(0, 2**63))
            b = int(rng.integers(0, 500)) if rng.random() < 0.7 else int(rng.integers(0, 2**63))
            sep = [" ", "\t", "  ", " \t "][int(rng.integers(0, 4))]
            lines.append(f"{a}{sep}{b}" + ("\r" if rng.random() < 0.1 else ""))
    cases["random_3000"] = "\n".join(lines) + "\n"
    return cases


def make_edge_lists():
    out = {}
    for name, text in edge_list_cases().items():
        try:
            g, ids = O.ref_load_edge_list(text.encode())
            out[name] = {"text": text, "n": g.n, "offsets": g.off.tolist(),
                         "neighbors": g.nbr.tolist(), "original_ids": [str(int(x)) for x in ids]}
        except ValueError as e:
            out[name] = {"text": text, "error_line": e.line, "error": str(e)}
        print(name, {k: v for k, v in out[name].items() if k in ("n", "error")}, flush=True)
    with open(os.path.join(GOLDEN, "edge_lists.json"), "w") as f:
        json.dump(out, f, indent=0)


def add_full_counters(which):
    """Both counter sets of a full-size config from ONE generation: the
    Jacobi replay's reference-rule RunReport without the tail (what the GPU's
    REFERENCE rule with hybrid_tail=false must reproduce) and the unmodified
    reference kcore::fastk_run with its defaults.  The coreness of both is
    checked against the committed peel digest."""
    path = os.path.join(GOLDEN, "configs.json")
    have = json.load(open(path))
    for cfg in which:
        n, pairs = gen(cfg)
        g = O.build_csr(n, pairs)
        del pairs
        rec = have[str(cfg)]
        assert sha(g.off) == rec["offsets_sha256"] and sha(g.nbr) == rec["neighbors_sha256"]
        j = O.jacobi(g, "ref_ext", clamp=True)
        assert sha(j["est"].astype(np.uint32)) == rec["coreness_sha256"]
        rec["jacobi_ref_ext"] = j["stats"]
        del j
        print(cfg, "jacobi", rec["jacobi_ref_ext"], flush=True)
        core, st = O.RefGraph(g).fastk(threads=O.physical_cores(), batch=256, ext=True, hybrid=True)
        assert sha(core.astype(np.uint32)) == rec["coreness_sha256"]
        rec["reference_fastk_default"] = {k: int(st[k]) for k in (
            "iterations", "messages_sent", "messages_drained", "tail_pops")}
        print(cfg, "reference", rec["reference_fastk_default"], flush=True)
        have = json.load(open(path))
        have[str(cfg)] = rec
        with open(path, "w") as f:
            json.dump(have, f, indent=1)


def add_ref_counters(which):
    """RunReport of the unmodified reference kcore::fastk_run with its
    defaults (batch 256, extended notify, hybrid tail) on the full-size
    configs: the GPU's REFERENCE rule + hybrid tail must reproduce it."""
    path = os.path.join(GOLDEN, "configs.json")
    have = json.load(open(path))
    for cfg in which:
        n, pairs = gen(cfg)
        g = O.build_csr(n, pairs)
        del pairs
        core, st = O.RefGraph(g).fastk(threads=8, batch=256, ext=True, hybrid=True)
        assert sha(core.astype(np.uint32)) == have[str(cfg)]["coreness_sha256"]
        have[str(cfg)]["reference_fastk_default"] = {k: int(st[k]) for k in (
            "iterations", "messages_sent", "messages_drained", "tail_pops")}
        print(cfg, have[str(cfg)]["reference_fastk_default"], flush=True)
        with open(path, "w") as f:
            json.dump(have, f, indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="", help="comma list of config ids to digest")
    ap.add_argument("--no-small", action="store_true")
    ap.add_argument("--ref-counters", default="", help="comma list: add the reference's RunReport")
    ap.add_argument("--full-counters", default="",
                    help="comma list: Jacobi replay + reference RunReport (one generation)")
    ap.add_argument("--edge-lists", action="store_true", help="edge-list loader fixtures")
    a = ap.parse_args()
    O.build(ref=True)
    if not a.no_small:
        make_small()
    if a.configs:
        make_configs([int(x) for x in a.configs.split(",")])
    if a.ref_counters:
        add_ref_counters([int(x) for x in a.ref_counters.split(",")])
    if a.full_counters:
        add_full_counters([int(x) for x in a.full_counters.split(",")])
    if a.edge_lists:
        make_edge_lists()
