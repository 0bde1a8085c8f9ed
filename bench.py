#!/usr/bin/env python3
"""bench.py — FastK coreness on B200: GTEPS and ms to converged coreness.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

One step = one complete FastK solve (estimates initialised, rounds run to the
fixed point) of BASELINE.json's config on one GPU.  Default workload:
configs[2], R-MAT scale 22 / edge factor 16 (the graph the north-star target
is quoted on; DESIGN.md §Measurement explains the choice).  N > 1 runs N
independent replicas (the path does not shard in this tier: "replicas only").

value   = ref-equivalent GTEPS = E_scan of the reference rule (fastk.cpp
          notify on settled values, computed by the same solver in REFERENCE
          mode, untimed) / device time to converged coreness, inputs resident
          in HBM; summed over replicas.  It is a time ratio against the
          reference arm (which reports the same E_scan over its own time);
          the solver's own GTEPS is config.gteps_own_rule.
e2e     = the same metric through the public C-ABI one-shot call
          kc_fastk_run with HOST buffers (H2D + layout + solve + D2H every
          step): pinned buffers (e2e) and the pageable arrays a reference
          Graph holds (e2e.pageable).
roofline= algorithmic bytes (8 * E_scan + 16 * V_eval of the run)
          / solver-kernel time vs MEASURED_PEAKS.json hbm_gbs.
also    = the second north-star graph (--also, default cfg5 = R-MAT scale
          26) measured in the same run, inside the same JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # cfg: (description, generator args (p0, p1, p2), seed)
    1: ("ER G(n=100000, m=1000000)", (100000, 1000000, 0), 1),
    2: ("grid 4096x4096, p=0.7, diag p=0.05", (4096, 0, 0), 2),
    3: ("R-MAT scale 22, edge factor 16, (0.57,0.19,0.19,0.05), ids permuted", (22, 16, 0), 3),
    4: ("Chung-Lu n=2e7, gamma 2.1, mean 20, cap 5e5, 200 cliques x 300", (20000000, 200, 300), 4),
    5: ("R-MAT scale 26, edge factor 16, ids permuted, int64 offsets in", (26, 16, 0), 5),
}
METRIC = "GTEPS to converged coreness (ref-equivalent edge entries / s)"
UNIT = "GTEPS"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """SM clock + throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line) — NVML every 5 ms on a thread; falls
    back to `nvidia-smi -lms 100` when NVML is unavailable."""

    REASONS = {  # nvmlClocksEventReason* bits
        "hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
        "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        if self._nvml is None:
            return self._run_smi()
        N = self._nvml
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self._h, N.NVML_CLOCK_SM))
                bits = N.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, b in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.005)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits", "-lms", "100"],
                                 stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in p.stdout:
            f = [x.strip() for x in line.split(",")]
            try:
                self.samples.append(float(f[0]))
                self.max_mhz = float(f[1])
            except (ValueError, IndexError):
                pass
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    self.reasons.add(nm)
            if self._stop.is_set():
                break
        p.terminate()

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=5)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


def reduce_max(value: float, dist, device="cuda"):
    """Max over ranks (timings are the slowest rank's); identity without dist."""
    if dist is None or not dist.is_initialized():
        return float(value)
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def solver_kernel(rule: int) -> str:
    """The persistent kernel that runs the rounds for this rule."""
    return "rounds_kernel" if rule == 0 else "count_rounds_kernel"


def profile_traffic(cfg: int, kernel: str):
    """DRAM bytes per launch of the solver kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        v = d.get(f"cfg{cfg}", {}).get(kernel, {})
        return v.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def measure(K, torch, cfg, args, local, steps, warmup, e2e_steps, dist=None, ws=1):
    """One workload: device-resident solves (CUDA events on the library's
    stream, L2 flushed before each), then the reference-facing one-shot call
    kc_fastk_run with host buffers (pinned, then pageable)."""
    desc, (p0, p1, p2), seed = CONFIGS[cfg]
    if args.scale and cfg == args.config:
        p0 = args.scale
    dcsr = K.gen_config(cfg, p0, p1, p2, seed=seed + args.seed_offset, device=local)
    n, nnz = dcsr.n, dcsr.nnz
    gg = K.GpuGraph(dcsr, device=local)
    _, t_prep_first = gg.timings()  # first layout: device memory comes fresh from the pool
    gg.free()
    gg = K.GpuGraph(dcsr, device=local)
    t_upload, t_prep = gg.timings()
    out = torch.empty(max(n, 1), dtype=torch.int32, device=f"cuda:{local}")
    opts = K.FastKOptions(rule=K.Rule(args.rule))
    ref_opts = K.FastKOptions(rule=K.Rule.REFERENCE, hybrid_tail=False)
    # reference-rule work (E_scan_ref) — untimed
    st_ref = gg.solve_device(out.data_ptr(), ref_opts)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def step():
        flush.fill_(1)  # evict L2 between steps (outside the event-timed solve)
        torch.cuda.synchronize()
        return gg.solve_device(out.data_ptr(), opts)

    for _ in range(warmup):
        step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    stats = []
    with Clocks(local) as clk:
        t0 = time.perf_counter()
        for _ in range(steps):
            stats.append(step())
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if dist:
        dist.barrier()
    ms = [x["t_solve_ms"] for x in stats]
    ms_step = reduce_max(sum(ms) / len(ms), dist, device=f"cuda:{local}")
    st = stats[-1]
    launches = sum(int(x["kernel_launches"]) for x in stats)
    # the gather ceiling of this graph: the solver's inner operation alone
    # (id stream + one estimate gather per adjacency entry), same L2 flush
    flush.fill_(1)
    torch.cuda.synchronize()
    probe_ms = gg.gather_probe(3)
    gg.free()
    del flush
    torch.cuda.synchronize()

    # e2e through the public C-ABI one-shot call (fastk_run semantics): host
    # CSR in, coreness out, every step.  Pinned host buffers, then the
    # pageable arrays a reference Graph holds (graph.hpp:72-73).
    host = dcsr.download()
    dcsr.free()
    off_p = torch.from_numpy(host.offsets().view(np.int64)).pin_memory()
    nbr_p = torch.from_numpy(host.neighbor_array().view(np.int32)).pin_memory()
    pinned = K.Graph(off_p.numpy().view(np.uint64), nbr_p.numpy().view(np.uint32))
    core_p = torch.empty(max(n, 1), dtype=torch.int32).pin_memory()
    core_np = core_p.numpy().view(np.uint32)

    def e2e(graph, out_arr, k):
        times, parts = [], []
        for i in range(k + 1):
            t = time.perf_counter()
            _, st2 = K.fastk_run_abi(graph, opts, out=out_arr)
            if i:  # the first call warms up
                times.append((time.perf_counter() - t) * 1e3)
                parts.append({kk: st2[kk] for kk in ("t_upload_ms", "t_prep_ms", "t_solve_ms",
                                                     "t_download_ms")})
        return (reduce_max(sum(times) / len(times), dist, device=f"cuda:{local}"),
                {kk: round(statistics.mean(p[kk] for p in parts), 3) for kk in parts[0]})

    e2e_ms, e2e_parts = e2e(pinned, core_np, e2e_steps)
    pinned_ok = bool(off_p.is_pinned() and nbr_p.is_pinned())
    del pinned, off_p, nbr_p, core_p, core_np
    core_pg = np.zeros(max(n, 1), dtype=np.uint32)
    e2e_pg_ms, e2e_pg_parts = e2e(host, core_pg, max(1, min(e2e_steps, 5)))
    return dict(cfg=cfg, desc=desc, n=n, nnz=nnz, host=host, st=st, st_ref=st_ref,
                ms_step=ms_step, wall=wall, clk=clk.summary(), launches=launches,
                t_upload=t_upload, t_prep=t_prep, t_prep_first=t_prep_first, e2e_ms=e2e_ms, e2e_parts=e2e_parts,
                e2e_pg_ms=e2e_pg_ms, e2e_pg_parts=e2e_pg_parts, pinned=pinned_ok,
                e2e_steps=e2e_steps, ws=ws, probe_ms=probe_ms)


def roofline(m, rule):
    peak, peak_src = measured_peak()
    st = m["st"]
    bytes_alg = 8 * st["e_scan"] + 16 * st["v_eval"]
    achieved = bytes_alg / (m["ms_step"] * 1e-3) / 1e9
    kname = solver_kernel(rule)
    # entries the solver actually streamed with a gather each (evaluate +
    # notify phases), against the measured gather rate of the same graph
    ent = int(st.get("scan_evaluate", 0)) + int(st.get("scan_notify", 0))
    gather_rate = m["nnz"] / (m["probe_ms"] * 1e-3)
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": profile_traffic(m["cfg"], kname),
            "peak_source": peak_src,
            "kernel": (f"{kname} (persistent: round 0 + PULL, small rounds) + count_phase_kernel<0|1> "
                       "(one per phase of the large rounds), whole solve" if kname == "count_rounds_kernel"
                       and int(m["st"].get("kernel_launches", 0)) > 6 else f"{kname} (persistent)"),
            "bytes_alg_per_launch": bytes_alg,
            "gather_ceiling": {
                "what": "kc_debug_gather_probe: id stream + one estimate gather per adjacency "
                        "entry of this graph, nothing else (L2-bandwidth bound, ncu lts 80%)",
                "probe_ms_per_pass": round(m["probe_ms"], 4),
                "gathers_per_s": round(gather_rate / 1e9, 1), "unit": "G/s",
                "solver_gathered_entries": ent or None,
                "solver_time_at_ceiling_ms": round(ent / gather_rate * 1e3, 3) if ent else None,
                "frac": round(ent / gather_rate * 1e3 / m["ms_step"], 4) if ent else None}}


def e2e_obj(m):
    n, nnz, ws = m["n"], m["nnz"], m["ws"]
    e_ref = m["st_ref"]["e_scan"]
    return {"value": round(ws * e_ref / (m["e2e_ms"] * 1e-3) / 1e9, 3), "unit": UNIT,
            "ms_per_step": round(m["e2e_ms"], 3), "steps": m["e2e_steps"],
            "h2d_bytes_per_step": int((n + 1) * 8 + nnz * 4),
            "d2h_bytes_per_step": int(n * 4),
            "device_ms": m["e2e_parts"],
            "call": "kc_fastk_run (pinned host CSR in, coreness to pinned host memory)",
            "pinned": m["pinned"],
            "pageable": {"value": round(ws * e_ref / (m["e2e_pg_ms"] * 1e-3) / 1e9, 3),
                         "ms_per_step": round(m["e2e_pg_ms"], 3), "device_ms": m["e2e_pg_parts"],
                         "call": "kc_fastk_run on pageable numpy arrays (a reference Graph's "
                                 "std::vector storage, graph.hpp:72-73)"}}


def run_ours(args, ws, rank, local):
    import torch
    import paper_2512_00233_b200 as K

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    m = measure(K, torch, args.config, args, local, args.steps, args.warmup,
                max(1, args.steps), dist, ws)
    st, e_ref = m["st"], m["st_ref"]["e_scan"]
    ms_step = m["ms_step"]
    line = {
        "metric": METRIC, "value": round(ws * e_ref / (ms_step * 1e-3) / 1e9, 3), "unit": UNIT,
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u16" if st["h_graph"] < 32768 else "u32",
        "data": "synthetic (kcgen v1 seeded generator, built in HBM)",
        "config": {"workload": f"cfg{args.config}: {m['desc']}", "n": m["n"], "nnz": m["nnz"],
                   "parallelism": f"replicas{ws}" if ws > 1 else "single GPU",
                   "rule": K.Rule(args.rule).name.lower(),
                   "l2": "flushed (256 MiB write) before every step; CSR > L2",
                   "ms_to_converged": round(ms_step, 4),
                   "value_is": "ref-equivalent GTEPS = the reference rule's E_scan (same graph, "
                               "untimed REFERENCE-rule solve) / this run's time to converged "
                               "coreness, summed over replicas: a time ratio against the "
                               "reference arm, whose value is the same E_scan / its time",
                   "e_scan_ref": e_ref, "e_scan": st["e_scan"], "v_eval": st["v_eval"],
                   "iterations": st["iterations"], "k_max": st["k_max"],
                   "h_graph": st["h_graph"],
                   "gteps_own_rule": round(st["e_scan"] / ms_step / 1e6, 3),
                   "t_upload_ms": round(m["t_upload"], 3), "t_prep_ms": round(m["t_prep"], 3),
                   "t_prep_first_ms": round(m["t_prep_first"], 3),
                   "wall_s_timed_region": round(m["wall"], 4)},
        "roofline": roofline(m, args.rule),
        "e2e": e2e_obj(m),
        "gpu_launches": m["launches"],
        "clocks": m["clk"],
    }
    host = m.pop("host")
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(host, args)
    del host, m
    # the second north-star graph (R-MAT scale 26), measured in the same run
    # and reported inside the same JSON line (rank 0 prints one line)
    if ws == 1 and args.also:
        also = {}
        for c in [int(x) for x in args.also.split(",") if x]:
            if c == args.config:
                continue
            torch.cuda.empty_cache()
            try:
                a = measure(K, torch, c, args, local, 5, 3, 3)
            except Exception as e:  # reported, never fatal to the headline line
                also[f"cfg{c}"] = {"error": f"{type(e).__name__}: {e}"}
                continue
            a.pop("host")
            sta = a["st"]
            also[f"cfg{c}"] = {
                "workload": f"cfg{c}: {a['desc']}", "n": a["n"], "nnz": a["nnz"],
                "value": round(a["st_ref"]["e_scan"] / (a["ms_step"] * 1e-3) / 1e9, 3),
                "unit": UNIT, "ms_to_converged": round(a["ms_step"], 4), "steps": 5,
                "e_scan_ref": a["st_ref"]["e_scan"], "e_scan": sta["e_scan"],
                "v_eval": sta["v_eval"], "iterations": sta["iterations"], "k_max": sta["k_max"],
                "t_prep_ms": round(a["t_prep"], 3),
                "roofline": roofline(a, args.rule), "e2e": e2e_obj(a),
                "gpu_launches": a["launches"], "clocks": a["clk"]}
            line["gpu_launches"] += a["launches"]
        line["also"] = also
    if dist:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def cpu_baseline(host, args):
    """The reference's own multithreaded FastK (oracle/_ref), one full solve."""
    from oracle import pyoracle as O
    try:
        if not O.ref_available():
            O.build(ref=True)
        cores = O.physical_cores()
        g = O.CSR(host.node_count(), host.offsets(), host.neighbor_array())
        rg = O.RefGraph(g)
        j = O.jacobi(g, "ref_ext")  # E_scan_ref of the reference rule (replay)
        t = time.perf_counter()
        core, st = rg.fastk(threads=cores, batch=256, ext=True, hybrid=True)
        dt = time.perf_counter() - t
        e_ref = j["stats"]["e_scan"]
        return {"value": round(e_ref / dt / 1e9, 4), "unit": UNIT, "cores": cores,
                "kind": "reference", "seconds": round(dt, 3),
                "sample": f"one full kcore::fastk_run (threads={cores}, batch=256, ext, "
                          f"hybrid) on the whole cfg{args.config} graph"}
    except Exception as e:  # reported, never fatal
        return {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                "sample": f"failed: {e}"}


def run_reference(args, ws, rank, local):
    """--impl reference: the reference C++ FastK (oracle/_ref) on the host cores."""
    if rank != 0:
        return
    from oracle import pyoracle as O
    desc, (p0, p1, p2), seed = CONFIGS[args.config]
    if args.scale:
        p0 = args.scale
    cfg = args.config
    if cfg == 1:
        n, pairs = p0, O.gen_er(p0, p1, seed + args.seed_offset)
    elif cfg == 2:
        n, pairs = p0 * p0, O.gen_grid(p0, seed + args.seed_offset)
    elif cfg in (3, 5):
        n, pairs = 1 << p0, O.gen_rmat(p0, p1, seed + args.seed_offset)
    else:
        n, pairs = p0, O.gen_chunglu(p0, seed + args.seed_offset, cliques=p1, csize=p2)
    g = O.build_csr(n, pairs)
    del pairs
    if not O.ref_available():
        O.build(ref=True)
    rg = O.RefGraph(g)
    cores = O.physical_cores()
    e_ref = O.jacobi(g, "ref_ext")["stats"]["e_scan"]
    budget_s = float(os.environ.get("KC_REF_BUDGET_S", "150"))
    for _ in range(args.warmup):
        rg.fastk(threads=cores)
    times = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t = time.perf_counter()
        rg.fastk(threads=cores)
        times.append(time.perf_counter() - t)
        if time.perf_counter() - t_all > budget_s:
            break
    sec = sum(times) / len(times)
    v = e_ref / sec / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT,
        "n_gpus": ws, "steps": len(times), "steps_requested": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (kcgen v1, CPU generator)",
        "config": {"workload": f"cfg{cfg}: {desc}", "n": g.n, "nnz": g.nnz,
                   "parallelism": f"{cores} host threads", "e_scan_ref": e_ref},
        "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"kcore::fastk_run (threads={cores}, batch=256) on the whole "
                                   f"cfg{cfg} graph, mean of {len(times)} runs"},
        "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    ap.add_argument("--scale", type=int, default=0, help="override p0 (R-MAT scale / n / side)")
    ap.add_argument("--seed-offset", type=int, default=0)
    ap.add_argument("--rule", type=int, default=2, help="0 reference, 1 counting, 2 auto (= counting)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--also", default="5",
                    help="further configs measured in the same run (N=1), reported under "
                         "'also' in the same JSON line ('' to skip)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
