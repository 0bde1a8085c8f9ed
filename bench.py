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
          in HBM; summed over replicas.
e2e     = the same metric through the public C-ABI call with HOST buffers:
          pinned CSR -> kc_graph_upload (H2D + layout) -> kc_solve -> coreness
          on the host, per step.
roofline= algorithmic bytes (8 * E_scan + 16 * V_eval of the run)
          / solver-kernel time vs MEASURED_PEAKS.json hbm_gbs.
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


def run_ours(args, ws, rank, local):
    import torch
    import paper_2512_00233_b200 as K

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    desc, (p0, p1, p2), seed = CONFIGS[args.config]
    if args.scale:
        p0 = args.scale
    dcsr = K.gen_config(args.config, p0, p1, p2, seed=seed + args.seed_offset, device=local)
    n, nnz = dcsr.n, dcsr.nnz
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

    for _ in range(args.warmup):
        step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    stats = []
    with Clocks(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            stats.append(step())
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if dist:
        dist.barrier()
    ms = [s["t_solve_ms"] for s in stats]
    ms_step = reduce_max(sum(ms) / len(ms), dist, device=f"cuda:{local}")
    st = stats[-1]
    e_ref, e_our, v_our = st_ref["e_scan"], st["e_scan"], st["v_eval"]
    gteps = ws * e_ref / (ms_step * 1e-3) / 1e9

    # e2e through the public C-ABI with pinned host buffers (rank-local)
    host = dcsr.download()
    off_p = torch.from_numpy(host.offsets().view(np.int64)).pin_memory()
    nbr_p = torch.from_numpy(host.neighbor_array().view(np.int32)).pin_memory()
    pinned = K.Graph(off_p.numpy().view(np.uint64), nbr_p.numpy().view(np.uint32))
    core_p = torch.empty(max(n, 1), dtype=torch.int32).pin_memory()
    core_np = core_p.numpy().view(np.uint32)
    e2e_steps = max(1, min(args.steps, 5))
    e2e_ms, parts = [], []
    for i in range(e2e_steps + 1):
        t = time.perf_counter()
        # kc_fastk_run: the reference-facing one-shot call (fastk_run semantics)
        _, st2 = K.fastk_run_abi(pinned, opts, out=core_np)
        if i:  # first call warms up
            e2e_ms.append((time.perf_counter() - t) * 1e3)
            parts.append({k: st2[k] for k in ("t_upload_ms", "t_prep_ms", "t_solve_ms",
                                              "t_download_ms")})
    e2e_ms_step = reduce_max(sum(e2e_ms) / len(e2e_ms), dist, device=f"cuda:{local}")

    peak, peak_src = measured_peak()
    bytes_alg = 8 * e_our + 16 * v_our
    achieved = bytes_alg / (ms_step * 1e-3) / 1e9
    kname = solver_kernel(args.rule)
    traffic = profile_traffic(args.config, kname)
    line = {
        "metric": METRIC, "value": round(gteps, 3), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16" if st["h_graph"] < 32768 else "u32",
        "data": "synthetic (kcgen v1 seeded generator, built in HBM)",
        "config": {"workload": f"cfg{args.config}: {desc}", "n": n, "nnz": nnz,
                   "parallelism": f"replicas{ws}" if ws > 1 else "single GPU",
                   "rule": K.Rule(args.rule).name.lower(),
                   "l2": "flushed (256 MiB write) before every step; CSR > L2",
                   "ms_to_converged": round(ms_step, 4),
                   "e_scan_ref": e_ref, "e_scan": e_our, "v_eval": v_our,
                   "iterations": st["iterations"], "k_max": st["k_max"],
                   "h_graph": st["h_graph"], "gteps_own_rule": round(e_our / ms_step / 1e6, 3),
                   "t_upload_ms": round(t_upload, 3), "t_prep_ms": round(t_prep, 3),
                   "wall_s_timed_region": round(wall, 4)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": peak_src, "kernel": f"{kname} (persistent)",
                     "bytes_alg_per_launch": bytes_alg},
        "e2e": {"value": round(ws * e_ref / (e2e_ms_step * 1e-3) / 1e9, 3), "unit": UNIT,
                "ms_per_step": round(e2e_ms_step, 3),
                "h2d_bytes_per_step": int((n + 1) * 8 + nnz * 4),
                "device_ms": {k: round(statistics.mean(p[k] for p in parts), 3) for k in parts[0]},
                "call": "kc_fastk_run (pinned host CSR in, coreness to pinned host memory)",
                "pinned": bool(off_p.is_pinned() and nbr_p.is_pinned()),
                "d2h_bytes_per_step": int(n * 4)},
        "gpu_launches": 4 * args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(host, args)
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
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
