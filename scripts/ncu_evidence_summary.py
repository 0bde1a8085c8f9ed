"""Summarise an ncu_evidence.sh capture: the north-star counters of one whole
solve — the persistent kernel (round 0 + PULL, and the small rounds after the
hand-off) plus the per-phase kernels of the large rounds, aggregated — and of
the estimate-gather probe, whose L2 hit rate with the id sectors taken out
(read once: they miss) is the hit rate of the estimate gathers.
usage: python scripts/ncu_evidence_summary.py <report.ncu-rep> <nnz> [peak_gbs]"""
import csv, io, json, subprocess, sys
rep, nnz = sys.argv[1], int(sys.argv[2])
peak = float(sys.argv[3]) if len(sys.argv) > 3 else json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "s": 1e3,
         "nsecond": 1e-6, "second": 1e3}
def g(r, k):
    """value in bytes for byte metrics, ms for durations, raw otherwise"""
    if k not in h:
        return float("nan")
    v = r[h.index(k)].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return float("nan")
    return x * SCALE.get(units[h.index(k)], 1.0)
def one(r):
    t_ms = g(r, "gpu__time_duration.sum")
    gl = g(r, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
    return {
        "time_ms": t_ms,
        "dram_bytes": g(r, "dram__bytes_read.sum") + g(r, "dram__bytes_write.sum"),
        "dram_pct": g(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "l2_hit_pct": g(r, "lts__t_sector_hit_rate.pct"),
        "l2_tput_pct": g(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "gl_bytes_per_sector": g(r, "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio"),
        "gl_sectors": gl,
        "gl_requests": g(r, "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
        "l1_hit_pct": g(r, "l1tex__t_sector_hit_rate.pct"),
        "local_ld_sectors": g(r, "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum"),
        "local_st_sectors": g(r, "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum"),
        "warps_active_pct": g(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "regs": g(r, "launch__registers_per_thread"),
        "inst": g(r, "smsp__inst_executed.sum"),
        "threads": g(r, "launch__block_size"),
    }
def agg(ks):
    T = sum(k["time_ms"] for k in ks)
    tw = lambda f: sum(k[f] * k["time_ms"] for k in ks) / T
    gls = sum(k["gl_sectors"] for k in ks)
    dram = sum(k["dram_bytes"] for k in ks)
    loc = sum(k["local_ld_sectors"] + k["local_st_sectors"] for k in ks)
    return {
        "launches": len(ks), "time_ms": T, "dram_bytes": dram,
        "dram_GBps": dram / (T * 1e-3) / 1e9,
        "dram_frac_of_measured_peak": dram / (T * 1e-3) / 1e9 / peak,
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed (time-weighted)": tw("dram_pct"),
        "lts__t_sector_hit_rate.pct (time-weighted)": tw("l2_hit_pct"),
        "lts__throughput.pct (time-weighted)": tw("l2_tput_pct"),
        "global_load_bytes_per_sector (smsp__sass_average_data_bytes_per_sector_mem_global_op_ld)":
            sum(k["gl_bytes_per_sector"] * k["gl_sectors"] for k in ks) / gls,
        "global_load_sectors_per_request": gls / sum(k["gl_requests"] for k in ks),
        "l1tex__t_sector_hit_rate.pct (time-weighted)": tw("l1_hit_pct"),
        "local_ld_sectors": sum(k["local_ld_sectors"] for k in ks),
        "local_st_sectors": sum(k["local_st_sectors"] for k in ks),
        "global_ld_sectors": gls,
        "local_over_global_ld_sectors": loc / gls,
        "sm__warps_active.avg.pct_of_peak_sustained_active (time-weighted)": tw("warps_active_pct"),
        "registers_per_thread": sorted({int(k["regs"]) for k in ks}),
        "threads_per_cta": sorted({int(k["threads"]) for k in ks}),
        "smsp__inst_executed.sum": sum(k["inst"] for k in ks),
    }
groups = {}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    if "est_gather_probe" in name:
        key = "gather_probe"
    elif "count_phase_kernel<0" in name or "count_phase_kernel<(int)0" in name:
        key = "phase_evaluate"
    elif "count_phase_kernel" in name:
        key = "phase_notify"
    elif "count_rounds" in name:
        key = "persistent"
    else:
        continue
    groups.setdefault(key, []).append((r, one(r)))
res = {}
solver = [k for key in ("persistent", "phase_evaluate", "phase_notify") for _, k in groups.get(key, [])]
if solver:
    res["solver"] = agg(solver)
    res["solver"]["kernels"] = "count_rounds_kernel (round 0 + PULL, small rounds) + count_phase_kernel<0|1> (EVALUATE | NOTIFY of the large rounds)"
    for key in ("persistent", "phase_evaluate", "phase_notify"):
        if key in groups:
            res["solver_" + key] = agg([k for _, k in groups[key]])
if "gather_probe" in groups:
    r, k = groups["gather_probe"][-1]
    d = agg([k])
    ids = nnz * 4 / 32
    rd = g(r, "lts__t_sectors_srcunit_tex_op_read.sum")
    hit = g(r, "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum")
    d["est_gather_l2_sectors"] = rd - ids
    d["est_gather_l2_hit_rate_pct"] = 100.0 * hit / max(rd - ids, 1)
    d["gathers_per_s"] = nnz / (k["time_ms"] * 1e-3)
    res["gather_probe"] = d
print(json.dumps(res, indent=1))
