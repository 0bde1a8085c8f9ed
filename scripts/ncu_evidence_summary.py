"""Summarise an ncu_evidence.sh capture: the north-star counters of the
solver kernel and of the estimate-gather probe, with the gather L2 hit rate
derived from the probe (its id stream is read once: those sectors miss).
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
    v = r[h.index(k)].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return float("nan")
    return x * SCALE.get(units[h.index(k)], 1.0)
res = {}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    key = "solver" if "count_rounds" in name else "gather_probe"
    t_ms = g(r, "gpu__time_duration.sum")
    dram = g(r, "dram__bytes_read.sum") + g(r, "dram__bytes_write.sum")
    d = {
        "kernel": name.split("(")[0],
        "time_ms": t_ms,
        "dram_bytes": dram,
        "dram_GBps": dram / (t_ms * 1e-3) / 1e9,
        "dram_frac_of_measured_peak": dram / (t_ms * 1e-3) / 1e9 / peak,
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": g(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "lts__t_sector_hit_rate.pct": g(r, "lts__t_sector_hit_rate.pct"),
        "global_load_bytes_per_sector (smsp__sass_average_data_bytes_per_sector_mem_global_op_ld)":
            g(r, "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio"),
        "global_load_sectors_per_request": g(r, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum") /
            g(r, "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
        "l1tex__t_sector_hit_rate.pct": g(r, "l1tex__t_sector_hit_rate.pct"),
        "local_ld_sectors": g(r, "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum"),
        "local_st_sectors": g(r, "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum"),
        "global_ld_sectors": g(r, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
        "sm__warps_active.avg.pct_of_peak_sustained_active": g(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers_per_thread": g(r, "launch__registers_per_thread"),
        "smsp__inst_executed.sum": g(r, "smsp__inst_executed.sum"),
        "lts__throughput.pct": g(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    }
    if key == "gather_probe":
        # L2 read sectors = id sectors (streamed once, miss) + gather sectors
        ids = nnz * 4 / 32
        rd = g(r, "lts__t_sectors_srcunit_tex_op_read.sum")
        hit = g(r, "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum")
        d["est_gather_l2_sectors"] = rd - ids
        d["est_gather_l2_hit_rate_pct"] = 100.0 * hit / max(rd - ids, 1)
        d["gathers_per_s"] = nnz / (t_ms * 1e-3)
    res[key] = d
print(json.dumps(res, indent=1))
