"""Summarise an .ncu-rep: duration, DRAM bytes, throughput, occupancy, top stall reasons."""
import csv, io, subprocess, sys, re
def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "idc__request_hit_rate.pct", "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
for path in sys.argv[1:]:
    rows, units = raw(path)
    for r in rows:
        print(f"== {path}  {r.get('Kernel Name','')[:60]}")
        for k in KEYS:
            if k in r:
                print(f"  {k:70s} {r[k]:>14s} {units.get(k,'')}")
        st = {k: float(v) for k, v in r.items() if re.fullmatch(r"smsp__pcsamp_warps_issue_stalled_\w+", k) and not k.endswith("not_issued") and v.replace('.','',1).isdigit()}
        tot = sum(st.values()) or 1
        top = sorted(st.items(), key=lambda kv: -kv[1])[:6]
        print("  stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')} {100*v/tot:.0f}%" for k, v in top))
