"""Key metrics of every kernel in an ncu report (raw page)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units, data = rows[0], rows[1], rows[2:]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]
stall = [x for x in h if x.startswith("smsp__average_warp_latency_issue_stalled") or
         (x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("_not_issued"))]
for r in data:
    print("====", r[h.index("Kernel Name")][:100])
    for k in keys:
        if k in h:
            print(f"   {k}: {r[h.index(k)]} {units[h.index(k)]}")
    st = []
    for k in stall:
        try:
            v = float(r[h.index(k)].replace(",", ""))
        except ValueError:
            continue
        st.append((v, k))
    st.sort(reverse=True)
    print("   top stalls:", [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), v) for v, k in st[:8]])
