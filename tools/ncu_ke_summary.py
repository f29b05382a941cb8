"""Integration-kernel ncu summary: duration, pipe utilisation, LSU wavefronts (shared / global) per
element, stall reasons.  python tools/ncu_ke_summary.py REPORT N_ELEMENTS [KERNEL_REGEX]"""
import csv
import subprocess
import sys

rep, n_el = sys.argv[1], float(sys.argv[2])
kern = sys.argv[3] if len(sys.argv) > 3 else "integrate_mesh_kernel"
raw = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, v = rows[0], rows[1], rows[2]
m = dict(zip(h, v))
u = dict(zip(h, units))


def f(name):
    try:
        return float(m[name].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")


print(f"duration {f('gpu__time_duration.sum')} {u.get('gpu__time_duration.sum', '')}")
for name in ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
             "smsp__issue_active.avg.pct_of_peak_sustained_active",
             "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
             "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
             "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
             "smsp__warps_eligible.avg.per_cycle_active"):
    print(f"{name}: {f(name):.2f}")
for name in ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
             "smsp__inst_executed.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
             "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"):
    print(f"{name} per element: {f(name) / n_el:.2f}")
