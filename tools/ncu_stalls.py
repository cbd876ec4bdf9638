"""Key metrics + stall breakdown of an ncu --set full report (raw page CSV on stdin or path)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    print("==", d.get("Kernel Name", "")[:60], d.get("gpu__time_duration.sum"))
    st = []
    for k in h:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("stalls/issue:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:10]))
    for k in ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_local_ld.sum",
              "smsp__sass_inst_executed_op_local_st.sum", "dram__bytes_read.sum",
              "dram__bytes_write.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
              "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
              "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
              "sm__sass_thread_inst_executed_op_dmul_pred_on.sum"]:
        if k in d:
            print(f"  {k} = {d[k]}")
