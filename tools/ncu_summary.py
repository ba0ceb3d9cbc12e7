"""Summarise an ncu --set full report (raw page CSV) for the pass kernels.

    ncu -i rep.ncu-rep --page raw --csv > raw.csv; python tools/ncu_summary.py raw.csv
"""
import csv
import sys

WANT = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.sum",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.sum",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__grid_size", "launch__block_size",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
]


def main(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    units = rows[1]
    ki = h.index("Kernel Name")
    for r in rows[2:]:
        print(f"== {r[ki][:90]}")
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"   {w:70s} {r[i]:>18s} {units[i]}")
        print()


if __name__ == "__main__":
    main(sys.argv[1])
