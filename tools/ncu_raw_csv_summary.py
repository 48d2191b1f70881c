"""Summarise an exported ncu raw page (ncu -i rep --page raw --csv) into the
metric list kept under profiles/.  usage: python tools/ncu_raw_csv_summary.py raw.csv 'header line' [launch index]"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2 + (int(sys.argv[3]) if len(sys.argv) > 3 else 0)]
print("#", sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
print("# (cold, serialised replay under ncu: use ratios and shares, not absolute times, as bench values)")
print("Kernel Name =", v[h.index("Kernel Name")])
for i, k in enumerate(h):
    if k in KEYS or ("issue_stalled" in k and k.endswith("per_issue_active.ratio") and k.startswith("smsp__average")):
        try:
            if k in KEYS or float(v[i]) > 0.05:
                print(f"{k} = {v[i]} {u[i]}".rstrip())
        except ValueError:
            pass
