"""Key metrics of one kernel from `ncu --page raw --csv` (development aid)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_active.avg",
        "gpc__cycles_elapsed.max"]
idx = {n: i for i, n in enumerate(h)}
for n in want:
    if n in idx:
        print(n, v[idx[n]], u[idx[n]])
st = [(float(v[i]), n) for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled_")
      and n.endswith("_per_issue_active.ratio") and v[i] not in ("", "n/a")]
for val, n in sorted(st, reverse=True)[:8]:
    print(n, f"{val:.6f}", "inst")
