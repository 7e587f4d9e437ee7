"""Print the key metrics of every kernel in an `ncu --page raw --csv` export."""
import csv
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "launch__grid_size", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__bytes.sum.per_second", "smsp__inst_executed.sum", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__maximum_warps_per_active_cycle_pct", "lts__t_bytes.sum",
        "l1tex__t_bytes.sum", "sass__inst_executed_register_spilling"]
rows = list(csv.reader(open(sys.argv[1])))
h, u = rows[0], rows[1]
for v in rows[2:]:
    print("=====", v[h.index("Kernel Name")][:100] if "Kernel Name" in h else "")
    for i, n in enumerate(h):
        if n in WANT or ("stalled" in n and n.endswith("per_issue_active.ratio") and float(v[i] or 0) > 0.3):
            print(f"  {n} {u[i]} {v[i]}")
