"""Print the key metrics of an ncu raw CSV (developer tool): python tools/ncu_keys.py raw.csv"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "memory_l1_wavefronts_shared_ideal", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sass__inst_executed_register_spilling", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]
STALLS = "smsp__average_warps_issue_stalled_"
rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, zip(v, u)))
for k in KEYS:
    if k in d:
        print(f"{k:70s} {d[k][0]:>16s} {d[k][1]}")
st = sorted(((float(d[k][0]), k[len(STALLS):]) for k in d if k.startswith(STALLS) and k.endswith("_per_issue_active.ratio")), reverse=True)
print("stalls per issue:", ", ".join(f"{n.replace('_per_issue_active.ratio','')}={x:.2f}" for x, n in st[:8]))
