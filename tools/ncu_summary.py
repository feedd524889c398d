"""Key numbers of one .ncu-rep (first kernel): python tools/ncu_summary.py file.ncu-rep"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_fp64", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct", "sm__cycles_active.avg"]
d = dict(zip(h, v))
u = dict(zip(h, rows[1])) if len(rows) > 2 else {}
for k in h:
    if any(k == w or k.startswith(w) for w in keys):
        print(f"{k:90s} {d[k]:>16s} {u.get(k, '')}")
st = [(float(d[k]), k) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued") and d[k] not in ("", "n/a")]
tot = sum(x for x, _ in st) or 1
print("stall samples:", ", ".join(f"{k.split('stalled_')[1]} {100 * x / tot:.0f}%" for x, k in sorted(st, reverse=True)[:7]))
