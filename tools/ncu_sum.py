"""Print the headline metrics of every kernel in an .ncu-rep (ncu -i ... --csv)."""
import csv
import subprocess
import sys

KEYS = ("Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Executed Ipc Active", "Issue Slots Busy")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio")
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
for r in csv.reader(out.splitlines()):
    if len(r) > 14 and r[12] in KEYS:
        print(f"{r[4][:50]:50s} {r[12]:28s} {r[14]} {r[13]}")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
for v in rows[2:]:
    for k, u, x in zip(h, units, v):
        if k in RAW:
            print(f"  {k:80s} {x} {u}")
