"""Summarise an ncu report: key metrics + warp stall reasons + top source lines.
    python profiles/ncu_summary.py gpurun_out/prof.ncu-rep [--source]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Issue Slots Busy", "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Grid Size", "Block Size", "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction",
        "Issued Instructions", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for r in rows[1:]:
    if r[-4] in KEYS:
        print(f"{r[-4]:40s} {r[-2]:>16s} {r[-3]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
names, units, vals = rr[0], rr[1], rr[2]
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__average_warp_latency_issue_stalled",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64",
        "lts__t_bytes.sum"]
for n, u, v in zip(names, units, vals):
    if any(n.startswith(w) for w in want) or ("warp_issue_stalled" in n and n.endswith("_per_warp_active.pct")):
        print(f"{n:80s} {v:>16s} {u}")
