"""Key metrics of an ncu report (details page): duration, throughputs, occupancy, stall reasons."""
import csv
import io
import subprocess
import sys

want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L2 Cache Throughput",
        "L1/TEX Cache Throughput", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
mn, mv, mu = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
for x in r[1:]:
    if x[mn] in want:
        print(f"{x[mn]:34s} {x[mv]:>14s} {x[mu]}")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hd, vals = rr[0], rr[2] if len(rr) > 2 else rr[1]
stalls = []
for i, name in enumerate(hd):
    if name.startswith("smsp__average_warp_latency_issue_stalled_") or name.startswith("smsp__pcsamp_warps_issue_stalled_"):
        try:
            stalls.append((float(vals[i].replace(",", "")), name))
        except ValueError:
            pass
for v, n in sorted(stalls, reverse=True)[:10]:
    print(f"  {n:80s} {v}")
for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_tmem_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"):
    if key in hd:
        print(f"{key:70s} {vals[hd.index(key)]} {rr[1][hd.index(key)] if len(rr) > 2 else ''}")
