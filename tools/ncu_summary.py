"""Summarise an ncu report (details page) into the key roofline/occupancy lines."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
si, mi, ui, vi, ki = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Unit", "Metric Value", "Kernel Name"))
keep = {"Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Achieved Active Warps Per SM", "Block Size", "Grid Size",
        "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Executed Instructions", "Eligible Warps Per Scheduler", "No Eligible", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Block Limit Shared Mem", "Block Limit Registers"}
seen = set()
for r in rows[1:]:
    if r[mi] in keep and (r[ki][:40], r[mi]) not in seen:
        seen.add((r[ki][:40], r[mi]))
        print(f"{r[ki][:40]:40s} {r[mi]:40s} {r[vi]:>16s} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hdr = rr[0]
for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
             "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"):
    if name in hdr:
        i = hdr.index(name)
        for row in rr[2:]:
            print(f"{name:60s} {row[i]:>16s} {rr[1][i]}")
