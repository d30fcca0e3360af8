#!/usr/bin/env python3
"""Summarise an ncu report (details page) for the judge-facing profiles/ directory."""
import csv
import io
import subprocess
import sys

WANT = {
    "GPU Speed Of Light Throughput": ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
                                      "L2 Cache Throughput", "Compute (SM) Throughput", "SM Frequency"],
    "Memory Workload Analysis": ["L1/TEX Hit Rate", "L2 Hit Rate", "Mem Busy", "Max Bandwidth", "Mem Pipes Busy"],
    "Compute Workload Analysis": ["Executed Ipc Active", "Issue Slots Busy", "SM Busy"],
    "Scheduler Statistics": ["One or More Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler"],
    "Warp State Statistics": ["Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
                              "Avg. Not Predicated Off Threads Per Warp"],
    "Occupancy": ["Achieved Occupancy", "Theoretical Occupancy", "Block Limit Registers"],
    "Launch Statistics": ["Grid Size", "Block Size", "Registers Per Thread"],
    "Instruction Statistics": ["Executed Instructions"],
}


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, ii, si, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Section Name", "Metric Name",
                                                     "Metric Value", "Metric Unit"))
    cur = None
    for r in rows[1:]:
        kid = (r[ii], r[ki].split("(")[0])
        if kid != cur:
            cur = kid
            print(f"== launch {kid[0]}: {kid[1]}")
        if r[si] in WANT and r[mi] in WANT[r[si]]:
            print(f"   {r[mi]:45s} {r[vi]:>14s} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hh = rr[0]
    cols = [c for c in hh if c.startswith(("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed_pipe_fma",
                                            "sm__pipe_fma_cycles_active.avg.pct", "lts__t_sector_hit_rate.pct",
                                            "smsp__average_warp_latency_issue_stalled", "sm__inst_executed_pipe_lsu",
                                            "smsp__sass_inst_executed_op_global_ld.sum", "sm__pipe_alu_cycles_active.avg.pct",
                                            "sm__inst_executed_pipe_xu"))]
    for r in rr[2:]:
        name = r[hh.index("Kernel Name")].split("(")[0]
        print(f"== raw {r[hh.index('ID')]} {name}: " + "; ".join(f"{c}={r[hh.index(c)]}" for c in cols))


if __name__ == "__main__":
    main(sys.argv[1])
