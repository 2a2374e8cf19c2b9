"""Print the key metrics of each kernel in an ncu --set full report.

    python profiles/ncu_details.py gpurun_out/x.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEEP = ("Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Issued Instructions", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size",
        "Block Size", "Theoretical Occupancy", "Achieved Occupancy", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "No Eligible", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Avg. Active Threads Per Warp", "Block Limit Registers", "Block Limit Shared Mem")


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, si, ni, vi, ui = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Value",
                                               "Metric Unit"))
    idx = h.index("ID")
    cur = None
    for r in rows[1:]:
        if r[idx] != cur:
            cur = r[idx]
            print(f"== launch {cur}: {r[ki][:110]}")
        if r[ni] in KEEP:
            print(f"   {r[ni]:40} {r[vi]:>16} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,"
                          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if rr:
        hh = rr[0]
        cols = [i for i, c in enumerate(hh) if c.startswith(("dram__bytes", "smsp__inst", "l1tex__data"))]
        for r in rr[2:]:
            print("   raw:", ", ".join(f"{hh[i]}={r[i]} {rr[1][i]}" for i in cols))


if __name__ == "__main__":
    main(sys.argv[1])
