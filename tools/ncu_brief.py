"""Brief digest of an `ncu --page details --csv` export: the speed-of-light,
occupancy, issue and stall numbers that decide what bounds a kernel."""
import csv
import sys

KEYS = ["Duration", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Achieved Occupancy", "Registers Per Thread",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Issue Slots Busy",
        "Executed Ipc Active", "Theoretical Occupancy", "No Eligible",
        "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block",
        "Block Limit Registers", "Block Limit Shared Mem", "Executed Instructions"]


def main(path):
    rows = list(csv.reader(open(path)))
    idx = {h: i for i, h in enumerate(rows[0])}
    for r in rows[1:]:
        name = r[idx["Metric Name"]]
        if name in KEYS:
            print(f"{r[idx['Kernel Name']][:24]:24s} | {name:36s} | {r[idx['Metric Value']]} "
                  f"{r[idx['Metric Unit']]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
