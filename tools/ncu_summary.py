"""Summarise an ncu --set full report: key metrics per kernel launch (CSV 'details' page)."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Waves Per SM", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Executed Instructions", "Block Limit Registers", "Block Limit Shared Mem"]


def main(path, extra=()):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki, ni, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("ID"), hdr.index("Metric Name"),
                          hdr.index("Metric Value"), hdr.index("Metric Unit"))
    by = {}
    for r in rows[1:]:
        by.setdefault((r[ni], r[ki][:60]), {})[r[mi]] = (r[vi], r[ui])
    for (i, k), m in by.items():
        print(f"== launch {i}: {k}")
        for key in list(KEYS) + list(extra):
            if key in m:
                print(f"   {key:40s} {m[key][0]} {m[key][1]}")


def raw(path, pats):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("== ", r[hdr.index("Kernel Name")][:60])
        for j, h in enumerate(hdr):
            if any(p in h for p in pats):
                print(f"   {h:70s} {r[j]} {units[j]}")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "raw":
        raw(sys.argv[1], sys.argv[3:])
    else:
        main(sys.argv[1], sys.argv[2:])
