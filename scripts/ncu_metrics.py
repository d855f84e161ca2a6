"""Prints selected metrics of every kernel in an ncu report (details page, csv)."""
import csv, io, subprocess, sys
WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "Executed Ipc Active",
        "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    seen = {}
    for r in rows[1:]:
        if len(r) <= vi or r[mi] not in WANT:
            continue
        seen.setdefault(r[ki].split("(")[0], {})[r[mi]] = f"{r[vi]} {r[ui]}"
    for k, m in seen.items():
        print("==", rep, k)
        for w in WANT:
            if w in m:
                print(f"   {w:36s} {m[w]}")
