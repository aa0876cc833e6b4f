"""One-page summary of an ncu --set full report (speed of light, memory, occupancy,
dram bytes) for committing under profiles/."""
import csv
import subprocess
import sys

KEEP = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Issue Slots Busy", "Executed Ipc Active",
        "Warp Cycles Per Issued Instruction", "Achieved Occupancy", "Achieved Active Warps Per SM",
        "Theoretical Occupancy", "Registers Per Thread", "Static Shared Memory Per Block",
        "Block Size", "Grid Size", "Executed Instructions", "Branch Efficiency",
        "Avg. Active Threads Per Warp"]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
name = None
for r in rows[1:]:
    d = dict(zip(h, r))
    name = d.get("Kernel Name", name)
    if d.get("Metric Name") in KEEP:
        print(f"{d['Section Name'][:28]:28s} {d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hdr, units = rr[0], rr[1]
for row in rr[2:]:
    for k, u, v in zip(hdr, units, row):
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
                 "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_read.sum",
                 "gpu__time_duration.sum", "launch__registers_per_thread",
                 "sm__warps_active.avg.pct_of_peak_sustained_active"):
            print(f"raw {k:50s} {v} {u}")
print("kernel:", name)
