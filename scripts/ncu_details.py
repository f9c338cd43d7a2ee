"""Key numbers from an `ncu --page details --csv` export:
python scripts/ncu_details.py file.csv"""
import csv
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Block Size", "Grid Size",
        "Warp Cycles Per Issued Instruction", "Issued Ipc Active", "Executed Ipc Active", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block", "Waves Per SM",
        "Stall Long Scoreboard", "No Eligible", "One or More Eligible"]
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
seen = set()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    name = d.get("Metric Name", "")
    if any(name.startswith(k) for k in KEYS) and name not in seen:
        seen.add(name)
        print(f"{name:45s} {d.get('Metric Value', ''):>14s} {d.get('Metric Unit', '')}")
print(rows[1][4][:90] if len(rows) > 1 else "")
