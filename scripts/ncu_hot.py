"""Summarise an ncu source page (SASS) into the hottest instructions."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(lines[1:]))
hdr = rows[0]
data = [r for r in rows[1:] if len(r) > 5 and r[hdr.index("Warp Stall Sampling (All Samples)")].isdigit()]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[i_s] or 0) for r in data)
print("total samples", tot, "instructions", len(data))
agg = {}
for r in data:
    op = r[i_src].split()[0] if r[i_src].split() else "?"
    if op.startswith("@"):
        op = r[i_src].split()[1]
    agg[op.split(".")[0]] = agg.get(op.split(".")[0], 0) + int(r[i_s] or 0)
print("by opcode:", sorted(agg.items(), key=lambda x: -x[1])[:15])
data.sort(key=lambda r: -int(r[i_s] or 0))
for r in data[:top]:
    st = sorted(((hdr[i][6:], int(r[i] or 0)) for i in stall_cols), key=lambda x: -x[1])[:3]
    print(f"{int(r[i_s]):6d} {r[i_src].strip()[:60]:60s} {st}")
