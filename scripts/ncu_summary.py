"""Summarise an ncu --set full report: per kernel time, DRAM bytes/throughput,
occupancy and the top stall reasons.  Optionally write profiles/*.json."""
import csv
import json
import subprocess
import sys

rep = sys.argv[1]
out_json = sys.argv[2] if len(sys.argv) > 2 else None
if rep.endswith(".csv.gz"):
    import gzip
    raw = gzip.open(rep, "rt").read()
elif rep.endswith(".csv"):
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}


def g(r, k, cast=float):
    i = col.get(k)
    if i is None or r[i] in ("", "n/a"):
        return None
    try:
        return cast(r[i].replace(",", ""))
    except ValueError:
        return r[i]


summary = {"report": rep, "kernels": {}}
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    short = name.split("(")[0].replace("void ", "").split("<")[0].replace("gs::", "")
    t_us = g(r, "gpu__time_duration.sum")
    if units[col["gpu__time_duration.sum"]] == "ms":
        t_us *= 1e3
    elif units[col["gpu__time_duration.sum"]] == "ns":
        t_us /= 1e3
    def mb(k):
        v = g(r, k)
        u = units[col[k]] if k in col else ""
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
        return None if v is None else v * scale
    rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
    st = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                  g(r, h)) for h in hdr if h.startswith("smsp__average_warps_issue_stalled")
                 and g(r, h) is not None), key=lambda x: -x[1])[:5]
    k = {"name": name[:120], "time_us": t_us, "dram_read_MB": rd, "dram_write_MB": wr,
         "dram_bytes": (rd + wr) * 1e6 if rd is not None else None,
         "dram_GBps": (rd + wr) / t_us * 1e3 if rd is not None else None,
         "dram_pct": g(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
         "sm_pct": g(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
         "warps_active_pct": g(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
         "registers": g(r, "launch__registers_per_thread"),
         "inst_executed": g(r, "smsp__inst_executed.sum"),
         "top_stalls": [(a, round(b, 2)) for a, b in st]}
    summary["kernels"].setdefault(short, k)
    print(f"{short:14s} {t_us:9.1f}us  dram {k['dram_GBps'] or 0:7.0f} GB/s ({k['dram_pct'] or 0:5.1f}%)  "
          f"R {rd or 0:8.1f}MB W {wr or 0:8.1f}MB  sm {k['sm_pct'] or 0:5.1f}%  occ {k['warps_active_pct'] or 0:5.1f}%  "
          f"regs {k['registers']}  {k['top_stalls'][:3]}")
if out_json:
    with open(out_json, "w") as fh:
        json.dump(summary, fh, indent=1)
