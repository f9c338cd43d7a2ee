"""Summarise an ncu launch list that carries gpu__time_duration.sum and
dram__bytes_{read,write}.sum per launch: per kernel launches, device time,
DRAM bytes and DRAM GB/s (cold-cache, serialised: compare shares).
python scripts/launch_traffic_summary.py in.csv[.gz] out.json"""
import collections
import csv
import gzip
import io
import json
import re
import sys

src, out = sys.argv[1], sys.argv[2]
txt = gzip.open(src, "rt").read() if src.endswith(".gz") else open(src).read()
rows = collections.OrderedDict()
for row in csv.DictReader(io.StringIO(txt[txt.find('"ID"'):])):
    try:
        v = float(row["Metric Value"].replace(",", ""))
    except (ValueError, KeyError):
        continue
    name = re.sub(r"\(.*", "", row["Kernel Name"]).replace("void ", "").replace("gs::", "")
    d = rows.setdefault(row["ID"], {"name": name, "ms": 0.0, "bytes": 0.0})
    u, m = row["Metric Unit"], row["Metric Name"]
    if m == "gpu__time_duration.sum":
        d["ms"] = v * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(u, 1.0)
    elif m.startswith("dram__bytes"):
        d["bytes"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
agg = {}
for d in rows.values():
    a = agg.setdefault(d["name"], {"launches": 0, "ms": 0.0, "dram_GB": 0.0, "live_launches": 0, "live_ms": 0.0})
    a["launches"] += 1
    a["ms"] += d["ms"]
    a["dram_GB"] += d["bytes"] / 1e9
    if d["ms"] > 0.01:          # launches past the stop flag exit at once
        a["live_launches"] += 1
        a["live_ms"] += d["ms"]
tot = sum(a["ms"] for a in agg.values())
for a in agg.values():
    a["share"] = a["ms"] / tot
    a["dram_GBps"] = a["dram_GB"] / (a["ms"] / 1e3) if a["ms"] else 0.0
    a["avg_live_ms"] = a["live_ms"] / a["live_launches"] if a["live_launches"] else 0.0
res = {"source": src, "total_ms": tot, "launches": sum(a["launches"] for a in agg.values()),
       "kernels": dict(sorted(agg.items(), key=lambda kv: -kv[1]["ms"]))}
json.dump(res, open(out, "w"), indent=1)
for k, a in list(res["kernels"].items())[:16]:
    print(f"{a['share']*100:6.2f}%  {a['launches']:5d} ({a['live_launches']:4d} live x {a['avg_live_ms']:7.4f} ms)  "
          f"{a['dram_GB']:8.3f} GB  {a['dram_GBps']:7.0f} GB/s  {k}")
