"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel counts, total device time and share (cold-cache, serialised:
compare shares, not absolutes)."""
import csv
import json
import re
import sys

src, out = sys.argv[1], sys.argv[2]
if src.endswith(".gz"):
    import gzip
    fh = gzip.open(src, "rt")
else:
    fh = open(src)
rows = [r for r in csv.reader(fh) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = {}
for r in rows[1:]:
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
    t = float(r[vi].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r[ui], 1e-6)
    a = agg.setdefault(name, {"launches": 0, "ms": 0.0})
    a["launches"] += 1
    a["ms"] += t
tot = sum(a["ms"] for a in agg.values())
for a in agg.values():
    a["share"] = a["ms"] / tot
    a["avg_ms"] = a["ms"] / a["launches"]
res = {"source": src, "total_ms": tot, "launches": sum(a["launches"] for a in agg.values()),
       "kernels": dict(sorted(agg.items(), key=lambda kv: -kv[1]["ms"]))}
json.dump(res, open(out, "w"), indent=1)
for k, a in list(res["kernels"].items())[:14]:
    print(f"{a['share']*100:6.2f}%  {a['launches']:5d} x {a['avg_ms']:8.4f} ms  {k}")
