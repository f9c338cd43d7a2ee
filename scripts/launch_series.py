"""Per-kernel totals and per-launch series of the second run in an ncu launch list (gz csv).
python scripts/launch_series.py file.csv.gz [kernel ...]"""
import collections
import csv
import gzip
import io
import re
import sys

with gzip.open(sys.argv[1], "rt") as f:
    txt = f.read()
r = csv.DictReader(io.StringIO(txt[txt.find('"ID"'):]))
per = collections.defaultdict(list)
for row in r:
    try:
        v = float(row["Metric Value"].replace(",", ""))
    except (ValueError, KeyError):
        continue
    u = row["Metric Unit"]
    ms = v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v
    name = re.sub(r"[<(].*", "", row["Kernel Name"]).replace("void ", "").replace("gs::", "")
    per[name].append(ms)
tot = sum(sum(v) for v in per.values())
print(f"total {tot:.2f} ms, {sum(len(v) for v in per.values())} launches")
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))[:28]:
    print(f"{k:24s} {sum(v):9.3f} ms {len(v):5d}")
for k in sys.argv[2:]:
    v = per[k]
    h = len(v) // 2
    print(k, " ".join(f"{x:.2f}" for x in v[h:h + 60]))
