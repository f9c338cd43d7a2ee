"""Summarise an ncu --csv launch list (gpu__time_duration.sum): total ms and
count per kernel.  python scripts/launch_table.py file.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1]).read().splitlines()))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
          "s": 1e3, "second": 1e3}.get(unit, 1.0)
    k = d["Kernel Name"].split("(")[0][:70]
    tot[k] += v
    cnt[k] += 1
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:10.3f} ms {cnt[k]:6d}  {k}")
print(f"total {sum(tot.values()):.3f} ms over {sum(cnt.values())} launches")
