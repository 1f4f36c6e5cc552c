"""Summarise an ncu launch-list CSV (gpu__time_duration.sum [+ dram bytes]) per kernel.
usage: python tools/launch_summary.py launches.csv [first_id] [last_id]"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else 10 ** 9
agg = OrderedDict()
for r in rows:
    i = int(r["ID"])
    if not lo <= i <= hi:
        continue
    name = r["Kernel Name"][:70]
    m = r["Metric Name"]
    v = float(r["Metric Value"].replace(",", ""))
    a = agg.setdefault((i, name), {})
    a[m] = v
tot = sum(a.get("gpu__time_duration.sum", 0) for a in agg.values())
for (i, name), a in agg.items():
    t = a.get("gpu__time_duration.sum", 0)
    gb = (a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)) / 1e9
    print(f"{i:4d} {name:70s} {t/1e3:9.1f} us {100*t/tot:5.1f}% {gb:7.3f} GB {gb/(t*1e-9)/1e3 if t else 0:6.0f} TB/s")
print(f"total {tot/1e6:.3f} ms")
