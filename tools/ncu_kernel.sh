#!/bin/bash
# Per-launch time and DRAM bytes of one kernel (regex) in a short bench run.
# usage: tools/ncu_kernel.sh <regex> <workload> [count]
mkdir -p gpurun_out
f=gpurun_out/ncuk_$2.csv
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "regex:$1" -c ${3:-2} --csv --log-file $f python bench.py --workload $2 --steps 1 --warmup 1 --no-cpu-baseline --no-memory > /dev/null 2>&1
python - $f <<'PY'
import csv, sys
rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
agg = {}
for r in rows:
    agg.setdefault((r["ID"], r["Kernel Name"][:50]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
for (i, n), a in agg.items():
    t = a["gpu__time_duration.sum"]; b = a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]
    print(i, n, "%.1f us" % (t / 1e3), "%.1f MB" % (b / 1e6), "%.0f GB/s" % (b / t))
PY
