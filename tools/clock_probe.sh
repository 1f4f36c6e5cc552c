#!/bin/bash
# SM clock + DRAM bytes per GEMM launch (ncu, clocks uncontrolled) for a list of libraries
# usage: tools/clock_probe.sh workload lib.so...
wl=$1; shift
mkdir -p gpurun_out
for so in "$@"; do
  n=$(basename $so .so)
  MOEBLAZE_LIB=$so timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:tc_gemm_kernel -s 12 -c 6 --csv --log-file gpurun_out/clk_${wl}_$n.csv \
    python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-memory > /dev/null 2>&1
  echo "== $n"; python - gpurun_out/clk_${wl}_$n.csv <<'PY'
import csv,sys
rows=list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
agg={}
for r in rows:
    k=(int(r["ID"]), r["Kernel Name"][:40]); agg.setdefault(k,{})[r["Metric Name"]]=r["Metric Value"]
for k,a in agg.items(): print(k, {m.split("__")[1][:28]:v for m,v in a.items()})
PY
done
