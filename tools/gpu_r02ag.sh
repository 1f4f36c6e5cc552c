# red.add with an L2 evict_last hint (MOEB_RED_EVICT_LAST) vs plain red.add
set -x
V=paper_2601_05296_b200/_variants
L=paper_2601_05296_b200/libmoeblaze.so
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
MOEBLAZE_LIB=$V/evl.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for W in deepseek mixtral; do
  for r in 1 2; do
    STEPS=30 bash tools/tune_variants.sh $W $L $V/evl.so
  done
done 2>&1 | tee gpurun_out/r02ag_variants.txt
for lib in $L $V/evl.so; do
  for W in deepseek mixtral; do
    n=$(basename $lib .so)
    MOEBLAZE_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k "regex:tc_gemm_kernel<\(int\)(1|3)," -s 4 -c 4 --csv --log-file gpurun_out/r02ag_ncu_${n}_$W.csv \
      python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --no-memory --no-graph > /dev/null 2>&1
    echo "$n $W"; python - <<PY
import csv
rows=[r for r in csv.DictReader(l for l in open("gpurun_out/r02ag_ncu_${n}_$W.csv") if not l.startswith("=="))]
for r in rows: print(r["Kernel Name"][:40], r["Metric Name"], r["Metric Unit"], r["Metric Value"])
PY
  done
done
