#!/bin/bash
# Launch lists (every kernel of 1 warm-up + 1 timed step, cold-cache serialised)
# for Mixtral and DeepSeek, and ncu --set full of selected GEMM kinds.
# usage: tools/prof_launches.sh TAG "mixtral:3 deepseek:2 ..."
TAG=${1:-r01}; FULL=${2:-}
mkdir -p gpurun_out
for W in mixtral deepseek; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__cycles_elapsed.avg.per_second --clock-control none \
    --csv --log-file gpurun_out/launches_${TAG}_${W}.csv \
    python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline --no-memory > gpurun_out/launches_${TAG}_${W}.log 2>&1
done
for WK in $FULL; do
  W=${WK%%:*}; K=${WK##*:}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:tc_gemm_kernel<\(int\)$K," -s 2 -c 1 -f -o gpurun_out/full_${TAG}_${W}_k$K \
    python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline --no-memory > gpurun_out/full_${TAG}_${W}_k$K.log 2>&1
done
ls -la gpurun_out
