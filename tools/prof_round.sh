#!/bin/bash
# Evidence pass for profiles/: parity subset, launch list, ncu --set full of BWD_DH and DW12.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 15 --csv \
  --log-file gpurun_out/launches_r01b.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-memory > /dev/null 2>&1
for K in 2 5; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:tc_gemm_kernel<\(int\)$K," -s 3 -c 1 -f -o gpurun_out/prof_k$K python bench.py --steps 1 --warmup 3 \
    --no-cpu-baseline --no-memory > gpurun_out/prof_k$K.log 2>&1
done
ls -la gpurun_out
