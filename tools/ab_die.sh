#!/bin/bash
# A/B of the die-aware scheduler split (MOEBLAZE_DIE=0 = one list) + DRAM bytes per GEMM launch.
mkdir -p gpurun_out
for W in ${WORKLOADS:-mixtral deepseek}; do
  for D in 1 0; do
    for rep in 1 2; do
      MOEBLAZE_DIE=$D timeout 300 python bench.py --workload $W --no-cpu-baseline --no-memory 2>/dev/null | python -c "
import json,sys
r=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$W die=$D', r['value'], r['ms_per_step'], json.dumps(r['roofline']['per_kernel_ms']), r['clocks'].get('sm_mhz'), r['clocks'].get('samples'))"
    done
  done
  for D in 1 0; do
    MOEBLAZE_DIE=$D timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_ltcfabric.sum \
      --clock-control none -k regex:tc_gemm_kernel -s 14 -c 7 --csv --log-file gpurun_out/dram_${W}_die$D.csv \
      python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-memory > /dev/null 2>&1
  done
done
