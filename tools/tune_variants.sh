#!/bin/bash
# Compile-time tuning sweep: run bench.py against each prebuilt variant library
# (paper_2601_05296_b200/_variants/*.so, built with `python -m
# paper_2601_05296_b200.build --out ... -D ...`) and print the per-kernel times.
# usage: bash tools/tune_variants.sh <workload> <variant.so>...
wl=$1; shift
for so in "$@"; do
  for rep in 1 2; do
    MOEBLAZE_LIB=$so timeout 300 python bench.py --workload $wl --steps ${STEPS:-40} --warmup 4 --no-cpu-baseline --no-memory 2>/dev/null \
      | python -c "
import json,sys
r=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$(basename $so)', '$wl', r['value'], r['ms_per_step'], json.dumps(r['roofline']['per_kernel_ms']), r['clocks'].get('sm_mhz'), r['clocks'].get('samples'), r['clocks'].get('power_w_max'))"
  done
done
