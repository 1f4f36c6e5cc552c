# DW3/DW12 longest-K-first tile order (MOEB_WG_LPT) vs baseline, balanced and skewed DeepSeek-like / Mixtral-like
set -x
V=paper_2601_05296_b200/_variants
L=paper_2601_05296_b200/libmoeblaze.so
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
MOEBLAZE_LIB=$V/lpt.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
MOEBLAZE_LIB=$V/lpt.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "deepseek-False-swiglu-False-ab or mixtral-False-swiglu-False-ab" 2>&1 | tail -2
for r in 1 2; do
  for W in deepseek mixtral; do
    for R in skewed balanced; do
      for lib in $L $V/lpt.so; do
        MOEBLAZE_LIB=$lib timeout 300 python bench.py --workload $W --routing $R --steps 30 --warmup 4 --no-cpu-baseline --no-memory --no-graph 2>/dev/null \
          | python -c "
import json,sys
r=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$(basename $lib)', '$W', '$R', r['value'], r['ms_per_step'], json.dumps(r['roofline']['per_kernel_ms']), r['clocks'].get('sm_mhz'))"
      done
    done
  done
done 2>&1 | tee gpurun_out/r02al_variants.txt
