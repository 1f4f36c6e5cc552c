# bulk-reduction combine (MOEB_BULK_RED) vs red.add.v4; skewed-routing bench lines
set -x
V=paper_2601_05296_b200/_variants
L=paper_2601_05296_b200/libmoeblaze.so
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
MOEBLAZE_LIB=$V/bulkred.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_ep.py -q -x 2>&1 | tail -2
MOEBLAZE_LIB=$V/bulkred.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "mixtral-False-swiglu-False-ab or deepseek-False-swiglu-False-ab" 2>&1 | tail -2
for W in deepseek mixtral; do
  for r in 1 2; do
    STEPS=30 bash tools/tune_variants.sh $W $L $V/bulkred.so
  done
done 2>&1 | tee gpurun_out/r02af_variants.txt
for W in mixtral deepseek; do
  timeout 900 python bench.py --workload $W --routing skewed --no-cpu-baseline --no-memory > gpurun_out/r02af_bench_${W}_skewed.json 2>/dev/null
  tail -1 gpurun_out/r02af_bench_${W}_skewed.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$W skewed', d['value'], d['ms_per_step'], d['expert_load'], json.dumps(d['roofline']['per_kernel_ms']), d['roofline']['all_gemms'], d['clocks']['sm_mhz'])"
done
