# fused accumulator zeroing (FWD_UP / BWD_DH epilogue warps) vs the separate pass; e2e PCIe floor
set -x
V=paper_2601_05296_b200/_variants
L=paper_2601_05296_b200/libmoeblaze.so
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_ep.py tests/test_gpu_r02.py tests/test_gpu_ep.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for W in deepseek mixtral; do
  for r in 1 2; do
    STEPS=30 bash tools/tune_variants.sh $W $L $V/nofuse.so
  done
done 2>&1 | tee gpurun_out/r02ac_variants.txt
timeout 900 python bench.py --workload deepseek --no-cpu-baseline > gpurun_out/r02ac_bench_deepseek.json 2>gpurun_out/r02ac_bench_deepseek.err
tail -1 gpurun_out/r02ac_bench_deepseek.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['e2e']['pcie']), d['e2e']['ms_per_step'], d['e2e']['floor_ms_per_step'], json.dumps(d['hbm_steps']['steps']))"
