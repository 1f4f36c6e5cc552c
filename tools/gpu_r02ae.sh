# down-projection split + y_ready (C3 overlap), sm_reserve; deterministic-combine cost
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_sparse_ep.py tests/test_gpu_ep.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_ep_fullsize.py -q -x 2>&1 | tail -2
for W in mixtral deepseek; do
  timeout 900 python bench.py --workload $W --deterministic --no-cpu-baseline --no-memory > gpurun_out/r02ae_bench_${W}_det.json 2>/dev/null
  timeout 900 python bench.py --workload $W --no-cpu-baseline --no-memory > gpurun_out/r02ae_bench_${W}.json 2>/dev/null
  for f in ${W}_det $W; do tail -1 gpurun_out/r02ae_bench_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], json.dumps(d['roofline']['per_kernel_ms']), d['clocks']['sm_mhz'])"; done
done
