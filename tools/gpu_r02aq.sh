# p2p exchange with the C3 overlap (y_ready -> Y signal on a side stream) + token_rows-bounded split finalize
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_ep.py tests/test_gpu_sparse_ep.py -q -x 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_ep_fullsize.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --workload ep --ep --ep-exchange p2p --no-cpu-baseline --no-memory > gpurun_out/r02aq_bench_ep_p2p.json 2>/dev/null
timeout 600 python bench.py --workload ep --ep --no-cpu-baseline --no-memory > gpurun_out/r02aq_bench_ep_nccl.json 2>/dev/null
timeout 600 python bench.py --workload ep --no-cpu-baseline --no-memory > gpurun_out/r02aq_bench_ep_direct.json 2>/dev/null
for f in p2p nccl direct; do tail -1 gpurun_out/r02aq_bench_ep_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['ms_per_step'], d['e2e']['value'])"; done
