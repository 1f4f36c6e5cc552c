set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_r02.py tests/test_gpu_ep.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --workload ep --ep --no-cpu-baseline --no-memory > gpurun_out/r02s_ep_p1.json 2>gpurun_out/r02s_ep_p1.err; tail -1 gpurun_out/r02s_ep_p1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'])"
timeout 900 python bench.py --workload ep --no-cpu-baseline --no-memory > gpurun_out/r02s_ep_direct.json 2>gpurun_out/r02s_ep_direct.err; tail -1 gpurun_out/r02s_ep_direct.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'])"
