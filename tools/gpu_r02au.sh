# ExpertParallelMoE with one reused side stream; bench line device info
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_ep.py tests/test_gpu_pipeline.py -q -x 2>&1 | tail -1
timeout 600 python bench.py --workload ep --ep --steps 20 --no-cpu-baseline --no-memory --no-graph 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['device'])"
