# e2e slow-mode hunt: traced host-fed pipeline, DeepSeek-like, several back-to-back runs
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x 2>&1 | tail -1
for i in 1 2 3 4 5; do
  R=balanced; [ $i = 3 ] && R=skewed
  timeout 600 python bench.py --workload deepseek --routing $R --no-cpu-baseline --no-memory > gpurun_out/r02bb_bench_$i.json 2>/dev/null
  tail -1 gpurun_out/r02bb_bench_$i.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$i $R', d['ms_per_step'], e['ms_per_step'], e['pcie']['concurrent']['floor_ms_per_step'], json.dumps(e['trace']), e['allocator_in_timed_loop'])"
done
