# default bench invocation (as the driver runs it) after the e2e warm-up change
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --gpus 1 > gpurun_out/r02bc_bench_default.json 2>gpurun_out/r02bc_bench_default.err
tail -1 gpurun_out/r02bc_bench_default.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['device'], d['cpu_baseline']['value'], d['memory']['peak_ratio'])"
