set -x
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/b_mix.json 2>gpurun_out/b_mix.err
timeout 600 python bench.py --workload deepseek --steps 10 --warmup 5 --no-cpu-baseline --no-memory > gpurun_out/b_ds.json 2>&1
timeout 600 python bench.py --workload deepseek --steps 10 --warmup 5 --no-cpu-baseline --no-memory --deterministic > gpurun_out/b_ds_det.json 2>&1
timeout 600 python bench.py --workload ep --ep --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_ep.json 2>&1
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --activation silu > gpurun_out/b_mix_silu.json 2>&1
