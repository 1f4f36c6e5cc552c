#!/bin/bash
# One GPU pass: full -m gpu suite, smoke, default bench (Mixtral) and DeepSeek bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_mixtral.json 2> gpurun_out/bench_mixtral.err
timeout 600 python bench.py --workload deepseek --no-cpu-baseline > gpurun_out/bench_deepseek.json 2> gpurun_out/bench_deepseek.err
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; cat gpurun_out/bench_mixtral.json gpurun_out/bench_deepseek.json
