#!/bin/bash
# parity subset + Mixtral/DeepSeek bench lines (no CPU baseline, no memory pass)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for W in mixtral deepseek; do
  timeout 600 python bench.py --workload $W --no-cpu-baseline --no-memory 2>gpurun_out/bq_$W.err | tee gpurun_out/bq_$W.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$W', d['value'], d['ms_per_step'], r['kernel'], r['frac'], r['per_kernel_ms'], r['all_gemms'], d['clocks'])"
done
