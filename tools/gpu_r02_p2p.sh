#!/bin/bash
# peer-memory EP exchange: GPU tests + a P = 1 bench of both exchanges
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/p2p_gpus.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_ep.py -x -q -k "p2p" -rs > gpurun_out/p2p_tests.txt 2>&1
echo "tests exit $?" >> gpurun_out/p2p_tests.txt
for X in p2p nccl; do
  timeout 900 python bench.py --ep --ep-exchange $X --steps 20 --warmup 5 --no-cpu-baseline \
    > gpurun_out/p2p_bench_mixtral_$X.json 2> gpurun_out/p2p_bench_mixtral_$X.err
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-memory \
  > gpurun_out/p2p_bench_mixtral_direct.json 2> gpurun_out/p2p_bench_mixtral_direct.err
