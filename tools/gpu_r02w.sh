mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_ep_fullsize.py tests/test_gpu_sparse_ep.py tests/test_gpu_ep.py -q -s -rs -k "fullsize or token_rows or p2p or sparse_layer" > gpurun_out/r02w_tests.txt 2>&1
echo "exit $?" >> gpurun_out/r02w_tests.txt
for X in p2p nccl; do
  timeout 900 python bench.py --workload ep --ep --ep-exchange $X --steps 10 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r02w_bench_ep_$X.json 2> gpurun_out/r02w_bench_ep_$X.err
done
timeout 900 python bench.py --workload ep --steps 10 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r02w_bench_ep_direct.json 2> gpurun_out/r02w_bench_ep_direct.err
