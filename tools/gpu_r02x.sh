mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_ep_fullsize.py tests/test_gpu_ep.py -q -s -rs -k "p2p" > gpurun_out/r02x_tests.txt 2>&1
echo "exit $?" >> gpurun_out/r02x_tests.txt
for W in mixtral ep; do
  timeout 900 python bench.py --workload $W --ep --ep-exchange p2p --steps 10 --warmup 3 --no-cpu-baseline --no-memory \
    > gpurun_out/r02x_bench_${W}_p2p.json 2> gpurun_out/r02x_bench_${W}_p2p.err
done
