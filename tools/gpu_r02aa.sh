for W in mixtral deepseek; do
  timeout 900 python bench.py --workload $W --steps 20 --warmup 4 --no-cpu-baseline > gpurun_out/r02aa_bench_$W.json 2> gpurun_out/r02aa_bench_$W.err
done
timeout 600 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2 > gpurun_out/r02aa_tests.txt
