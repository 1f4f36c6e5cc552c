mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ep.py tests/test_gpu_sparse_ep.py -x -q 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_rt_deepseek.csv python bench.py --workload deepseek --steps 1 --warmup 1 --no-cpu-baseline --no-memory > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_rt_deepseek.csv | grep -v tc_gemm | tail -12
