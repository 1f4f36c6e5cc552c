set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ep.py tests/test_gpu_sparse_ep.py -q -x 2>&1 | tail -2
for W in deepseek mixtral; do
  for LIB in paper_2601_05296_b200/libmoeblaze.so paper_2601_05296_b200/_variants/prev.so; do
    MOEBLAZE_LIB=$LIB timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k "regex:router_dx" -c 4 --csv --log-file gpurun_out/r02q_rdx_${W}_$(basename $LIB .so).csv python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-memory > /dev/null 2>&1
    python tools/launch_summary.py gpurun_out/r02q_rdx_${W}_$(basename $LIB .so).csv | tail -2
  done
done
