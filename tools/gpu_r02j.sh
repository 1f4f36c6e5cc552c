set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -s 2>&1 | grep -v "^$" > gpurun_out/r02j_pytest_full.txt
tail -2 gpurun_out/r02j_pytest_full.txt
grep -E "FAILED|Error" gpurun_out/r02j_pytest_full.txt | head -20
grep -E "^(mixtral|deepseek|sweep_4k|ep) " gpurun_out/r02j_pytest_full.txt | head -20
for W in deepseek mixtral; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 60 -c 60 --csv \
    --log-file gpurun_out/launches_r02j_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --no-memory > /dev/null 2>&1
  echo "ncu $W $?"
done
