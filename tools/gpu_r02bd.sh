# launch lists at the round's final code (ncu gpu__time_duration + DRAM bytes, --clock-control none)
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for W in mixtral deepseek; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 60 -c 60 --csv \
    --log-file gpurun_out/launches_r02bd_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --no-memory --no-graph > /dev/null 2>&1
  echo "ncu $W exit $?"
done
