set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
for W in mixtral deepseek; do
  timeout 600 python bench.py --workload $W --no-cpu-baseline --no-memory > gpurun_out/r02a_bench_$W.json 2>gpurun_out/r02a_bench_$W.err
  tail -c 3000 gpurun_out/r02a_bench_$W.json | head -c 1500; echo
done
tools/ncu_full.sh 7 mixtral r02a
tools/ncu_full.sh 7 deepseek r02a
tools/ncu_full.sh 3 mixtral r02a
