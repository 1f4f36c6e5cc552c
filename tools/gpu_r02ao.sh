# Final evidence pass of round 2: full GPU suite, smoke, bench lines, launch lists,
# ncu --set full of the top kernels
set -x
python -c "import __graft_entry__ as g; g.build()"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -s 2>&1 | grep -v "^$" > gpurun_out/r02ao_pytest_full.txt
tail -1 gpurun_out/r02ao_pytest_full.txt
grep -E "FAILED" gpurun_out/r02ao_pytest_full.txt | head
timeout 900 python bench.py > gpurun_out/r02ao_bench_default.json 2>gpurun_out/r02ao_bench_default.err
timeout 900 python bench.py --workload deepseek --no-cpu-baseline > gpurun_out/r02ao_bench_deepseek.json 2>gpurun_out/r02ao_bench_deepseek.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02ao_bench_reference.json 2>gpurun_out/r02ao_bench_reference.err
for f in default deepseek; do tail -1 gpurun_out/r02ao_bench_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['floor_ms_per_step'], r['kernel'], r['frac'], r['all_gemms'], d['clocks'])"; done
for W in mixtral deepseek; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 60 -c 60 --csv \
    --log-file gpurun_out/launches_r02ao_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --no-memory --no-graph > /dev/null 2>&1
done
tools/ncu_full.sh 3 mixtral r02ao --no-graph
tools/ncu_full.sh 5 mixtral r02ao --no-graph
tools/ncu_full.sh 7 deepseek r02ao --no-graph
tools/ncu_full.sh 1 deepseek r02ao --no-graph
timeout 900 python bench.py --workload deepseek --routing skewed --no-cpu-baseline --no-memory > gpurun_out/r02ao_bench_deepseek_skewed.json 2>/dev/null
timeout 900 python bench.py --workload mixtral --routing skewed --no-cpu-baseline --no-memory > gpurun_out/r02ao_bench_mixtral_skewed.json 2>/dev/null
timeout 900 python bench.py --workload ep --ep --no-cpu-baseline --no-memory > gpurun_out/r02ao_bench_ep_p1.json 2>/dev/null
for f in deepseek_skewed mixtral_skewed ep_p1; do tail -1 gpurun_out/r02ao_bench_$f.json | cut -c1-300; done
