set -x
python -c "import __graft_entry__ as g; g.build()"
cp paper_2601_05296_b200/libmoeblaze.so gpurun_out/r02u_lib.so
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -s 2>&1 | grep -v "^$" > gpurun_out/r02u_pytest_full.txt
tail -1 gpurun_out/r02u_pytest_full.txt
grep -E "FAILED" gpurun_out/r02u_pytest_full.txt | head
timeout 900 python bench.py > gpurun_out/r02u_bench_default.json 2>gpurun_out/r02u_bench_default.err
timeout 900 python bench.py --workload deepseek --no-cpu-baseline > gpurun_out/r02u_bench_deepseek.json 2>gpurun_out/r02u_bench_deepseek.err
for f in default deepseek; do tail -1 gpurun_out/r02u_bench_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], r['kernel'], r['frac'], r['all_gemms'], d['clocks']['sm_mhz'])"; done
for W in mixtral deepseek; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 60 -c 60 --csv \
    --log-file gpurun_out/launches_r02u_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --no-memory > /dev/null 2>&1
done
tools/ncu_full.sh 3 mixtral r02u
tools/ncu_full.sh 5 mixtral r02u
tools/ncu_full.sh 7 deepseek r02u
