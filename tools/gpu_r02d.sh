set -x
python -c "import __graft_entry__ as g; g.build()"
cp paper_2601_05296_b200/libmoeblaze.so gpurun_out/r02d_lib.so
timeout 1800 python -m pytest tests -m gpu -q -s 2>&1 | grep -v "^$" > gpurun_out/r02d_pytest_full.txt
tail -3 gpurun_out/r02d_pytest_full.txt
grep -E "FAILED|rowwise" gpurun_out/r02d_pytest_full.txt | head -20
for W in mixtral deepseek; do
  timeout 600 python bench.py --workload $W --no-cpu-baseline --no-memory > gpurun_out/r02d_bench_$W.json 2>gpurun_out/r02d_bench_$W.err
  python -c "import json;d=json.loads(open('gpurun_out/r02d_bench_$W.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$W',d['value'],d['ms_per_step'],r['per_kernel_ms'],r['all_gemms'],d['clocks']['sm_mhz'])"
done
tools/ncu_full.sh 7 deepseek r02d
tools/ncu_full.sh 9 mixtral r02d
tools/ncu_full.sh 1 deepseek r02d
