set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -v "^$" | tail -40 > gpurun_out/r02b_pytest.txt
tail -5 gpurun_out/r02b_pytest.txt
grep -E "rowwise|PASS|FAIL|Error|error" gpurun_out/r02b_pytest.txt | head -20
for W in mixtral deepseek; do
  timeout 600 python bench.py --workload $W --no-cpu-baseline > gpurun_out/r02b_bench_$W.json 2>gpurun_out/r02b_bench_$W.err
  python -c "import json;d=json.load(open('gpurun_out/r02b_bench_$W.json'));r=d['roofline'];print('$W',d['value'],d['ms_per_step'],r['per_kernel_ms'],r['all_gemms'],d['clocks']['sm_mhz'],json.dumps(d['memory']))"
done
timeout 600 python bench.py --workload ep --ep --no-cpu-baseline --no-memory > gpurun_out/r02b_bench_ep_p1.json 2>gpurun_out/r02b_bench_ep_p1.err
timeout 600 python bench.py --workload ep --no-cpu-baseline --no-memory > gpurun_out/r02b_bench_ep_direct.json 2>gpurun_out/r02b_bench_ep_direct.err
for f in ep_p1 ep_direct; do python -c "import json;d=json.load(open('gpurun_out/r02b_bench_$f.json'));print('$f',d['value'],d['ms_per_step'],d['roofline']['per_kernel_ms'],d['e2e']['value'])"; done
