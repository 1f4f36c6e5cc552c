# Final full check (router dX prefetch on): full GPU suite, smoke, bench lines
set -x
python -c "import __graft_entry__ as g; g.build()"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -s 2>&1 | grep -v "^$" > gpurun_out/r02ba_pytest_full.txt
tail -1 gpurun_out/r02ba_pytest_full.txt
grep -E "FAILED" gpurun_out/r02ba_pytest_full.txt | head
timeout 900 python bench.py > gpurun_out/r02ba_bench_default.json 2>gpurun_out/r02ba_bench_default.err
timeout 900 python bench.py --workload deepseek --no-cpu-baseline > gpurun_out/r02ba_bench_deepseek.json 2>gpurun_out/r02ba_bench_deepseek.err
for f in default deepseek; do tail -1 gpurun_out/r02ba_bench_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['trace'], r['kernel'], r['frac'], r['all_gemms'], d['clocks'])"; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02ba_bench_reference.json 2>/dev/null; tail -1 gpurun_out/r02ba_bench_reference.json | cut -c1-200
