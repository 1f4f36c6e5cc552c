set -x
python -c "import __graft_entry__ as g; g.build()"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2700 python -m pytest tests -m gpu -q -s -rs 2>&1 | grep -v "^$" > gpurun_out/r02v_pytest_full.txt
tail -3 gpurun_out/r02v_pytest_full.txt
grep -E "FAILED" gpurun_out/r02v_pytest_full.txt | head
timeout 900 python bench.py > gpurun_out/r02v_bench_default.json 2>gpurun_out/r02v_bench_default.err
tail -1 gpurun_out/r02v_bench_default.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], d['e2e']['value'], r['kernel'], r['frac'], d['clocks']['sm_mhz'])"
