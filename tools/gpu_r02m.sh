set -x
python -c "import __graft_entry__ as g; g.build()"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -q -s 2>&1 | grep -v "^$" > gpurun_out/r02m_pytest_full.txt
tail -2 gpurun_out/r02m_pytest_full.txt
grep -E "FAILED|deepseek full tensors" gpurun_out/r02m_pytest_full.txt | cut -c1-600
timeout 900 python bench.py > gpurun_out/r02m_bench_default.json 2>gpurun_out/r02m_bench_default.err
tail -c 600 gpurun_out/r02m_bench_default.json
timeout 900 python bench.py --workload deepseek --no-cpu-baseline > gpurun_out/r02m_bench_deepseek.json 2>gpurun_out/r02m_bench_deepseek.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02m_bench_reference.json 2>gpurun_out/r02m_bench_reference.err
tail -c 400 gpurun_out/r02m_bench_reference.json
