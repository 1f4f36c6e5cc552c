set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_ep.py tests/test_gpu_r02.py tests/test_gpu_sparse_ep.py -x -q -s 2>&1 | grep -v "^$" | tail -30 > gpurun_out/r02c_pytest.txt
tail -3 gpurun_out/r02c_pytest.txt
grep -E "rowwise" gpurun_out/r02c_pytest.txt | head -10
V=paper_2601_05296_b200/_variants
for W in deepseek mixtral; do
  STEPS=30 bash tools/tune_variants.sh $W paper_2601_05296_b200/libmoeblaze.so $V/nopf.so $V/epi4.so $V/epi4nopf.so paper_2601_05296_b200/libmoeblaze.so $V/nopf.so
done 2>&1 | tee gpurun_out/r02c_variants.txt
