set -x
python -c "import __graft_entry__ as g; g.build()"
V=paper_2601_05296_b200/_variants
for W in deepseek mixtral; do
  STEPS=30 bash tools/tune_variants.sh $W paper_2601_05296_b200/libmoeblaze.so $V/prev.so paper_2601_05296_b200/libmoeblaze.so $V/prev.so paper_2601_05296_b200/libmoeblaze.so $V/prev.so
done 2>&1 | tee gpurun_out/r02k_variants.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sched.py -q -x 2>&1 | tail -2
