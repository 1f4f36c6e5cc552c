set -x
python -c "import __graft_entry__ as g; g.build()"
V=paper_2601_05296_b200/_variants
MOEBLAZE_LIB=$V/wide.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r02.py tests/test_gpu_sched.py -q -x 2>&1 | tail -3
MOEBLAZE_LIB=$V/wide.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "mixtral-False-swiglu-False-ab or deepseek-False-swiglu-False-ab" 2>&1 | tail -2
for W in deepseek mixtral; do
  STEPS=30 bash tools/tune_variants.sh $W paper_2601_05296_b200/libmoeblaze.so $V/wide.so paper_2601_05296_b200/libmoeblaze.so $V/wide.so
done 2>&1 | tee gpurun_out/r02t_variants.txt
