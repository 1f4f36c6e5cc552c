set -x
V=paper_2601_05296_b200/_variants
MOEBLAZE_LIB=$V/widerow.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r02.py tests/test_gpu_sched.py tests/test_gpu_sparse_ep.py -q -x 2>&1 | tail -3
MOEBLAZE_LIB=$V/widerow.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "mixtral-False-swiglu-False-ab or deepseek-False-swiglu-False-ab" 2>&1 | tail -2
for W in mixtral deepseek; do
  STEPS=30 bash tools/tune_variants.sh $W paper_2601_05296_b200/libmoeblaze.so $V/widerow.so $V/widedx.so paper_2601_05296_b200/libmoeblaze.so $V/widerow.so $V/widedx.so
done 2>&1 | tee gpurun_out/r02y_variants.txt
