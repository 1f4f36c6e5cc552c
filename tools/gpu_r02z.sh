set -x
V=paper_2601_05296_b200/_variants
L=paper_2601_05296_b200/libmoeblaze.so
MOEBLAZE_LIB=$V/dieexp.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sched.py -q -x 2>&1 | tail -2
MOEBLAZE_LIB=$V/dieexp.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "mixtral-False-swiglu-False-ab or deepseek-False-swiglu-False-ab" 2>&1 | tail -2
for W in deepseek mixtral; do
  for r in 1 2; do
    STEPS=30 bash tools/tune_variants.sh $W $L $V/dieexp.so
    MOEBLAZE_DIE=0 STEPS=30 bash tools/tune_variants.sh $W $L | sed 's/^libmoeblaze.so/nodie/'
  done
done 2>&1 | tee gpurun_out/r02z_variants.txt
