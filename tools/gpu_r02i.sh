set -x
python -c "import __graft_entry__ as g; g.build()"
V=paper_2601_05296_b200/_variants
for W in deepseek mixtral; do
  STEPS=30 bash tools/tune_variants.sh $W paper_2601_05296_b200/libmoeblaze.so $V/dh5.so $V/tight.so paper_2601_05296_b200/libmoeblaze.so $V/dh5.so $V/tight.so
done 2>&1 | tee gpurun_out/r02i_variants.txt
MOEBLAZE_LIB=$V/dh5.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "layer" 2>&1 | tail -2
