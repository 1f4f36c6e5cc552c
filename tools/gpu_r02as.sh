# 8-warp epilogues for FWD_UP (MOEB_UP_EPI8) and FWD_DOWN/BWD_DX (MOEB_RED_EPI8) on both shapes
set -x
V=paper_2601_05296_b200/_variants
L=paper_2601_05296_b200/libmoeblaze.so
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for lib in $V/up8.so $V/red8.so; do MOEBLAZE_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1; done
for W in deepseek mixtral; do
  for r in 1 2; do
    STEPS=30 bash tools/tune_variants.sh $W $L $V/up8.so $V/red8.so
  done
done 2>&1 | tee gpurun_out/r02as_variants.txt
