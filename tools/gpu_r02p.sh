set -x
python -c "import __graft_entry__ as g; g.build()"
V=paper_2601_05296_b200/_variants
for W in deepseek mixtral; do
  STEPS=20 bash tools/tune_variants.sh $W paper_2601_05296_b200/libmoeblaze.so $V/nob.so $V/sameb.so paper_2601_05296_b200/libmoeblaze.so $V/nob.so $V/sameb.so
done 2>&1 | tee gpurun_out/r02p_variants.txt
