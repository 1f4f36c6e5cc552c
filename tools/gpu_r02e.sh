set -x
python -c "import __graft_entry__ as g; g.build()"
./tools/smem_align_probe | tee gpurun_out/r02e_smem_probe.txt
V=paper_2601_05296_b200/_variants
for W in deepseek mixtral; do
  STEPS=30 bash tools/tune_variants.sh $W paper_2601_05296_b200/libmoeblaze.so $V/rel.so paper_2601_05296_b200/libmoeblaze.so $V/rel.so
done 2>&1 | tee gpurun_out/r02e_variants.txt
