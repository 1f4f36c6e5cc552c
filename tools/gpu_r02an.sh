# rasterisation group size for the row kinds (MOEB_RG 4 vs 8): Mixtral-like DRAM bytes and time
set -x
V=paper_2601_05296_b200/_variants
L=paper_2601_05296_b200/libmoeblaze.so
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
MOEBLAZE_LIB=$V/rg4.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for lib in $L $V/rg4.so; do
  n=$(basename $lib .so)
  MOEBLAZE_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base demangled -k "regex:tc_gemm_kernel<\(int\)(0|1|3|9)," -s 8 -c 8 --csv --log-file gpurun_out/r02an_ncu_$n.csv \
    python bench.py --workload mixtral --steps 2 --warmup 3 --no-cpu-baseline --no-memory --no-graph > /dev/null 2>&1
done
for r in 1 2; do STEPS=30 bash tools/tune_variants.sh mixtral $L $V/rg4.so; done 2>&1 | tee gpurun_out/r02an_variants.txt
