# K-snake (alternate waves walk K backwards) for FWD_DOWN / BWD_DX: DRAM bytes and time
set -x
V=paper_2601_05296_b200/_variants
L=paper_2601_05296_b200/libmoeblaze.so
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
MOEBLAZE_LIB=$V/ksnake.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
MOEBLAZE_LIB=$V/ksnake.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "mixtral-False-swiglu-False-ab or deepseek-False-swiglu-False-ab" 2>&1 | tail -1
for lib in $L $V/ksnake.so; do
  n=$(basename $lib .so)
  MOEBLAZE_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none \
    --kernel-name-base demangled -k "regex:tc_gemm_kernel<\(int\)(1|3)," -s 4 -c 4 --csv --log-file gpurun_out/r02be_ncu_$n.csv \
    python bench.py --workload mixtral --steps 2 --warmup 3 --no-cpu-baseline --no-memory --no-graph > /dev/null 2>&1
done
for r in 1 2; do STEPS=30 bash tools/tune_variants.sh mixtral $L $V/ksnake.so; STEPS=30 bash tools/tune_variants.sh deepseek $L $V/ksnake.so; done 2>&1 | tee gpurun_out/r02be_variants.txt
