# DW12 under skewed routing with the LPT order: balance across SMs (ncu --set full)
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for R in balanced skewed; do
  timeout 900 ncu --set full --clock-control none --kernel-name-base demangled \
    -k "regex:tc_gemm_kernel<\(int\)5," -s 3 -c 1 -f -o gpurun_out/full_r02av_deepseek_k5_$R \
    python bench.py --workload deepseek --routing $R --steps 1 --warmup 3 --no-cpu-baseline --no-memory --no-graph > /dev/null 2>&1
  echo "ncu $R exit $?"
done
