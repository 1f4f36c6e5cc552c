# skewed-routing weight-gradient kinds: ncu launch list + --set full of DW3 (kind 4), balanced vs skewed
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for R in balanced skewed; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:tc_gemm_kernel<\(int\)4," -s 3 -c 1 -f -o gpurun_out/full_r02ak_deepseek_k4_$R \
    python bench.py --workload deepseek --routing $R --steps 1 --warmup 3 --no-cpu-baseline --no-memory --no-graph > gpurun_out/full_r02ak_$R.log 2>&1
  echo "ncu $R exit $?"
done
