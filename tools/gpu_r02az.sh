# K1 routing: L2 prefetch of the CTA's X block (MOEB_ROUTE_PF)
set -x
V=paper_2601_05296_b200/_variants
L=paper_2601_05296_b200/libmoeblaze.so
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
MOEBLAZE_LIB=$V/rtpf.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for r in 1 2; do
  for W in deepseek mixtral; do
    for lib in $L $V/rtpf.so; do
      MOEBLAZE_LIB=$lib timeout 300 python bench.py --workload $W --steps 30 --warmup 4 --no-cpu-baseline --no-memory --no-graph 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); h=d['hbm_steps']['steps']
print('$(basename $lib)', '$W', d['ms_per_step'], h['route']['us_per_launch'], h['route']['frac_of_hbm'])"
    done
  done
done 2>&1 | tee gpurun_out/r02az_variants.txt
for lib in $L $V/rtpf.so; do
  n=$(basename $lib .so)
  for W in deepseek mixtral; do
  MOEBLAZE_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
    --kernel-name-base demangled -k "regex:tc_gemm_kernel<\(int\)8" -s 4 -c 3 --csv --log-file gpurun_out/r02az_ncu_${n}_$W.csv \
    python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --no-memory --no-graph > /dev/null 2>&1
  grep gpu__time_duration gpurun_out/r02az_ncu_${n}_$W.csv | awk -F'","' '{print "'$n' '$W'", $NF}'
  done
done
