# accumulator zeroing: library kernel vs cudaMemsetAsync (ZERO_KERNEL)
set -x
V=paper_2601_05296_b200/_variants
L=paper_2601_05296_b200/libmoeblaze.so
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
MOEBLAZE_LIB=$V/zk.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for r in 1 2; do
  for W in deepseek mixtral; do
    for lib in $L $V/zk.so; do
      MOEBLAZE_LIB=$lib timeout 300 python bench.py --workload $W --steps 30 --warmup 4 --no-cpu-baseline --no-memory --no-graph 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); h=d['hbm_steps']['steps']
print('$(basename $lib)', '$W', d['ms_per_step'], h['zero_acc']['us_per_launch'], h['zero_acc']['frac_of_hbm'], h['finalize_dx']['us_per_launch'])"
    done
  done
done 2>&1 | tee gpurun_out/r02ay_variants.txt
