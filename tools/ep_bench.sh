mkdir -p gpurun_out
for a in "--workload ep" "--workload ep --ep" "--workload mixtral --ep"; do
  echo "== $a"; timeout 600 python bench.py $a --no-cpu-baseline --no-memory --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['per_kernel_ms'], d['roofline']['all_gemms'], d.get('e2e',{}).get('value'))"
done
