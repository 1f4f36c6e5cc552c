set -x
python -c "import __graft_entry__ as g; g.build()"
for WC in deepseek:abu deepseek:ab deepseek:abu mixtral:ab deepseek:ab; do
  W=${WC%%:*}; C=${WC#*:}
  timeout 900 python bench.py --workload $W --checkpoint $C --no-cpu-baseline --no-memory > gpurun_out/r02h_bench_${W}_$C.json 2>gpurun_out/r02h_bench_${W}_$C.err
  python -c "import json;d=json.loads(open('gpurun_out/r02h_bench_${W}_$C.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$W $C',d['value'],d['ms_per_step'],d['e2e']['value'],d['e2e']['ms_per_step'],d['e2e']['allocator_in_timed_loop'],r['per_kernel_ms']['BWD_DH'],d['clocks']['sm_mhz'])"
done
