set -x
python -c "import __graft_entry__ as g; g.build()"
for WC in deepseek:ab mixtral:ab mixtral:abu deepseek:abu deepseek:ab; do
  W=${WC%%:*}; C=${WC#*:}
  timeout 900 python bench.py --workload $W --checkpoint $C --no-cpu-baseline --no-memory > gpurun_out/r02g_bench_${W}_$C.json 2>gpurun_out/r02g_bench_${W}_$C.err
  python -c "import json;d=json.loads(open('gpurun_out/r02g_bench_${W}_$C.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$W $C',d['value'],d['ms_per_step'],d['e2e']['value'],d['e2e']['pcie'],d['e2e']['host_numa'],r['per_kernel_ms'],d['clocks']['sm_mhz'])"
done
