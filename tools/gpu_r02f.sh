set -x
python -c "import __graft_entry__ as g; g.build()"
for W in mixtral deepseek; do
  for C in ab abu none; do
    timeout 900 python bench.py --workload $W --checkpoint $C --no-cpu-baseline > gpurun_out/r02f_bench_${W}_$C.json 2>gpurun_out/r02f_bench_${W}_$C.err
    python -c "import json;d=json.loads(open('gpurun_out/r02f_bench_${W}_$C.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$W $C',d['value'],d['ms_per_step'],d['e2e']['value'],r['per_kernel_ms'],d['clocks']['sm_mhz'],json.dumps(d['memory']['ours'] if d['memory'] else None))"
  done
done
timeout 1500 python bench_sweep.py --T 4096 8192 16384 > gpurun_out/r02f_sweep.jsonl 2>gpurun_out/r02f_sweep.err
python -c "
import json
for l in open('gpurun_out/r02f_sweep.jsonl'):
    d=json.loads(l)
    if 'memory' in d: m=d['memory']; print(d['T'], d['tokens_per_s'], m['ours']['peak_gb'], m['materialized_baseline']['peak_gb'], m['ours']['activation_peak_gb'], m['materialized_baseline']['activation_peak_gb'], m['ours']['saved_gb'], m['materialized_baseline']['saved_gb'])
    else: print(d)
"
