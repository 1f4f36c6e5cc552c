set -x
python -c "import __graft_entry__ as g; g.build()"
for TOOL in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $TOOL --print-limit 20 python tools/sanitize_small.py > gpurun_out/r02n_san_$TOOL.txt 2>&1
  echo "$TOOL exit $?"; tail -3 gpurun_out/r02n_san_$TOOL.txt
done
timeout 1800 python bench_table1.py > gpurun_out/r02n_table1.jsonl 2>gpurun_out/r02n_table1.err
python -c "
import json
for l in open('gpurun_out/r02n_table1.jsonl'):
    r=json.loads(l); print(r['conf'], r['activation'], r.get('speedup'), r.get('memory_ratio'), r.get('peak_ratio'), r['moeblaze'].get('tokens_per_s'))
"
