# A/B timing of the expert-GEMM engines (MOEBLAZE_GEMM = pair | cta | tma)
for G in ${ENGINES:-pair cta}; do
  echo "engine $G: $(MOEBLAZE_GEMM=$G timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-memory 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_kernel_ms"])')"
done
