# EP config at P = 1: direct vs NCCL EP path vs peer-memory EP path, interleaved x3
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for r in 1 2 3; do
  for m in direct nccl p2p; do
    A=""; [ $m = nccl ] && A="--ep"; [ $m = p2p ] && A="--ep --ep-exchange p2p"
    timeout 600 python bench.py --workload ep $A --steps 30 --warmup 4 --no-cpu-baseline --no-memory --no-graph 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'])"
  done
done 2>&1 | tee gpurun_out/r02ar_ep_p1.txt
