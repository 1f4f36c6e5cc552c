# FWD_UP row split (moe_ffn_fwd_ex / moe_dispatch_row_split) + EP forward overlap; zero-fusion reverted
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_sparse_ep.py tests/test_gpu_parity.py tests/test_gpu_ep.py -q -x 2>&1 | tail -3
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_sparse_ep.py -q -x -k "row_split" 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_ep_fullsize.py -q -x 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --ep --workload ep --no-cpu-baseline --no-memory > gpurun_out/r02ad_bench_ep_p1.json 2>gpurun_out/r02ad_bench_ep_p1.err
tail -1 gpurun_out/r02ad_bench_ep_p1.json | cut -c1-400
