# EP stream orchestration with received rows (gloo_overlap: x_ready / y_ready / sm_reserve / C4b / C5)
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_ep.py -q -x 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_sparse_ep.py -q -x -k row_split 2>&1 | tail -2
