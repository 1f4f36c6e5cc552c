set -x
MOEBLAZE_LIB=paper_2601_05296_b200/_variants/lpt.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | grep -v "^$" | tail -40
