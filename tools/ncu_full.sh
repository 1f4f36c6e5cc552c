#!/bin/bash
# ncu --set full of one expert-GEMM kind (TcKind id) at steady state.
# usage: tools/ncu_full.sh <kind-id> <workload> <tag> [extra bench args]
# kinds: 0 FWD_UP 1 FWD_DOWN 2 BWD_DH 3 BWD_DX 4 DW3 5 DW12 7 BWD_DH_LK
mkdir -p gpurun_out
K=$1; W=$2; TAG=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:tc_gemm_kernel<\(int\)$K," -s 3 -c 1 -f -o gpurun_out/full_${TAG}_${W}_k$K \
  python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-memory "$@" > gpurun_out/full_${TAG}_${W}_k$K.log 2>&1
echo "ncu k$K $W exit $?"
