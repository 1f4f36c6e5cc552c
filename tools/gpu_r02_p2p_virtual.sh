#!/bin/bash
mkdir -p gpurun_out
for P in 2 4 8; do
  S=$(date +%s); timeout 600 python -m tests._p2p_virtual $P balanced > gpurun_out/p2p_virtual_$P.txt 2>&1
  echo "exit $? in $(( $(date +%s) - S )) s" >> gpurun_out/p2p_virtual_$P.txt
done
