#!/bin/bash
# ncu capture of one large dual-pipe launch (sweep slice at 3584..4096)
mkdir -p gpurun_out/pd
timeout 300 python tools/exp_dual.py 3584:4096:512 > gpurun_out/pd/plain.txt 2>&1; echo plain=$?
MDGEMM_DUAL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_dual -s 3 -c 1 \
  -o gpurun_out/pd/dual -f python tools/exp_dual.py 3584:4096:512 > gpurun_out/pd/ncu.log 2>&1; echo ncu=$?
