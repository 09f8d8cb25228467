#!/bin/bash
# One ncu --set full capture of a dual launch of the 3584/4096 sweep slice with the per-instruction
# (SASS) sampling table, for the per-region stall analysis (tools/ncu_regions.py).
set -u
O=gpurun_out/dualsrc
mkdir -p $O
CMD="python bench.py --sizes 3584:4096:512 --steps 1 --warmup 1 --no-e2e --no-cpu --no-serial"
$CMD > $O/plain.json 2> $O/plain.err; echo plain_rc=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_dual -s 3 -c 1 -o $O/prof_dual -f $CMD > $O/ncu_dual.log 2>&1
echo dual_rc=$?
ncu -i $O/prof_dual.ncu-rep --page source --csv --print-source sass > $O/ncu_dual_source.csv 2>/dev/null
gzip -f $O/ncu_dual_source.csv
ls -la $O
echo done
