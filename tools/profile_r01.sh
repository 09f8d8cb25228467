#!/bin/bash
# Round-1 profiling on one B200: launch list of a short bench run, then one
# `ncu --set full` capture per gemm kernel family (each only after the same
# command exited 0 without ncu).
set -u
mkdir -p gpurun_out
CMD="python bench.py --labels dddd,zzzd,ssss,cccs,dssd,sddd --size 4096 --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo launches_rc=$?
$CMD > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma -s 1 -c 1 -o gpurun_out/prof_dmma -f $CMD > gpurun_out/ncu_dmma.log 2>&1
echo dmma_rc=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 1 -c 1 -o gpurun_out/prof_ffma -f $CMD > gpurun_out/ncu_ffma.log 2>&1
echo ffma_rc=$?
ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 4 -c 2 -o gpurun_out/prof_pack -f $CMD > gpurun_out/ncu_pack.log 2>&1
echo pack_rc=$?
