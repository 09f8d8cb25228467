#!/bin/bash
# ncu --set full of one kernel launch of a workload: prof_one.sh <workload> <kernel-regex> <name>
W=$1; K=$2; N=$3
CMD="python bench.py --workload $W --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain_$N.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 0 -c 1 -o gpurun_out/prof_$N -f $CMD > gpurun_out/ncu_$N.log 2>&1
echo ncu_rc=$?
