#!/bin/bash
# ncu --set full of one launch of a kernel in a bench.py slice:
#   prof_k.sh <name> <kernel-regex> <bench args...>
N=$1; K=$2; shift 2
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu $*"
$CMD > gpurun_out/prof_plain_$N.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_$N -f $CMD > gpurun_out/ncu_$N.log 2>&1
echo ncu_rc=$?
