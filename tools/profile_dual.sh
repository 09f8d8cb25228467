#!/bin/bash
# Dual-pipe kernel profiling on one B200: the ncu launch list of a bench slice
# (batched steps only), then one `ncu --set full` capture of a dual launch,
# each only after the same command exited 0 without ncu.
set -u
O=gpurun_out/profd
mkdir -p $O
CMD="python bench.py --sizes 3584:4096:512 --steps 1 --warmup 1 --no-e2e --no-cpu --no-serial"
$CMD > $O/plain.json 2> $O/plain.err; echo plain_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_dual -s 3 -c 1 -o $O/prof_dual -f $CMD > $O/ncu_dual.log 2>&1
echo dual_rc=$?
ncu -i $O/prof_dual.ncu-rep --page raw --csv > $O/ncu_dual_raw.csv 2>/dev/null
ncu -i $O/prof_dual.ncu-rep --page details --csv > $O/ncu_dual_details.csv 2>/dev/null
ncu -i $O/prof_dual.ncu-rep --page source --csv --print-source sass > $O/ncu_dual_source.csv 2>/dev/null
echo done
