#!/bin/bash
# Round-1 profiling on one B200: launch list of a short bench run, then one
# `ncu --set full` capture per kernel family (each only after the same
# command exited 0 without ncu), exported to CSV for profiles/r01/.
set -u
mkdir -p gpurun_out/prof
O=gpurun_out/prof
CMD="python bench.py --labels dddd,zzzd,ssss,cccs,dssd,sddd --size 4096 --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1
echo launches_rc=$?
# one kernel each: zzzd (DMMA, 1m: me=8192 ne=4096 ke=8192), cccs (FFMA, same dims), a 1e pack
for spec in "dmma gemm_dmma zzzd" "ffma gemm_ffma cccs" "pack pack_kernel zzzd"; do
  set -- $spec
  C1="python bench.py --labels $3 --size 4096 --steps 1 --warmup 1 --no-e2e --no-cpu"
  $C1 > $O/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 -o $O/prof_$1 -f $C1 > $O/ncu_$1.log 2>&1
  echo $1_rc=$?
  ncu -i $O/prof_$1.ncu-rep --page raw --csv > $O/ncu_$1_raw.csv 2>/dev/null
  ncu -i $O/prof_$1.ncu-rep --page details --csv > $O/ncu_$1_details.csv 2>/dev/null
done
# the warp-specialised persistent DMMA kernel (lone call, real C): dddd 4096
C2="python tools/exp_shape.py dddd 4096 4096 4096"
$C2 > $O/plain_ws.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_ws -s 1 -c 1 -o $O/prof_dmma_ws -f $C2 > $O/ncu_dmma_ws.log 2>&1
echo dmma_ws_rc=$?
ncu -i $O/prof_dmma_ws.ncu-rep --page raw --csv > $O/ncu_dmma_ws_raw.csv 2>/dev/null
ncu -i $O/prof_dmma_ws.ncu-rep --page details --csv > $O/ncu_dmma_ws_details.csv 2>/dev/null
# the epilogue-warp variant of the WS DMMA kernel (real single-precision C): cfg5 k=64
C3="python bench.py --workload cfg5-k64 --steps 1 --warmup 1 --no-e2e --no-cpu --no-serial"
$C3 > $O/plain_ws_epi.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_ws_epi -s 1 -c 1 -o $O/prof_dmma_ws_epi -f $C3 > $O/ncu_dmma_ws_epi.log 2>&1
echo dmma_ws_epi_rc=$?
ncu -i $O/prof_dmma_ws_epi.ncu-rep --page raw --csv > $O/ncu_dmma_ws_epi_raw.csv 2>/dev/null
ncu -i $O/prof_dmma_ws_epi.ncu-rep --page details --csv > $O/ncu_dmma_ws_epi_details.csv 2>/dev/null
# the dual-pipe kernel (batched sweep slice)
bash tools/profile_dual.sh
cp gpurun_out/profd/ncu_dual_raw.csv gpurun_out/profd/ncu_dual_details.csv gpurun_out/profd/launches.csv $O/ 2>/dev/null
