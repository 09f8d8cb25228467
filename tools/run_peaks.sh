#!/bin/bash
# Runs the arithmetic-peak microbenchmarks on the GPU box with clock sampling.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/peaks 20 > gpurun_out/peaks.json
RC=$?
kill $SMI
nproc > gpurun_out/host_nproc.txt; lscpu > gpurun_out/host_lscpu.txt; nvidia-smi > gpurun_out/nvidia_smi.txt
cat gpurun_out/peaks.json
exit $RC
