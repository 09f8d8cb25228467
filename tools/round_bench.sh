#!/bin/bash
# Round-end style measurement on one GPU: tests, default bench, launch list, ncu of the top kernels.
mkdir -p gpurun_out/rb
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/rb/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/rb/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/rb/bench.json 2> gpurun_out/rb/bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/rb/bench.json'));print({k:d[k] for k in ('value','ms_per_step','peak_fraction','gpu_launches')}, d['roofline']['achieved'], d['kernel_share'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
CMD="python bench.py --labels dddd,zzzd,ssss,cccs,dssd,sddd --size 4096 --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/rb/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rb/launches.csv $CMD > gpurun_out/rb/ncu_launches.log 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma -s 1 -c 1 -o gpurun_out/rb/prof_dmma -f $CMD > gpurun_out/rb/ncu_dmma.log 2>&1; echo dmma_rc=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 1 -c 1 -o gpurun_out/rb/prof_ffma -f $CMD > gpurun_out/rb/ncu_ffma.log 2>&1; echo ffma_rc=$?
