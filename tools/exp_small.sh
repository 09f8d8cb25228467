#!/bin/bash
for mode in default pair; do
  if [ $mode = pair ]; then export MDGEMM_DMMA_TILE=64128 MDGEMM_FFMA_TILE=64128; else unset MDGEMM_DMMA_TILE MDGEMM_FFMA_TILE; fi
  for s in 512 1024 1536 2048; do
    timeout 300 python bench.py --size $s --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/e.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/e.json'));k=d['kernels'];print('$mode $s', 'dmma', k['dmma']['frac_of_peak'], 'ffma', k['ffma']['frac_of_peak'], 'pack', k['pack']['frac_of_hbm'], 'serial_ms', round(d['serialized_step_ms'],1), 'conc_ms', round(d['ms_per_step'],1))"
  done
done
