#!/bin/bash
# cfg5 rank-k updates (+ dddd/ssss 4096 lone calls): swizzled WS C tile on/off
for sw in 1 0; do
  for w in cfg5-k64 cfg5-k256 cfg5-k1024; do
    MDGEMM_C_SWIZZLE=$sw timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c5_$w.json 2>gpurun_out/c5_$w.err
    python -c "
import json;d=json.load(open('gpurun_out/c5_$w.json'));r=d['roofline']
print('sw=$sw $w', round(d['value']), 'frac', round(d['peak_fraction'],3), 'ms', round(d['ms_per_step'],3))" || tail -3 gpurun_out/c5_$w.err
  done
done
