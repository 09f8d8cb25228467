#!/bin/bash
# tile-raster group height vs kernel rates at long k (cfg2 slices)
for sz in ${SIZES:-4096 2048}; do
  for g in ${GROUPS_:-8 16 24 32}; do
    MDGEMM_GROUP_ROWS=$g timeout 300 python bench.py --size $sz --labels ${LABELS:-dddd,zzzd,ssss,cccs} --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/g2.json 2>gpurun_out/g2.err
    python -c "
import json;d=json.loads([l for l in open('gpurun_out/g2.json') if l.startswith('{')][-1]);k=d['kernels']
print('size $sz group $g', round(d['value']), k.get('dmma',{}).get('TFLOP/s'), k.get('ffma',{}).get('TFLOP/s'))" || tail -3 gpurun_out/g2.err
  done
done
