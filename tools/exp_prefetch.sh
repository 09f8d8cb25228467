#!/bin/bash
# L2 prefetch distance sweep on cfg2 slices: per-kind kernel rates
for sz in ${SIZES:-4096 2048}; do
  for pf in ${PFS:-0 4 8 16}; do
    MDGEMM_PREFETCH=$pf timeout 300 python bench.py --size $sz --labels "${LABELS-ssss,dddd,zzzd,cccs}" --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/pf.json 2>gpurun_out/pf.err
    python -c "
import json;d=json.loads([l for l in open('gpurun_out/pf.json') if l.startswith('{')][-1]);k=d['kernels']
print('size $sz pf $pf', round(d['value']), {n:(v.get('TFLOP/s') or v.get('GB/s')) for n,v in k.items()})" || tail -3 gpurun_out/pf.err
  done
done
