#!/bin/bash
# A/B of FFMA kernel variants on the comp=s labels of the sweep.
L=ssss,ddds,cccs,zzzs,sdds,zczs,cdds,szzs
for v in 0 2; do
  MDGEMM_FFMA_VARIANT=$v python bench.py --labels $L --size 4096 --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ab_ffma_$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/ab_ffma_$v.json'));print('variant $v', round(d['value']), d['roofline']['achieved'], d['kernel_share'])"
done
./tools/peaks 10 > gpurun_out/peaks2.json; cat gpurun_out/peaks2.json
