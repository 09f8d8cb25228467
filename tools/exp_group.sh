#!/bin/bash
for g in 0 8 1; do
  for w in cfg5-k64 cfg5-k1024; do
    if [ $g = 0 ]; then unset MDGEMM_GROUP_ROWS; else export MDGEMM_GROUP_ROWS=$g; fi
    timeout 300 python bench.py --workload $w --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/g.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/g.json'));print('group $g $w', round(d['value']), round(d['ms_per_step'],2))"
  done
done
