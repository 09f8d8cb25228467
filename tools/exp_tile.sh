#!/bin/bash
for t in 128 64; do
  for w in cfg5-k64 cfg5-k1024; do
    MDGEMM_DMMA_TILE=$t timeout 300 python bench.py --workload $w --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/t_$t_$w.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/t_$t_$w.json'));print('tile $t $w', round(d['value']), round(d['ms_per_step'],2))"
  done
done
