#!/bin/bash
# cfg5 k=64: kernel variants
for v in "base" "MDGEMM_STREAMK=-1" "MDGEMM_DMMA_WS=-1" "MDGEMM_C_SWIZZLE=0 MDGEMM_STREAMK=-1"; do
  if [ "$v" = base ]; then E=""; else E="$v"; fi
  env $E timeout 300 python bench.py --workload cfg5-k64 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c5b.json 2>gpurun_out/c5b.err
  python -c "
import json;d=json.load(open('gpurun_out/c5b.json'))
print('$v', round(d['value']), 'ms', round(d['ms_per_step'],3), d['kernels'].get('dmma'))" || tail -3 gpurun_out/c5b.err
done
