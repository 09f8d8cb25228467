#!/bin/bash
# Spare SMs of the dual launches (packs of the next launches run on them) with the vector pack tiles.
for sp in 2 1 0 3 2 1; do
  MDGEMM_DUAL_SPARE_SMS=$sp timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-serial 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('spare $sp', round(d['value']), round(d['ms_per_step'],1), 'dual ms', round(d['roofline']['kernel_ms_per_step'],1))"
done
