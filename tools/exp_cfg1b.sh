#!/bin/bash
# cfg1 (dssd 1024^3) tile / split-K sweep: ms per step and the DMMA kernel rate.
for t in 64 64128 128; do for s in 0 1 2 3 4 6; do
  MDGEMM_DMMA_TILE=$t MDGEMM_SPLITK=$s timeout 120 python bench.py --workload cfg1 --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/c1.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/c1.json'));k=d['kernels']
print('tile=$t split=$s', round(d['ms_per_step']*1000,1),'us', round(d['peak_fraction'],3), {n:(v['launches'],v['ms']) for n,v in k.items()})"
done; done
