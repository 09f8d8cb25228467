#!/bin/bash
for t in 128 64128; do
  for w in cfg5-k64 cfg5-k256 cfg5-k1024 cfg3; do
    MDGEMM_DMMA_TILE=$t timeout 300 python bench.py --workload $w --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/t.json 2>gpurun_out/t.err
    python -c "import json;d=json.load(open('gpurun_out/t.json'));print('tile $t $w', round(d['value']), round(d['ms_per_step'],2), round(d['peak_fraction'],3))" || tail -3 gpurun_out/t.err
  done
done
MDGEMM_DMMA_TILE=64128 timeout 600 python -m pytest tests/test_gemm_fast_gpu.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -1
