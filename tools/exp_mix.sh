#!/bin/bash
# Sweep throughput under tile-shape / stream-count variants (dual-pipe co-residency experiments).
mkdir -p gpurun_out/mix
run() {
  name=$1; shift
  env "$@" timeout 300 python bench.py --no-e2e --no-cpu --steps 2 --warmup 2 > gpurun_out/mix/$name.json 2> gpurun_out/mix/$name.err
  python -c "
import json;d=json.load(open('gpurun_out/mix/$name.json'))
print('$name', round(d['value']), 'frac', round(d['peak_fraction'],3), 'step', d['step_ms'], 'serial', round(d['serialized_step_ms']), {k:(v.get('TFLOP/s') or v.get('GB/s')) for k,v in d['kernels'].items()})" || tail -3 gpurun_out/mix/$name.err
}
run base
run d64 MDGEMM_DMMA_TILE=64
run d64s8 MDGEMM_DMMA_TILE=64 MDGEMM_STREAMS=8
run s8 MDGEMM_STREAMS=8
run d64f64 MDGEMM_DMMA_TILE=64 MDGEMM_FFMA_TILE=64
run s2 MDGEMM_STREAMS=2
