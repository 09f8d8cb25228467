#!/bin/bash
# cfg1 (lone dssd 1024 call): tile / split-K variants (kernel times from the profiled serialized pass)
run() {
  name=$1; shift
  env "$@" timeout 120 python bench.py --workload cfg1 --steps 50 --warmup 10 --no-e2e --no-cpu > gpurun_out/c1_$name.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/c1_$name.json'))
print('$name', round(d['value']), 'ms', round(d['ms_per_step'],4), d['step_ms'][:3], {k:(v['ms'],v.get('TFLOP/s') or v.get('GB/s')) for k,v in d['kernels'].items()})"
}
run base
run t64128_s2 MDGEMM_DMMA_TILE=64128 MDGEMM_SPLITK=2
run t64128_s3 MDGEMM_DMMA_TILE=64128 MDGEMM_SPLITK=3
run t64_s2 MDGEMM_DMMA_TILE=64 MDGEMM_SPLITK=2
run t128_s2 MDGEMM_DMMA_TILE=128 MDGEMM_SPLITK=2
run t128_s4 MDGEMM_DMMA_TILE=128 MDGEMM_SPLITK=4
