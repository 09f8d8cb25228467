#!/bin/bash
# cfg1 (lone dssd 1024 call): tile / stream-K variants
run() {
  name=$1; shift
  env "$@" timeout 120 python bench.py --workload cfg1 --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/c1_$name.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/c1_$name.json'))
print('$name', round(d['value']), 'ms', round(d['ms_per_step'],4), {k:(v['ms'],v.get('TFLOP/s') or v.get('GB/s')) for k,v in d['kernels'].items()})"
}
run base
run t64128 MDGEMM_DMMA_TILE=64128
run sk64128 MDGEMM_DMMA_TILE=64128 MDGEMM_STREAMK=1
run sk64 MDGEMM_STREAMK=1
run split2 MDGEMM_SPLITK=2
