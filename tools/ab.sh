#!/bin/bash
# A/B of the default sweep: _ab/old (another commit's build) vs this tree, alternating
ARGS=${ARGS:---steps 3 --warmup 3 --no-e2e --no-cpu}
for r in 1 2; do
  for side in old new; do
    dir=$GRAFT_REPO_ROOT; [ $side = old ] && dir=$GRAFT_REPO_ROOT/_ab/old
    (cd $dir && timeout 600 python bench.py $ARGS > $GRAFT_REPO_ROOT/gpurun_out/ab_$side.json 2>$GRAFT_REPO_ROOT/gpurun_out/ab_$side.err)
    python -c "
import json;d=json.loads([l for l in open('gpurun_out/ab_$side.json') if l.startswith('{')][-1])
print('$side', round(d['value']), round(d['ms_per_step'],1), {k:(v.get('TFLOP/s') or v.get('GB/s')) for k,v in d.get('kernels',{}).items()})" || tail -3 gpurun_out/ab_$side.err
  done
done
