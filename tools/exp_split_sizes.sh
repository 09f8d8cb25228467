#!/bin/bash
# forced split-K factor vs size (serialized per-kind kernel rates)
for sz in ${SIZES:-1024 1536 2048 2560 3072 3584 3840}; do
  line="size $sz"
  for S in ${SPLITS:-1 2 3 4}; do
    MDGEMM_SPLITK=$S timeout 300 python bench.py --size $sz --labels ${LABELS:-dddd,ssss} --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/sp.json 2>gpurun_out/sp.err
    line="$line | S=$S $(python -c "
import json;d=json.loads([l for l in open('gpurun_out/sp.json') if l.startswith('{')][-1]);k=d['kernels']
print(round(d['value']), k.get('dmma',{}).get('TFLOP/s'), k.get('ffma',{}).get('TFLOP/s'))" 2>&1 | tail -1)"
  done
  echo "$line"
done
