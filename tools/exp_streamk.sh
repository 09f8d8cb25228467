#!/bin/bash
# stream-K off vs auto per size (serialized per-kind kernel rates)
for sz in ${SIZES:-1536 2048 2560 3072 3328 3584 3840 4096}; do
  line="size $sz"
  for S in ${MODES:--1 0}; do
    MDGEMM_STREAMK=$S timeout 300 python bench.py --size $sz --labels ${LABELS:-dddd,ssss} --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/skx.json 2>gpurun_out/skx.err
    line="$line | sk=$S $(python -c "
import json;d=json.loads([l for l in open('gpurun_out/skx.json') if l.startswith('{')][-1]);k=d['kernels']
print(round(d['value']), k.get('dmma',{}).get('TFLOP/s'), k.get('ffma',{}).get('TFLOP/s'))" 2>&1 | tail -1)"
  done
  echo "$line"
done
