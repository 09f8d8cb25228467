#!/bin/bash
# classic vs the three stream-K / persistent modes per size (serialized kernel rates)
for sz in ${SIZES:-2048 2560 3328 3840 4096}; do
  line="size $sz"
  for M in classic 0 1 2; do
    if [ $M = classic ]; then E="MDGEMM_STREAMK=-1"; else E="MDGEMM_STREAMK=1 MDGEMM_SKMODE=$M"; fi
    env $E timeout 300 python bench.py --size $sz --labels ${LABELS:-dddd,ssss} --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/skm.json 2>gpurun_out/skm.err
    line="$line | $M $(python -c "
import json;d=json.loads([l for l in open('gpurun_out/skm.json') if l.startswith('{')][-1]);k=d['kernels']
print(k.get('dmma',{}).get('TFLOP/s'), k.get('ffma',{}).get('TFLOP/s'))" 2>&1 | tail -1)"
  done
  echo "$line"
done
