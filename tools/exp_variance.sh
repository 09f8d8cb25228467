#!/bin/bash
# run-to-run spread of the default sweep value for 1..4 compute streams
for n in ${NS:-4 2 1}; do
  vals=""
  for r in $(seq 1 ${REPS:-4}); do
    v=$(MDGEMM_STREAMS=$n python bench.py --steps ${STEPS:-2} --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d['value']))")
    vals="$vals $v"
  done
  echo "streams=$n:$vals"
done
