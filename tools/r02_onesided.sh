#!/bin/bash
# A/B of MDGEMM_DUAL_ONESIDED (share of the ready work a one-sided dual launch takes; default 0.5) on the sweep.
set -u
O=gpurun_out/onesided
mkdir -p $O
for part in 0.5 0.25 0.35 0.7 0.5; do
  MDGEMM_DUAL_ONESIDED=$part timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-serial > $O/b_$part.json 2> $O/b_$part.err
  python - $O/b_$part.json $part <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("onesided", sys.argv[2], round(d["value"]), round(d["ms_per_step"], 1), "dual ms", round(d["roofline"]["kernel_ms_per_step"], 1), "launches", d["roofline"]["launches"])
PY
done
