#!/bin/bash
for r in 256:1024:256 1280:2048:256 2304:3072:256 3328:4096:256; do
  timeout 600 python bench.py --sizes $r --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/s.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/s.json'));print('$r', round(d['value']), 'ms/step', round(d['ms_per_step'],1), 'frac', round(d['peak_fraction'],3), d['kernel_share'])"
done
