#!/bin/bash
for s in 512 1024 1536 2048 2560 3072 3328 3584 3840 4096; do
  timeout 300 python bench.py --size $s --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/d.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/d.json'));r=d['roofline'];print('$s', r['kernel'][:9], round(r['achieved'],2), 'frac', round(r['frac'],3), 'value', round(d['value']), 'serial_ms', round(d['serialized_step_ms'],1), 'conc_ms', round(d['ms_per_step'],1))"
done
