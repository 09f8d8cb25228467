#!/bin/bash
timeout 600 python -m pytest tests/test_pack_gpu.py tests/test_golden_gpu.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -1
for w in cfg1; do
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/p.json
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$w', round(d['value']), d['kernel_share'])"
done
timeout 300 python bench.py --labels ssss,dddd,zzzz,cccc,zczd,sddd,dssd,cdds --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/p.json
python - <<'PY'
import json
d = json.load(open('gpurun_out/p.json'))
print('8-label sweep', round(d['value']), d['kernel_share'])
PY
