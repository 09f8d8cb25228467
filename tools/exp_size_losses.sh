#!/bin/bash
# per-size serialized kernel time vs the ideal at measured peaks (all 128 labels)
for sz in ${SIZES:-256 512 768 1024 1280 1536 1792 2048 2304 2560 2816 3072 3328 3584 3840 4096}; do
  timeout 300 python bench.py --size $sz --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/sl.json 2>gpurun_out/sl.err
  python - $sz <<'PY'
import json,sys
d=json.loads([l for l in open('gpurun_out/sl.json') if l.startswith('{')][-1]);k=d['kernels']
dm=k.get('dmma',{}); ff=k.get('ffma',{}); pk=k.get('pack',{})
idd=dm.get('ms',0)*dm.get('frac_of_peak',0); idf=ff.get('ms',0)*ff.get('frac_of_peak',0)
print(f"size {sys.argv[1]:>5} step {d['ms_per_step']:8.2f} ms  value {d['value']:8.0f} | dmma {dm.get('ms',0):8.2f} ms ({dm.get('frac_of_peak',0):.3f}) ffma {ff.get('ms',0):8.2f} ms ({ff.get('frac_of_peak',0):.3f}) pack {pk.get('ms',0):7.2f} ms | ideal {idd+idf:8.2f} ms  loss {d['ms_per_step']-idd-idf:7.2f} ms")
PY
done
