#!/bin/bash
# Every BASELINE.json config through bench.py on one GPU (device-resident value + roofline).
mkdir -p gpurun_out/all
for w in cfg1 cfg3 cfg4-cdds cfg4-szzs cfg4-zczd cfg5-k64 cfg5-k256 cfg5-k1024; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 5 --no-e2e --no-cpu > gpurun_out/all/$w.json 2> gpurun_out/all/$w.err
  python - "$w" <<'PY'
import json, sys
w = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/all/{w}.json"))
    r = d["roofline"]
    print(f"{w:12s} {d['value']:10.0f} GFLOPS  peak_frac={d['peak_fraction']:.3f}  {r['kernel'][:9]} {r['achieved']:.2f}/{r['peak']} {r['unit']}  ms/step={d['ms_per_step']:.2f} share={d['kernel_share']}")
except Exception as e:
    print(w, "FAILED", e, open(f"gpurun_out/all/{w}.err").read()[-500:])
PY
done
