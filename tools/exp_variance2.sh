#!/bin/bash
# repeated default sweeps: value, per-step device ms and host enqueue ms
for r in $(seq 1 ${REPS:-5}); do
  MDGEMM_STREAMS=${N:-4} python bench.py --steps ${STEPS:-2} --warmup 3 --no-e2e --no-cpu 2>/dev/null > gpurun_out/var.json
  python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/var.json") if l.startswith("{")][-1])
print(round(d["value"]), d.get("step_ms"), d.get("host_enqueue_ms"))
PY
done
