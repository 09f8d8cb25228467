#!/bin/bash
# Round-2 measurement on one GPU: smoke, GPU tests, default bench, reference arm, launch list of smoke.
O=${1:-gpurun_out/r02}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref_rc=$?
python - $O <<'PY'
import json, sys
o = sys.argv[1]
for f in ("bench.json", "bench_ref.json"):
    try:
        d = json.loads(open(f"{o}/{f}").read().strip().splitlines()[-1])
        print(f, {k: d.get(k) for k in ("value", "ms_per_step", "peak_fraction", "gpu_launches")},
              d.get("roofline", {}).get("frac"), (d.get("e2e") or {}).get("value"), d.get("clocks"))
    except Exception as e:
        print(f, "unreadable", e)
PY
