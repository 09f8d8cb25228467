#!/bin/bash
# Head-of-tree check on one B200: smoke, the GPU suite, the default bench line and the reference arm.
set -u
O=gpurun_out/verify
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref_rc=$?
python - $O <<'PY'
import json, sys
o = sys.argv[1]
for f in ["bench.json", "bench_ref.json"]:
    try:
        d = json.loads(open(f"{o}/{f}").read().strip().splitlines()[-1])
        r = d.get("roofline") or {}
        print(f"{f:16s} value={d['value']:.0f} ms={d.get('ms_per_step')} roofline={r.get('achieved')}/{r.get('peak')} frac={r.get('frac')} e2e={(d.get('e2e') or {}).get('value')} clocks={d.get('clocks')}")
    except Exception as e:
        print(f, "unreadable", e)
PY
echo done
