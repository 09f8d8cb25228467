#!/bin/bash
# Device-resident bench lines of the lone-call BASELINE configs + the dual slice
# (short runs, no e2e / CPU / serialized pass): tools/r02_configs.sh OUTDIR [workloads...]
set -u
O=${1:-gpurun_out/r02cfg}; shift
mkdir -p $O
WL=${*:-slice cfg1 cfg3 cfg4-cdds cfg4-zczd cfg5-k64 cfg5-k1024}
for w in $WL; do
  if [ $w = slice ]; then
    python bench.py --sizes 3584:4096:512 --steps 2 --warmup 1 --no-e2e --no-cpu --no-serial > $O/$w.json 2> $O/$w.err
  else
    python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu --no-serial > $O/$w.json 2> $O/$w.err
  fi
  python - "$O/$w.json" "$w" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    extra = ""
    if "pipes" in r:
        extra = f"dmma {r['pipes']['dmma']['frac']:.3f} ffma {r['pipes']['ffma']['frac']:.3f}"
    print(f"{sys.argv[2]:12s} {d['value']:9.0f} GFLOPS  peak_frac {d['peak_fraction']:.3f}  ms/step {d['ms_per_step']:.2f} "
          f"kernel {r.get('kernel','')[:20]} {r['achieved']:.2f} {r['unit']} frac {r['frac']:.3f} {extra} clocks {d['clocks'].get('sm_mhz')}")
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
