#!/bin/bash
# Round-2 closing measurement on one B200 (profiles/r02/): smoke, the GPU
# suite, the default bench line + reference arm, every BASELINE config, the
# ncu launch list of a batched sweep slice, and ncu --set full captures of the
# kernel families -- each ncu run only after its command exited 0 without ncu.
set -u
O=gpurun_out/final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref_rc=$?
mkdir -p $O/configs
for w in cfg1 cfg3 cfg4-cdds cfg4-szzs cfg4-zczd cfg5-k64 cfg5-k256 cfg5-k1024; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 5 --no-e2e --no-cpu > $O/configs/$w.json 2> $O/configs/$w.err
done
python - $O <<'PY'
import json, sys, glob, os
o = sys.argv[1]
for f in ["bench.json", "bench_ref.json"] + sorted(os.path.relpath(p, o) for p in glob.glob(f"{o}/configs/*.json")):
    try:
        d = json.loads(open(f"{o}/{f}").read().strip().splitlines()[-1])
        r = d.get("roofline") or {}
        print(f"{f:24s} value={d['value']:.0f} peak_frac={d.get('peak_fraction')} roofline={r.get('achieved')}/{r.get('peak')} frac={r.get('frac')} e2e={(d.get('e2e') or {}).get('value')} clocks={d.get('clocks')}")
    except Exception as e:
        print(f, "unreadable", e)
PY
SLICE="python bench.py --sizes 3584:4096:512 --steps 1 --warmup 1 --no-e2e --no-cpu --no-serial"
$SLICE > $O/slice.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_slice.csv $SLICE > $O/ncu_launches.log 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_dual -s 3 -c 1 -o $O/prof_dual -f $SLICE > $O/ncu_dual.log 2>&1; echo dual_rc=$?
for spec in "dmma gemm_dmma_kernel zzzd" "ffma gemm_ffma_kernel cccs" "pack pack zzzd"; do
  set -- $spec
  C1="python tools/exp_lone.py --label $3 --m 4096 --n 4096 --k 4096 --reps 2"
  $C1 > $O/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 -o $O/prof_$1 -f $C1 > $O/ncu_$1.log 2>&1
  echo $1_rc=$?
done
for k in dual dmma ffma pack; do
  ncu -i $O/prof_$k.ncu-rep --page raw --csv > $O/ncu_${k}_raw.csv 2>/dev/null
  ncu -i $O/prof_$k.ncu-rep --page details --csv > $O/ncu_${k}_details.csv 2>/dev/null
done
ncu -i $O/prof_dual.ncu-rep --page source --csv --print-source sass > $O/ncu_dual_source.csv 2>/dev/null
python tools/ncu_stalls.py $O/ncu_dual_source.csv > $O/dual_stalls.txt 2>&1
rm -f $O/ncu_dual_source.csv
rm -f $O/*.ncu-rep   # gpurun brings back at most 64 MiB: the CSV exports are what profiles/ keeps
echo done
