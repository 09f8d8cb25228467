#!/bin/bash
# Round-2 dual-kernel check on one B200: correctness tests, a bench slice,
# the default bench line, then one ncu --set full capture of a dual launch.
set -u
O=gpurun_out/r02dual
mkdir -p $O
python -m pytest tests/test_dual_gpu.py tests/test_batch_gpu.py -x -q > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -2 $O/pytest.log
CMD="python bench.py --sizes 3584:4096:512 --steps 2 --warmup 1 --no-e2e --no-cpu --no-serial"
$CMD > $O/slice.json 2> $O/slice.err; echo slice_rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02dual/slice.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("slice ms/step", round(d["ms_per_step"], 1), "GFLOPS", round(d["value"]), "dual", round(r["achieved"], 2),
      "frac", round(r["frac"], 3), "dmma", round(r["pipes"]["dmma"]["frac"], 3), "ffma", round(r["pipes"]["ffma"]["frac"], 3))
PY
if [ "${FULL:-1}" = 1 ]; then
  python bench.py --no-cpu > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
  python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print('bench', round(d['value']), d['roofline']['frac'], d['e2e']['value'] if d.get('e2e') else None, d['clocks'])"
fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dual -s 3 -c 1 -o $O/prof_dual -f $CMD > $O/ncu_dual.log 2>&1
echo ncu_rc=$?
ncu -i $O/prof_dual.ncu-rep --page raw --csv > $O/ncu_dual_raw.csv 2>/dev/null
ncu -i $O/prof_dual.ncu-rep --page details --csv > $O/ncu_dual_details.csv 2>/dev/null
ncu -i $O/prof_dual.ncu-rep --page source --csv --print-source sass > $O/ncu_dual_source.csv 2>/dev/null
echo done
