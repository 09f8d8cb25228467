# A/B of the dual kernel's tuning knobs on a sweep slice (device-resident value)
O=gpurun_out/r02k
mkdir -p $O
for v in "" "MDGEMM_DUAL_STAGES=1" "MDGEMM_DUAL_SLEEP=0" "MDGEMM_DUAL_SLEEP=2000" "MDGEMM_DUAL_PREFETCH=0" "MDGEMM_DUAL_DYNAMIC=1" ""; do
  env $v python bench.py --sizes 2048:4096:1024 --steps 3 --warmup 2 --no-e2e --no-cpu --no-serial > $O/run.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/run.json').read().strip().splitlines()[-1]); r=d['roofline']; print('${v:-default}', round(d['value']), round(d['ms_per_step'],1), 'dual', round(r['achieved'],2), 'dmma', round(r['pipes']['dmma']['frac'],3), 'ffma', round(r['pipes']['ffma']['frac'],3), d['clocks'].get('sm_mhz'))"
done
