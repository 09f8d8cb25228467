O=gpurun_out/r02s3
mkdir -p $O
for v in 0 2 0 2 0 2 1; do
  MDGEMM_DUAL_SPARE_SMS=$v python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-serial > $O/run.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/run.json').read().strip().splitlines()[-1]); r=d['roofline']; print('spare $v', round(d['value']), round(d['ms_per_step'],1), 'dual ms', round(r['kernel_ms_per_step'],1), 'dual', round(r['achieved'],2), d['clocks'].get('sm_mhz'))"
done
