O=gpurun_out/r02r
mkdir -p $O
MDGEMM_DUAL_REGS=1 python -m pytest tests/test_dual_gpu.py -q -x 2>&1 | tail -1
for v in 0 1 0 1; do
  MDGEMM_DUAL_REGS=$v python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-serial > $O/run.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/run.json').read().strip().splitlines()[-1]); r=d['roofline']; print('regs $v', round(d['value']), round(d['ms_per_step'],1), 'dual ms', round(r['kernel_ms_per_step'],1), 'dual', round(r['achieved'],2), 'dmma', round(r['pipes']['dmma']['frac'],3), d['clocks'].get('sm_mhz'))"
done
