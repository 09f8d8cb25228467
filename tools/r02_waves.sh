O=gpurun_out/r02w
mkdir -p $O
python -m pytest tests/test_dual_gpu.py tests/test_bench_parity_gpu.py -q -x 2>&1 | tail -1
for v in 1 2 3; do
  python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-serial > $O/run.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/run.json').read().strip().splitlines()[-1]); r=d['roofline']; print('waves', round(d['value']), round(d['ms_per_step'],1), 'dual ms', round(r['kernel_ms_per_step'],1), 'launches', r['launches'], 'dual', round(r['achieved'],2), d['clocks'].get('sm_mhz'))"
done
MDGEMM_DUAL_LOG=$O/dual.log python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-serial > /dev/null 2>&1
grep measured $O/dual.log | tail -130 | awk '{print $3, $8, $9, $10, $15, $17, $18}' | sort -k7 -n | tail -3
