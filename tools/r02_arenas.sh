O=gpurun_out/r02a3
mkdir -p $O
MDGEMM_DUAL_ARENAS=3 python -m pytest tests/test_dual_gpu.py tests/test_batch_gpu.py -q -x 2>&1 | tail -1
for v in "1 2" "1 3" "2 3" "2 4" "3 3" "1 2"; do set -- $v
  MDGEMM_DUAL_SPARE_SMS=$1 MDGEMM_DUAL_ARENAS=$2 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-serial > $O/run.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/run.json').read().strip().splitlines()[-1]); r=d['roofline']; print('spare $1 arenas $2', round(d['value']), round(d['ms_per_step'],1), 'dual ms', round(r['kernel_ms_per_step'],1), 'dual', round(r['achieved'],2), d['clocks'].get('sm_mhz'))"
done
