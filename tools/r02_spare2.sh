O=gpurun_out/r02s2
mkdir -p $O
python -m pytest tests/test_pack_gpu.py tests/test_golden_gpu.py -q -x 2>&1 | tail -1
for v in 0 2 3 0 2; do
  MDGEMM_DUAL_SPARE_SMS=$v python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-serial > $O/run.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/run.json').read().strip().splitlines()[-1]); r=d['roofline']; print('spare $v', round(d['value']), round(d['ms_per_step'],1), 'dual ms', round(r['kernel_ms_per_step'],1), 'dual', round(r['achieved'],2), d['clocks'].get('sm_mhz'))"
done
python tools/exp_lone.py --label dssd; python tools/exp_lone.py --label zzzd --m 4096 --n 4096 --k 4096 --reps 3
