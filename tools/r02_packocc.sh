python -m pytest tests/test_pack_gpu.py tests/test_golden_gpu.py -q -x 2>&1 | tail -1
for l in dddd zzzd cccs dssd; do for s in 512 1024 2048 4096; do
  echo "$(python tools/exp_lone.py --label $l --m $s --n $s --k $s --reps 5 2>&1 | grep -E 'GFLOPS|pack' | tr '\n' ' ')"
done; done
for i in 1 2; do
python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/po.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/po.json').read().strip().splitlines()[-1]); print('sweep', round(d['value']), round(d['ms_per_step'],1), 'serial pack', d['kernels']['pack'], 'per_case', {k:v['frac_of_peak'] for k,v in d['per_case'].items()})"
done
