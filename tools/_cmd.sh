python -m pytest tests/test_dual_gpu.py tests/test_batch_gpu.py tests/test_pack_gpu.py -q -x 2>&1 | tail -2
for cfg in "4" "0" "4" "0"; do
  MDGEMM_DUAL_PAD=$cfg python bench.py --no-cpu --no-e2e --no-serial --steps 3 --warmup 2 > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('pad $cfg', round(d['value']), round(d['ms_per_step'],1), d['step_kernels']['dual_d']['ms'], d['step_kernels']['pack']['ms'], d['clocks']['sm_mhz'])"
done
