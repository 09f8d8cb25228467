python -m pytest tests/test_dual_gpu.py tests/test_batch_gpu.py tests/test_bench_parity_gpu.py tests/test_host_staging_gpu.py tests/test_large_index_gpu.py -q -x 2>&1 | tail -2
for i in 1 2; do python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-serial 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sweep', round(d['value']), round(d['ms_per_step'],1), d['step_kernels']['pack'], 'enqueue', d['host_enqueue_ms'])"; done
python tools/exp_same_config.py --size 512 --steps 2 | head -4
python tools/exp_same_config.py --size 1024 --steps 2 | head -4
