python -m pytest tests/test_pack_gpu.py tests/test_golden_gpu.py tests/test_dual_gpu.py -q -x 2>&1 | tail -1
for i in 1 2; do python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-serial 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sweep', round(d['value']), round(d['ms_per_step'],1))"; done
python bench.py --workload cfg1 --steps 10 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1', round(d['value']), d['peak_fraction'], d['clocks'])"
python tools/exp_lone.py --label zzzd --m 4096 --n 4096 --k 4096 --reps 3 | grep pack
