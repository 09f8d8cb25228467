#!/bin/bash
# quick correctness + perf check: fast-path tests, then selected workloads
timeout 900 python -m pytest tests/test_gemm_fast_gpu.py tests/test_sharded_gpu.py tests/test_golden_gpu.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -2
for w in ${WORKLOADS:-cfg5-k64 cfg5-k256 cfg1}; do
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/q_$w.json 2>gpurun_out/q_$w.err
  python -c "
import json;d=json.load(open('gpurun_out/q_$w.json'));r=d['roofline']
print('$w', round(d['value']), 'GFLOPS frac', round(d['peak_fraction'],3), r['kernel'][:9], round(r['achieved'],2), 'ms/step', round(d['ms_per_step'],3), d['kernel_share'])" || tail -5 gpurun_out/q_$w.err
done
