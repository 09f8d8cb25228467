#!/bin/bash
for p in 200 1000 5000; do
  MDGEMM_BENCH_CLOCK_MS=$p timeout 300 python bench.py --workload cfg3 --steps 10 --warmup 5 --no-e2e --no-cpu > gpurun_out/st.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/st.json'));print('$p', round(d['value']), [round(x,1) for x in d['step_ms']], d['host_enqueue_ms'], d['clocks']['samples'])"
done
