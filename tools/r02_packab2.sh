#!/bin/bash
# A/B of pack-kernel builds (_ab/lib_<v>.so: source tiles per CTA x minimum CTAs per SM): bitwise pack tests,
# the packs' time inside lone calls, and the sweep.
for v in old t1b6 t2b6 t2b4 t4b3 t4b4; do
  L=$PWD/_ab/lib_$v.so
  t=$(MDGEMM_LIBRARY=$L timeout 600 python -m pytest tests/test_pack_gpu.py tests/test_golden_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1)
  r=""
  for spec in "dssd 1024" "dddd 2048" "zzzd 2048" "zzzd 4096" "cccs 1024" "dddd 4096" "ssss 4096" "sdds 512"; do set -- $spec
    r="$r | $1 $2 $(MDGEMM_LIBRARY=$L python tools/exp_lone.py --label $1 --m $2 --n $2 --k $2 --reps 5 2>&1 | grep pack | awk '{print $4}')"
  done
  s=$(MDGEMM_LIBRARY=$L timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step'],1), 'serial pack', d['kernels']['pack'])")
  echo "pack $v: [$t] sweep $s $r"
done
