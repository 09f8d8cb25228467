#!/bin/bash
# Small and medium lone calls, 40 reps: pack us per call for pack-kernel builds.
for round in 1 2; do
for v in old t1b6 t1b5 t1b4; do
  L=$PWD/_ab/lib_$v.so
  r=""
  for spec in "dssd 1024" "cccs 1024" "sdds 512" "ssss 2048" "dddd 1024" "zzzd 1024" "dssd 256" "dddd 4096" "zzzd 4096"; do set -- $spec
    r="$r | $1 $2 $(MDGEMM_LIBRARY=$L python tools/exp_lone.py --label $1 --m $2 --n $2 --k $2 --reps 40 2>&1 | grep pack | awk '{print $4}')"
  done
  echo "pack $v: $r"
done
done
