#!/bin/bash
# dual-kernel variants: ring stages, C prefetch (F-only, D-only and mixed large slices, full sweep)
for v in "0 1" "1 1" "2 1" "0 0" "1 0"; do
  set -- $v
  echo "== stages $1 prefetch $2"
  for c in s ""; do
    MDGEMM_DUAL_STAGES=$1 MDGEMM_DUAL_PREFETCH=$2 timeout 300 python tools/exp_dual.py 3584:4096:512 "$c" 2 2>&1 | cut -c1-200
  done
done
for v in 0 1 2; do MDGEMM_DUAL_STAGES=$v timeout 300 python tools/exp_dual.py 256:4096:256 "" 1 2>&1 | cut -c1-200; done
