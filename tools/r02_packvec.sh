#!/bin/bash
# Vector pack tiles: bitwise pack / golden / fuzz tests, then pack us inside lone calls with and without them.
timeout 900 python -m pytest tests/test_pack_gpu.py tests/test_golden_gpu.py tests/test_fuzz_gpu.py tests/test_gemm_exact_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -3
for vec in 1 0 1 0; do
  r=""
  for spec in "dssd 1024" "ssss 2048" "dddd 1024" "sdds 512" "dssd 256" "dddd 4096" "ssss 4096" "sdds 4096" "dsss 4096" "zzzd 4096" "cccs 1024"; do set -- $spec
    r="$r | $1 $2 $(MDGEMM_PACK_VEC=$vec python tools/exp_lone.py --label $1 --m $2 --n $2 --k $2 --reps 40 2>&1 | grep pack | awk '{print $4}')"
  done
  echo "vec $vec: $r"
done
