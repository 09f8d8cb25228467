O=gpurun_out/r02f
mkdir -p $O
timeout 900 python -m pytest tests/test_sksum_gpu.py tests/test_streamk_gpu.py tests/test_splitk_gpu.py tests/test_gemm_fast_gpu.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -5 $O/pytest.log
for l in dssd ssss; do for s in 512 768 1024 1536; do
  for v in "MDGEMM_SKSUM=0" "MDGEMM_SKSUM=1 MDGEMM_SKSUM_PER_SM=1" "MDGEMM_SKSUM=1 MDGEMM_SKSUM_PER_SM=2" "MDGEMM_SKSUM=1 MDGEMM_SKSUM_PER_SM=3"; do
    echo "$l $s $v: $(env $v timeout 60 python tools/exp_lone.py --label $l --m $s --n $s --k $s | head -1)"
  done; done; done > $O/sksum.txt 2>&1; cat $O/sksum.txt
