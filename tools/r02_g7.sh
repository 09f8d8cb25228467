O=gpurun_out/r02g
mkdir -p $O
for l in dssd ssss zzzd cccs; do for s in 512 768 1024 1536; do
  for v in "MDGEMM_SKSUM=0" "MDGEMM_SKSUM=1"; do
    echo "$l $s $v: $(env $v timeout 60 python tools/exp_lone.py --label $l --m $s --n $s --k $s 2>&1 | tail -3 | tr '\n' ' ')"
  done; done; done > $O/sksum.txt 2>&1; cat $O/sksum.txt
for shape in "256 256 8192" "128 2048 4096" "2048 128 2048" "300 300 300"; do set -- $shape
  for v in "MDGEMM_SKSUM=0" "MDGEMM_SKSUM=1"; do
    echo "dddd $shape $v: $(env $v timeout 60 python tools/exp_lone.py --label dddd --m $1 --n $2 --k $3 2>&1 | tail -3 | tr '\n' ' ')"
  done; done >> $O/sksum.txt 2>&1; tail -8 $O/sksum.txt
timeout 900 python -m pytest tests/test_sksum_gpu.py tests/test_pack_gpu.py tests/test_golden_gpu.py tests/test_splitk_gpu.py tests/test_streamk_gpu.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -5 $O/pytest.log
