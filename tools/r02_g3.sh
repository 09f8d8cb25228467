O=gpurun_out/r02c
mkdir -p $O
timeout 900 python -m pytest tests/test_host_staging_gpu.py tests/test_batch_gpu.py tests/test_dual_gpu.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest.log
for s in 512 1024; do
  echo "== size $s ring"; timeout 300 python tools/exp_same_config.py --size $s
  echo "== size $s driver pageable"; MDGEMM_PAGEABLE_RING=0 timeout 300 python tools/exp_same_config.py --size $s
done > $O/same.txt 2>&1; cat $O/same.txt
MDGEMM_DUAL_LOG=$O/dual512.log timeout 300 python tools/exp_same_config.py --size 512 --steps 1 > /dev/null 2>&1; head -50 $O/dual512.log
