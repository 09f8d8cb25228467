O=gpurun_out/r02e
mkdir -p $O
timeout 300 ./tools/copy_probe 1 2 4 8 16 64 256 > $O/copy_probe.txt 2>&1; cat $O/copy_probe.txt
timeout 900 python -m pytest tests/test_host_staging_gpu.py tests/test_streamk_gpu.py tests/test_dmma_ws_gpu.py tests/test_tile_configs_gpu.py tests/test_large_index_gpu.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest.log
for s in 512 1024 2048; do
  echo "== size $s ring"; timeout 300 python tools/exp_same_config.py --size $s --steps 2
  echo "== size $s driver pageable"; MDGEMM_PAGEABLE_RING=0 timeout 300 python tools/exp_same_config.py --size $s --steps 2
done 2>&1 | grep -v "^ " > $O/same.txt; cat $O/same.txt
