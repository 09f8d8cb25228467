O=gpurun_out/r02b
mkdir -p $O
timeout 900 python -m pytest tests/test_conformance_grid_gpu.py tests/test_cli.py -q -x -p no:cacheprovider > $O/pytest_new.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest_new.log
FULL=0 bash tools/r02_dual_check.sh
mkdir -p $O/dual; mv gpurun_out/r02dual/* $O/dual/ 2>/dev/null
python tools/ncu_stalls.py $O/dual/ncu_dual_source.csv > $O/dual/stalls.txt 2>&1; head -40 $O/dual/stalls.txt
