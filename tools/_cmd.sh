python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu_r02.log 2>&1; echo pytest_rc=$?; tail -22 gpurun_out/pytest_gpu_r02.log
tools/r02_configs.sh gpurun_out/r02cfg_v3 slice
O=gpurun_out/r02dual4; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dual -s 3 -c 1 -o $O/prof_dual -f python bench.py --sizes 3584:4096:512 --steps 2 --warmup 1 --no-e2e --no-cpu --no-serial > $O/ncu_dual.log 2>&1; echo ncu_rc=$?
ncu -i $O/prof_dual.ncu-rep --page raw --csv > $O/ncu_dual_raw.csv 2>/dev/null
ncu -i $O/prof_dual.ncu-rep --page details --csv > $O/ncu_dual_details.csv 2>/dev/null
ncu -i $O/prof_dual.ncu-rep --page source --csv --print-source sass > $O/ncu_dual_source.csv 2>/dev/null
rm -f $O/prof_dual.ncu-rep
