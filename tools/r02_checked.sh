# The GPU test suite against the checked build (device-side index checks,
# common.cuh: MDG_CHECK) -- the substitute for compute-sanitizer, which this
# pool does not allow.  A failed check prints "mdgemm device check failed"
# and traps, failing the test that launched the kernel.
O=gpurun_out/r02chk
mkdir -p $O
make -C paper_1901_06015_b200/csrc -j8 checked > $O/build.log 2>&1; echo build_rc=$?
strings paper_1901_06015_b200/libmdgemm_b200_checked.so | grep -c "device check failed" > $O/checks_compiled_in.txt
MDGEMM_LIBRARY=checked timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
   --deselect tests/test_baseline_scale_gpu.py --deselect tests/test_large_index_gpu.py > $O/pytest_checked.log 2>&1
echo checked_rc=$?; tail -3 $O/pytest_checked.log; grep -c "device check failed" $O/pytest_checked.log
python -c "import os; os.environ['MDGEMM_LIBRARY']='checked'; import paper_1901_06015_b200 as M; print(M._LIB_PATH)" >> $O/checks_compiled_in.txt
