O=gpurun_out/r02d
mkdir -p $O
nproc; python -c "import os; print(os.cpu_count())"
timeout 300 ./tools/copy_probe 1 2 4 8 16 64 256 > $O/copy_probe.txt 2>&1; cat $O/copy_probe.txt
for v in "" "MDGEMM_DMMA_TILE=128" "MDGEMM_STREAMK=1" "MDGEMM_SPLITK=2"; do
  echo "== $v"; env $v timeout 120 python tools/exp_lone.py
done > $O/cfg1.txt 2>&1; cat $O/cfg1.txt
for l in ddds dddd sssd zzzd; do timeout 120 python tools/exp_lone.py --label $l; done >> $O/cfg1.txt 2>&1; tail -12 $O/cfg1.txt
