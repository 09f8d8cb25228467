for v in 4_4 8_8 6_6 8_6; do
  L=$PWD/_ab/lib_$v.so
  r=""
  for spec in "dssd 1024" "dddd 2048" "zzzd 2048" "zzzd 4096" "cccs 1024" "dddd 4096"; do set -- $spec
    r="$r | $1 $2 $(MDGEMM_LIBRARY=$L python tools/exp_lone.py --label $1 --m $2 --n $2 --k $2 --reps 5 2>&1 | grep pack | awk '{print $4}')"
  done
  s=skip
  echo "pack $v: sweep $s $r"
done
