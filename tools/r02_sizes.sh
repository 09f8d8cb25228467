for l in ssss cccs dddd zzzd sdds; do for s in 256 512 1024 1536 2048 3072 4096; do
  echo "$(python tools/exp_lone.py --label $l --m $s --n $s --k $s --reps 5 2>&1 | tr '\n' ' ')"
done; done
