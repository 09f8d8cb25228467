#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py), one
# tool per invocation:  tools/sanitize.sh racecheck|synccheck|memcheck|initcheck [families...]
# Logs: gpurun_out/sanitize/<tool>_<family>.log; summary on stdout.
set -u
TOOL=${1:?tool}
shift
FAMS=${*:-classic ws streamk splitk dual exact pack}
OUT=${SANITIZE_OUT:-gpurun_out/sanitize}
mkdir -p "$OUT"
EXTRA=""
case "$TOOL" in
  racecheck) EXTRA="--racecheck-report all" ;;
  memcheck) EXTRA="--leak-check full" ;;
esac
rc_all=0
for f in $FAMS; do
  log="$OUT/${TOOL}_${f}.log"
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool "$TOOL" $EXTRA --print-limit 200 \
      python tools/sanitize_cases.py --family "$f" > "$log" 2>&1
  rc=$?
  summary=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize_cases" "$log" | tr '\n' ' ')
  echo "$TOOL $f rc=$rc :: $summary"
  [ $rc -ne 0 ] && rc_all=1
done
exit $rc_all
