#!/bin/bash
# compute-sanitizer over every libmlmcp kernel family (scripts/sanitize_cases.py).
# Writes gpurun_out/sanitize/<tool>_<case>.log; a summary line per run.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize
CASES=${CASES:-"fused small cluster tile coop ell graph direct"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck initcheck"}
for tool in $TOOLS; do
  for c in $CASES; do
    log=gpurun_out/sanitize/${tool}_${c}.log
    extra=""
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 900 compute-sanitizer --tool $tool $extra --kernel-name-exclude regex:native \
      --print-limit 20 python scripts/sanitize_cases.py $c > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok$' $log | tr '\n' ' ')"
  done
done
