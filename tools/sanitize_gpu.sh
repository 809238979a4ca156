#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over tools/sanitize.py's cases.
# Logs -> gpurun_out/sanitize_<tool>_<case>.log, summary -> gpurun_out/sanitize_summary.txt
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
: > gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  for c in ${CASES:-sample onestage rank update sts prodlev}; do
    log=gpurun_out/sanitize_${tool}_${c}.log
    timeout ${SAN_TIMEOUT:-600} $CS --tool $tool --target-processes all --print-limit 50 \
        python tools/sanitize.py $c > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize case' $log | tr '\n' ' ')" >> gpurun_out/sanitize_summary.txt
  done
done
cat gpurun_out/sanitize_summary.txt
