#!/bin/bash
# compute-sanitizer over every launch path (tools/sanitize_runs.py); logs to gpurun_out/$TAG/
TAG=${1:-r02_sanitize}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  for mode in fused separate exchange split full ls rwm; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_runs.py $mode > $OUT/${tool}_${mode}.log 2>&1
    echo "$tool $mode rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|No hazards|hazard' $OUT/${tool}_${mode}.log | tail -1)" | tee -a $OUT/summary.txt
  done
done
