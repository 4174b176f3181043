#!/bin/bash
# round-2 evidence session: sanitizers over the new paths (compact scan, NN tour, device lists),
# then the standard session (tests, smoke, benches, ncu)
OUT=gpurun_out/r02v2; mkdir -p $OUT/sanitize
export PYTHONUNBUFFERED=1
for tool in memcheck racecheck synccheck initcheck; do
  for mode in compact fused ls; do
    timeout 900 compute-sanitizer --tool $tool python tools/sanitize_runs.py $mode > $OUT/sanitize/${tool}_$mode.log 2>&1
    echo "$tool $mode rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/sanitize/${tool}_$mode.log | tail -1)" >> $OUT/sanitize/summary.txt
  done
done
cat $OUT/sanitize/summary.txt
bash scripts/gpu_session.sh r02v2 facts tests smoke bench benchC1 benchC2x8 benchC3 benchC4 benchC4CT benchC5 benchC5L benchC65KL reference ncu ncuC3 ncuC5
