#!/bin/bash
# A/B of libmmas builds in one GPU session: bash scripts/ab.sh TAG "bench args" lib1 lib2 ...
# (alternating runs, 3 rounds; each line: lib, ms_per_step, value, fallbacks per tour)
TAG=$1; ARGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in 1 2 3; do
  for L in "$@"; do
    MMAS_LIB=$PWD/$L timeout 600 python bench.py $ARGS --no-cpu-baseline > $OUT/ab_$(basename $L)_$r.json 2>> $OUT/ab.err
    python - "$L" $OUT/ab_$(basename $L)_$r.json >> $OUT/ab.txt <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().splitlines()[0])
print(sys.argv[1], round(d["ms_per_step"], 5), round(d["value"]), d.get("fallback_steps_per_tour"), d["roofline"].get("kernel_ms"))
PY
  done
done
cat $OUT/ab.txt
