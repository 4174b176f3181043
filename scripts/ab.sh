#!/bin/bash
# A/B of libmmas builds / environment knobs in one GPU session:
#   bash scripts/ab.sh TAG "bench args" VARIANT1 VARIANT2 ...
# VARIANT = path/to/libmmas.so[@VAR=val,VAR=val]  (alternating runs, 3 rounds; each output line:
# variant, ms_per_step, tours/s, fallbacks per tour, construction kernel ms)
TAG=$1; ARGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in 1 2 3; do
  for V in "$@"; do
    L=${V%%@*}; E=""; [[ $V == *@* ]] && E=${V#*@}
    name=$(basename $L)_$(echo "$E" | tr ',=' '__')
    env $(echo "$E" | tr ',' ' ') MMAS_LIB=$PWD/$L timeout 600 python bench.py $ARGS --no-cpu-baseline > $OUT/ab_${name}_$r.json 2>> $OUT/ab.err
    python - "$V" $OUT/ab_${name}_$r.json >> $OUT/ab.txt <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().splitlines()[0])
print(sys.argv[1], round(d["ms_per_step"], 5), round(d["value"]), d.get("fallback_steps_per_tour"), d["roofline"].get("kernel_ms"))
PY
  done
done
cat $OUT/ab.txt
