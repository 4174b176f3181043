#!/bin/bash
# round-2 session z6: C2 A/B -- c66ac99 vs variants of the compacted-scan refactor
OUT=gpurun_out/r02z6; mkdir -p $OUT
export PYTHONUNBUFFERED=1
bash scripts/ab.sh r02z6/c2 "--steps 20 --warmup 5" tools/ab_prev.so tools/ab_v2.so tools/ab_v3.so > /dev/null 2>&1
cat $OUT/c2/ab.txt
