#!/bin/bash
# round-2 session z5: C2 A/B -- c66ac99 (before the lean compact branch) vs HEAD vs the
# out-of-line lean compact branch
OUT=gpurun_out/r02z5; mkdir -p $OUT
export PYTHONUNBUFFERED=1
L=paper_2003_11902_b200/libmmas.so
bash scripts/ab.sh r02z5/c2 "--steps 20 --warmup 5" tools/ab_prev.so tools/ab_head.so $L > /dev/null 2>&1
cat $OUT/c2/ab.txt
bash scripts/ab.sh r02z5/c2s "--steps 300 --warmup 100" tools/ab_prev.so tools/ab_head.so $L > /dev/null 2>&1
cat $OUT/c2s/ab.txt
