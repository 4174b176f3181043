#!/bin/bash
# round-2 session z4: A/B of the compacted scan inlined / with a 2-wide round
OUT=gpurun_out/r02z4; mkdir -p $OUT
export PYTHONUNBUFFERED=1
L=paper_2003_11902_b200/libmmas.so
bash scripts/ab.sh r02z4/c2 "--steps 20 --warmup 5" $L tools/ab_inline.so tools/ab_w2.so tools/ab_inline_w2.so > /dev/null 2>&1
cat $OUT/c2/ab.txt
bash scripts/ab.sh r02z4/c2s "--steps 300 --warmup 100" $L tools/ab_inline.so tools/ab_w2.so tools/ab_inline_w2.so > /dev/null 2>&1
cat $OUT/c2s/ab.txt
