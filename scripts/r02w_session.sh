#!/bin/bash
# round-2 session w: C2x8 ant warps per block (each warp loops over ceil(ants / slots) ants)
OUT=gpurun_out/r02w; mkdir -p $OUT
L=paper_2003_11902_b200/libmmas.so
bash scripts/ab.sh r02w/c2x8 "--config C2x8 --steps 20 --warmup 5" $L $L@MMAS_CONS_WARPS=14 $L@MMAS_CONS_WARPS=12 $L@MMAS_CONS_WARPS=8 $L@MMAS_CONS_WARPS=7 > /dev/null 2>&1
cat $OUT/c2x8/ab.txt
