#!/bin/bash
# round-2 session g3: C3 grid (4-warp blocks, warps loop over their ants): balanced waves
OUT=gpurun_out/r02g3; mkdir -p $OUT
L=paper_2003_11902_b200/libmmas.so
bash scripts/ab.sh r02g3/c3 "--config C3 --steps 20 --warmup 5" $L $L@MMAS_CONS_GRID=475 $L@MMAS_CONS_GRID=592 $L@MMAS_CONS_GRID=317 > /dev/null 2>&1
cat $OUT/c3/ab.txt
