#!/bin/bash
# round-2 session u: lane-compacted fallback -- parity, cycles per fallback, A/B of the cap
OUT=gpurun_out/r02u; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -x -q tests/test_fallback_compact_gpu.py tests/test_parity_full_gpu.py -k "compact or driver" > $OUT/pytest_compact.log 2>&1; echo "rc=$?" >> $OUT/pytest_compact.log
tail -3 $OUT/pytest_compact.log
CAPS=0,4,8,16,32 python tools/fb_cycles.py C2 5 20 > $OUT/fb.txt 2>&1
CAPS=0,4,8,32 python tools/fb_cycles.py C1 5 20 >> $OUT/fb.txt 2>&1
CAPS=0,8,32 python tools/fb_cycles.py C3 5 5 >> $OUT/fb.txt 2>&1
cat $OUT/fb.txt
L=paper_2003_11902_b200/libmmas.so
bash scripts/ab.sh r02u/c2 "--steps 20 --warmup 5" $L@MMAS_FB_COMPACT=0 $L@MMAS_FB_COMPACT=8 $L@MMAS_FB_COMPACT=16 $L > /dev/null 2>&1
cat $OUT/c2/ab.txt
bash scripts/ab.sh r02u/c2s "--steps 300 --warmup 100" $L@MMAS_FB_COMPACT=0 $L > /dev/null 2>&1
cat $OUT/c2s/ab.txt
bash scripts/ab.sh r02u/c2x8 "--config C2x8 --steps 20 --warmup 5" $L@MMAS_FB_COMPACT=0 $L > /dev/null 2>&1
cat $OUT/c2x8/ab.txt
