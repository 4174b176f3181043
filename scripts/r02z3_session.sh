#!/bin/bash
# round-2 session z3: U-capped compacted fallback with early loads + no re-evaluation of a known
# fallback step -- parity, A/B against the previous commit (tools/ab_prev.so, lane cap 12)
OUT=gpurun_out/r02z3; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -x -q tests/test_fallback_compact_gpu.py tests/test_parity_full_gpu.py tests/test_parity_gpu.py > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
L=paper_2003_11902_b200/libmmas.so
bash scripts/ab.sh r02z3/c2 "--steps 20 --warmup 5" tools/ab_prev.so $L@MMAS_FB_COMPACT=0 $L@MMAS_FB_COMPACT=160 $L $L@MMAS_FB_COMPACT=288 $L@MMAS_FB_COMPACT=384 > /dev/null 2>&1
cat $OUT/c2/ab.txt
bash scripts/ab.sh r02z3/c2s "--steps 300 --warmup 100" tools/ab_prev.so $L > /dev/null 2>&1
cat $OUT/c2s/ab.txt
