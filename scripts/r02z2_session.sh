#!/bin/bash
# round-2 session z2: lane-compacted fallback (fixed word select) -- parity, cycles, A/B of the cap
OUT=gpurun_out/r02z2; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -x -q tests/test_fallback_compact_gpu.py tests/test_parity_full_gpu.py -k "compact or driver" > $OUT/pytest_compact.log 2>&1; echo "rc=$?" >> $OUT/pytest_compact.log
tail -3 $OUT/pytest_compact.log
(CAPS=0,4,8,12,16 python tools/fb_cycles.py C2 5 20; CAPS=0,2,4 python tools/fb_cycles.py C1 5 20; CAPS=0,4,8 python tools/fb_cycles.py C3 5 5) > $OUT/fb.txt 2>&1
python - $OUT/fb.txt <<'PY'
import sys, json
for l in open(sys.argv[1]):
    if '{' in l:
        h, j = l.split(': ', 1); d = json.loads(j)
        print(h, round(d['cycles_per_fallback']), d['compact'], round(d['ms_per_iteration'], 4), {k: v[1] for k, v in d['by_unvisited'].items()})
    else:
        print(l.strip()[:300])
PY
L=paper_2003_11902_b200/libmmas.so
bash scripts/ab.sh r02z2/c2 "--steps 20 --warmup 5" $L@MMAS_FB_COMPACT=0 $L@MMAS_FB_COMPACT=8 $L@MMAS_FB_COMPACT=12 $L@MMAS_FB_COMPACT=16 $L@MMAS_FB_COMPACT=24 > /dev/null 2>&1
cat $OUT/c2/ab.txt
bash scripts/ab.sh r02z2/c2s "--steps 300 --warmup 100" $L@MMAS_FB_COMPACT=0 $L@MMAS_FB_COMPACT=12 > /dev/null 2>&1
cat $OUT/c2s/ab.txt
