#!/bin/bash
# round-2 session y: branch-free lane-compacted fallback -- cycles per fallback and A/B of the cap
OUT=gpurun_out/r02y; mkdir -p $OUT
export PYTHONUNBUFFERED=1
(CAPS=0,4,8,16,32 python tools/fb_cycles.py C2 5 20; CAPS=0,4,8 python tools/fb_cycles.py C1 5 20; CAPS=0,8,16 python tools/fb_cycles.py C3 5 5) > $OUT/fb.txt 2>&1
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
bash scripts/ab.sh r02y/c2 "--steps 20 --warmup 5" $L@MMAS_FB_COMPACT=0 $L@MMAS_FB_COMPACT=8 $L@MMAS_FB_COMPACT=16 $L > /dev/null 2>&1
cat $OUT/c2/ab.txt
