#!/bin/bash
# round-2 session m: compacted fallback caps on C3 (shared-memory tabu, L2 rows) and C5 (HBM rows)
OUT=gpurun_out/r02m; mkdir -p $OUT
export PYTHONUNBUFFERED=1
for r in 1 2; do
 for cap in 0 64 128 256 512; do
  MMAS_FB_COMPACT=$cap timeout 900 python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/c3.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c3.json').readline()); print('C3 cap=$cap', round(d['ms_per_step'],4), round(d['phases_ms_per_step']['construct'],4))"
 done
 for cap in 0 32 64 128; do
  MMAS_FB_COMPACT=$cap timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/c5.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c5.json').readline()); print('C5 cap=$cap', round(d['ms_per_step'],3), round(d['phases_ms_per_step']['construct'],3))"
 done
done
