#!/bin/bash
# round-2 session y2: larger compacted-fallback caps on the lean and HBM-row configs
OUT=gpurun_out/r02y2; mkdir -p $OUT
export PYTHONUNBUFFERED=1
for cap in 16384 32768 65535; do
  MMAS_FB_COMPACT=$cap timeout 900 python bench.py --config C65KL --steps 3 --warmup 2 --no-cpu-baseline > $OUT/c65.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c65.json').readline()); print('C65KL cap=$cap', round(d['ms_per_step'],1))"
done
for cap in 4096 9256 18512; do
  MMAS_FB_COMPACT=$cap timeout 900 python bench.py --config C5L --steps 3 --warmup 3 --no-cpu-baseline > $OUT/c5l.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c5l.json').readline()); print('C5L cap=$cap', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['construct'],2))"
done
for cap in 2048 4096 9256 18512; do
  MMAS_FB_COMPACT=$cap timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/c5.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c5.json').readline()); print('C5 cap=$cap', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['construct'],2))"
done
for cap in 64 128 256 512; do
  MMAS_FB_COMPACT=$cap timeout 900 python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/c3.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c3.json').readline()); print('C3 cap=$cap', round(d['ms_per_step'],4))"
done
