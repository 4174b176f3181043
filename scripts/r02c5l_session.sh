#!/bin/bash
OUT=gpurun_out/r02c5l; mkdir -p $OUT
L=paper_2003_11902_b200/libmmas.so
for r in 1 2 3; do for v in tools/ab_base.so $L; do
  MMAS_LIB=$PWD/$v timeout 900 python bench.py --config C5L --steps 3 --warmup 2 --no-cpu-baseline > $OUT/x.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/x.json').readline()); print('$v C5L', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['construct'],2))"
done; done
