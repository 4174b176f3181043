#!/bin/bash
OUT=gpurun_out/r02prof; mkdir -p $OUT
for r in 1 2 3; do for v in 0 1; do
  E="X=1"; [ $v == 1 ] && E="BENCH_NO_PROFILE=1"
  env $E timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/b.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/b.json').readline()); print('noprof=$v', round(d['ms_per_step'],5), d['roofline'].get('kernel_ms'))"
done; done
