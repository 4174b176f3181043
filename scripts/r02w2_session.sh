#!/bin/bash
# round-2 session w2: bounds-checked parity runs; C65KL paired vs unpaired lean fallback; C5 caps
OUT=gpurun_out/r02w2; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1800 python tools/checked_runs.py -q > $OUT/checked.log 2>&1; echo "checked rc=$?" >> $OUT/checked.log
tail -3 $OUT/checked.log
for v in 1 0; do
  MMAS_COOP_FB=$v timeout 900 python bench.py --config C65KL --steps 3 --warmup 2 --no-cpu-baseline > $OUT/c65.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c65.json').readline()); print('C65KL coop=$v', round(d['ms_per_step'],1), d['phases_ms_per_step'])"
done
for cap in 128 256 512; do
  MMAS_FB_COMPACT=$cap timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/c5.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c5.json').readline()); print('C5 cap=$cap', round(d['ms_per_step'],3), round(d['phases_ms_per_step']['construct'],3))"
done
