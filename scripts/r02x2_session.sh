#!/bin/bash
# round-2 session x2: lean compacted fallback -- parity (checked build too); C65KL / C5L caps
OUT=gpurun_out/r02x2; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest -x -q tests/test_lean_gpu.py tests/test_fallback_compact_gpu.py tests/test_parity_gpu.py -k "lean or compact or staged or pruned" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
MMAS_LIB=$PWD/tools/libmmas_checked.so timeout 900 python -m pytest -x -q tests/test_lean_gpu.py -k compact > $OUT/checked.log 2>&1; echo "checked rc=$?" >> $OUT/checked.log
tail -2 $OUT/checked.log
for cap in 0 def 16384; do
  E="X=1"; [ $cap != def ] && E="MMAS_FB_COMPACT=$cap"
  env $E timeout 900 python bench.py --config C65KL --steps 3 --warmup 2 --no-cpu-baseline > $OUT/c65.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c65.json').readline()); print('C65KL cap=$cap', round(d['ms_per_step'],1))"
done
for cap in 0 def 4096; do
  E="X=1"; [ $cap != def ] && E="MMAS_FB_COMPACT=$cap"
  env $E timeout 900 python bench.py --config C5L --steps 3 --warmup 3 --no-cpu-baseline > $OUT/c5l.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c5l.json').readline()); print('C5L cap=$cap', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['construct'],2))"
done
for cap in 512 1024 2048; do
  MMAS_FB_COMPACT=$cap timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/c5.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c5.json').readline()); print('C5 cap=$cap', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['construct'],2))"
done
