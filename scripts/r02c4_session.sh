#!/bin/bash
# round-2 session c4: compacted last steps of the full-row construction -- parity, A/B of the cap
OUT=gpurun_out/r02c4; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -x -q tests/test_fallback_compact_gpu.py tests/test_parity_gpu.py tests/test_parity_full_gpu.py -k "full_row or small_cases or C4 or colon" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for r in 1 2; do for cap in 0 250 398 600 1000; do
  MMAS_FB_COMPACT=$cap timeout 900 python bench.py --config C4 --steps 6 --warmup 3 --no-cpu-baseline > $OUT/c4.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c4.json').readline()); print('C4 cap=$cap', round(d['ms_per_step'],3))"
done; done
