#!/bin/bash
# round-2 session cnt: shared-memory-tabu compacted scan sized by ballots (no word count)
OUT=gpurun_out/r02cnt; mkdir -p $OUT
export PYTHONUNBUFFERED=1
L=paper_2003_11902_b200/libmmas.so
timeout 1200 python -m pytest -x -q tests/test_fallback_compact_gpu.py tests/test_lean_gpu.py tests/test_parity_full_gpu.py -k "compact or C3 or lean or staged or C5" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
bash scripts/ab.sh r02cnt/c3 "--config C3 --steps 20 --warmup 5" tools/ab_base.so $L $L@MMAS_FB_COMPACT=128 $L@MMAS_FB_COMPACT=256 > /dev/null 2>&1
cat $OUT/c3/ab.txt
for v in tools/ab_base.so $L; do for cfg in C5 C5L C65KL; do
  st=3; [ $cfg == C65KL ] && st=2
  MMAS_LIB=$PWD/$v timeout 900 python bench.py --config $cfg --steps $st --warmup 2 --no-cpu-baseline > $OUT/x.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/x.json').readline()); print('$v $cfg', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['construct'],2))"
done; done
