#!/bin/bash
# round-2 session s: compacted fallback -- parity, then A/B of the cap on C2 (driver window,
# steady state), C1, C3, C5
OUT=gpurun_out/r02s; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -x -q tests/test_fallback_compact_gpu.py tests/test_parity_full_gpu.py -k "compact or driver" > $OUT/pytest_compact.log 2>&1; echo "rc=$?" >> $OUT/pytest_compact.log
tail -3 $OUT/pytest_compact.log
L=paper_2003_11902_b200/libmmas.so
bash scripts/ab.sh r02s/c2 "--steps 20 --warmup 5" $L@MMAS_FB_COMPACT=0 $L $L@MMAS_FB_COMPACT=200 $L@MMAS_FB_COMPACT=600 $L@MMAS_FB_COMPACT=1008 > /dev/null 2>&1
cat $OUT/c2/ab.txt
bash scripts/ab.sh r02s/c2s "--steps 300 --warmup 100" $L@MMAS_FB_COMPACT=0 $L > /dev/null 2>&1
cat $OUT/c2s/ab.txt
for cfg in C1 C3 C5; do
  steps=50; [ $cfg == C5 ] && steps=3
  for r in 1 2; do for v in 0 def; do
    if [ $v == 0 ]; then E="MMAS_FB_COMPACT=0"; else E="X=1"; fi
    env $E timeout 900 python bench.py --config $cfg --steps $steps --warmup 5 --no-cpu-baseline > $OUT/b_${cfg}_${v}_$r.json 2>>$OUT/b.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).readline()); print(sys.argv[2], sys.argv[3], round(d['ms_per_step'],4), d.get('fallback_steps_per_tour'), d['phases_ms_per_step'])" $OUT/b_${cfg}_${v}_$r.json $cfg $v >> $OUT/cfgs.txt
  done; done
done
cat $OUT/cfgs.txt
