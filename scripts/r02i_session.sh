#!/bin/bash
# round-2 session i: grouped 2-opt (coordinates in shared memory) -- parity, C5 A/B
OUT=gpurun_out/r02i; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest -x -q tests/test_parity_gpu.py tests/test_parity_full_gpu.py tests/test_lean_gpu.py tests/test_colonies_gpu.py -k "two_opt or c5 or C5 or lean or colon" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
L=paper_2003_11902_b200/libmmas.so
for r in 1 2; do for v in 0 1; do
  MMAS_LS_GROUP=$v timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/c5_$v_$r.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c5_$v_$r.json').readline()); print('group=$v', round(d['ms_per_step'],2), d['phases_ms_per_step'], d.get('local_search_moves_per_tour'))"
done; done
