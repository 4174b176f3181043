#!/bin/bash
# round-2 session l: 2-opt with sticky tickets + one-round prefetch of queue value and neighbour row
OUT=gpurun_out/r02l; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest -x -q tests/test_parity_gpu.py tests/test_parity_full_gpu.py tests/test_lean_gpu.py tests/test_colonies_gpu.py tests/test_checkpoint_gpu.py -k "two_opt or c5 or C5 or lean or colon or ls or checkpoint or resume" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for r in 1 2; do for L in tools/ab_prev.so paper_2003_11902_b200/libmmas.so paper_2003_11902_b200/libmmas.so@G; do
  E=""; [[ $L == *@G ]] && E="MMAS_LS_GROUP=1"; LL=${L%@G}
  env $E MMAS_LIB=$PWD/$LL timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/c5.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/c5.json').readline()); print('$L', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['local_search'],2), d.get('local_search_moves_per_tour'))"
done; done
