#!/bin/bash
# round-2 session rpf: L1 prefetch of the unvisited candidates' rows in the L2-table kernel
OUT=gpurun_out/r02rpf; mkdir -p $OUT
export PYTHONUNBUFFERED=1
L=paper_2003_11902_b200/libmmas.so
bash scripts/ab.sh r02rpf/c3 "--config C3 --steps 20 --warmup 5" tools/ab_base.so $L $L@MMAS_ROW_PF=1 > /dev/null 2>&1
cat $OUT/c3/ab.txt
for v in tools/ab_base.so "$L@MMAS_ROW_PF=1"; do
  LL=${v%@*}; E="X=1"; [[ $v == *@* ]] && E=${v#*@}
  env $E MMAS_LIB=$PWD/$LL timeout 900 python bench.py --config C5 --steps 3 --warmup 2 --no-cpu-baseline > $OUT/x.json 2>>$OUT/b.err
  python -c "import json; d=json.loads(open('$OUT/x.json').readline()); print('$v C5', round(d['ms_per_step'],2), round(d['phases_ms_per_step']['construct'],2))"
done
MMAS_ROW_PF=1 timeout 900 python -m pytest -x -q tests/test_parity_gpu.py tests/test_parity_full_gpu.py -k "C3 or clustered or pruned or l2" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
