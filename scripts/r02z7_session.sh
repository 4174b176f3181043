#!/bin/bash
# round-2 session z7: C2 A/B c66ac99 vs v4 (no lean compact in the smem-table kernels); lean parity
OUT=gpurun_out/r02z7; mkdir -p $OUT
export PYTHONUNBUFFERED=1
bash scripts/ab.sh r02z7/c2 "--steps 20 --warmup 5" tools/ab_prev.so tools/ab_v4.so > /dev/null 2>&1
cat $OUT/c2/ab.txt
bash scripts/ab.sh r02z7/c2s "--steps 300 --warmup 100" tools/ab_prev.so tools/ab_v4.so > /dev/null 2>&1
cat $OUT/c2s/ab.txt
timeout 900 python -m pytest -x -q tests/test_lean_gpu.py tests/test_fallback_compact_gpu.py > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
timeout 900 python bench.py --config C65KL --steps 3 --warmup 2 --no-cpu-baseline > $OUT/c65.json 2>>$OUT/b.err
python -c "import json; d=json.loads(open('$OUT/c65.json').readline()); print('C65KL', round(d['ms_per_step'],1))"
