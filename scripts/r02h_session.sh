#!/bin/bash
# round-2 session h: 2-opt neighbour lists on the device -- parity and the C5 create profile
OUT=gpurun_out/r02h; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest -x -q tests/test_parity_gpu.py tests/test_lean_gpu.py tests/test_parity_full_gpu.py -k "two_opt or c5 or C5 or lean" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
MMAS_CREATE_PROFILE=1 timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_C5.json 2> $OUT/bench_C5.err
grep "mmas_create" $OUT/bench_C5.err | tail -7
python -c "import json; d=json.loads(open('$OUT/bench_C5.json').readline()); print(d['value'], d['e2e']['value'], d['e2e']['seconds'])"
