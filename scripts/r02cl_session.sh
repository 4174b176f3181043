#!/bin/bash
OUT=gpurun_out/r02cl; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "nn_tour or candidate or small_cases or c1" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for cfg in C2 C1; do
  MMAS_CREATE_PROFILE=1 timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > $OUT/b_$cfg.json 2> $OUT/b_$cfg.err
  echo "== $cfg"; grep -E "candidate|NN tour kernel" $OUT/b_$cfg.err | tail -2
  python -c "import json; d=json.loads(open('$OUT/b_$cfg.json').readline()); print(round(d['value']), round(d['e2e']['value']), d['e2e']['seconds'])"
done
