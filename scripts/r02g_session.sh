#!/bin/bash
# round-2 session g: NN tour with the candidate fast path -- parity (limits depend on the NN
# length) and the create profile of C2 / C3 / C5
OUT=gpurun_out/r02g; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest -x -q tests/test_parity_gpu.py tests/test_parity_full_gpu.py tests/test_lean_gpu.py tests/test_colonies_gpu.py tests/test_parity_ct_gpu.py > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for cfg in C2 C3 C4 C5; do
  steps=20; [ $cfg == C5 ] && steps=2; [ $cfg == C4 ] && steps=3
  MMAS_CREATE_PROFILE=1 timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err
  echo "== $cfg"; grep "NN tour kernel" $OUT/bench_$cfg.err | head -3
  python -c "import json; d=json.loads(open('$OUT/bench_$cfg.json').readline()); print(d['value'], d['e2e']['value'], d['e2e']['seconds'])"
done
