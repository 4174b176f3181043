#!/bin/bash
# round-2 last check of HEAD: GPU suite, smoke, checked suites, the driver's bench command
OUT=gpurun_out/r02head; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -2 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log; tail -2 $OUT/smoke.log
timeout 1500 python tools/checked_runs.py -q > $OUT/checked.log 2>&1; echo "checked rc=$?" >> $OUT/checked.log; tail -2 $OUT/checked.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_driver.json 2> $OUT/bench_driver.err; head -c 600 $OUT/bench_driver.json; echo
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; head -c 400 $OUT/bench_reference.json; echo
