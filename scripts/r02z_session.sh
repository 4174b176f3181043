# final-build session: GPU suite, smoke, benches, ncu (driver launch list, C2 at it 10 / 400, C2x8),
# digests into gpurun_out/r02z
set -x
OUT=gpurun_out/r02z; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_driver.json 2> $OUT/bench_driver.err; head -c 300 $OUT/bench_driver.json; echo
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; head -c 300 $OUT/bench.json; echo
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; head -c 300 $OUT/bench_reference.json; echo
for cfg in C1 C2x8 C3 C4 C4CT C5 C5L; do
  steps=20; [[ $cfg == C5* ]] && steps=6
  timeout 1200 python bench.py --config $cfg --steps $steps --warmup 5 --no-cpu-baseline > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err
  head -c 200 $OUT/bench_$cfg.json; echo
done
bash scripts/gpu_session.sh r02z ncu ncuC2x8 ncuC1
