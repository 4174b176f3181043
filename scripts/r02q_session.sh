mkdir -p gpurun_out/r02q
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/r02q/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02q/pytest.log; tail -3 gpurun_out/r02q/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02q/smoke.log 2>&1; tail -1 gpurun_out/r02q/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02q/bench_driver.json 2> gpurun_out/r02q/bench_driver.err; head -c 300 gpurun_out/r02q/bench_driver.json; echo
for mode in fused exchange full split; do timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_runs.py $mode > gpurun_out/r02q/racecheck_$mode.log 2>&1; echo $mode $(tail -1 gpurun_out/r02q/racecheck_$mode.log); done
