mkdir -p gpurun_out/r02n
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/r02n/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02n/pytest.log; tail -3 gpurun_out/r02n/pytest.log
bash scripts/ab.sh r02n_c5 "--config C5 --steps 3 --warmup 3" abx/libmmas_col2.so abx/libmmas_ls1.so abx/libmmas_ls1.so@MMAS_LS_CARVEOUT=70 abx/libmmas_ls1.so@MMAS_LS_CARVEOUT=50
for cfg in C5L C65KL; do timeout 900 python bench.py --config $cfg --steps 4 --warmup 5 --no-cpu-baseline > gpurun_out/r02n/bench_$cfg.json 2>gpurun_out/r02n/bench_$cfg.err; python -c "
import json;d=json.loads(open('gpurun_out/r02n/bench_$cfg.json').read().splitlines()[0]);print('$cfg',d['value'],d['ms_per_step'],d['phases_ms_per_step'])"; done
MMAS_CREATE_PROFILE=1 timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02n/bench_driver.json 2> gpurun_out/r02n/bench_driver.err; python -c "
import json;d=json.loads(open('gpurun_out/r02n/bench_driver.json').read().splitlines()[0]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['e2e']['seconds'])"; grep mmas_create gpurun_out/r02n/bench_driver.err | tail -6
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_runs.py full > gpurun_out/r02n/racecheck_full.log 2>&1; tail -2 gpurun_out/r02n/racecheck_full.log
