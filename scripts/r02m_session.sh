set -x
mkdir -p gpurun_out/r02m
timeout 1200 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/r02m/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02m/pytest.log; tail -3 gpurun_out/r02m/pytest.log
for cfg in C5L C65KL; do timeout 900 python bench.py --config $cfg --steps 4 --warmup 5 --no-cpu-baseline > gpurun_out/r02m/bench_$cfg.json 2>gpurun_out/r02m/bench_$cfg.err; head -c 250 gpurun_out/r02m/bench_$cfg.json; echo; done
MMAS_CREATE_PROFILE=1 timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02m/bench_driver.json 2> gpurun_out/r02m/bench_driver.err; head -c 300 gpurun_out/r02m/bench_driver.json; echo
bash scripts/gpu_session.sh r02m ncu ncuC1 ncuC3 ncuC4 ncuC4CT ncuC5 ncuC5L ncuC2x8
timeout 2400 bash scripts/sanitize.sh r02m_sanitize
