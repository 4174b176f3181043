mkdir -p gpurun_out/r02ab
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02ab/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02ab/pytest.log; tail -2 gpurun_out/r02ab/pytest.log
for k in 1 2 3; do MMAS_CREATE_PROFILE=1 timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02ab/bench_driver_$k.json 2> gpurun_out/r02ab/bench_driver_$k.err; python -c "
import json;d=json.loads(open('gpurun_out/r02ab/bench_driver_$k.json').read().splitlines()[0]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['e2e']['seconds'])"; grep mmas_create gpurun_out/r02ab/bench_driver_$k.err | tail -6; done
