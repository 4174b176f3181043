mkdir -p gpurun_out/r02ac
bash scripts/ab.sh r02ac_c5 "--config C5 --steps 3 --warmup 3" abx/libmmas_cur2.so abx/libmmas_lsw4.so abx/libmmas_lsw12.so abx/libmmas_lsw16.so
for k in 1 2 3; do MMAS_CREATE_PROFILE=1 timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02ac/bench_driver_$k.json 2> gpurun_out/r02ac/bench_driver_$k.err; python -c "
import json;d=json.loads(open('gpurun_out/r02ac/bench_driver_$k.json').read().splitlines()[0]);print(d['value'],d['e2e']['value'],d['e2e']['seconds'])"; grep mmas_create gpurun_out/r02ac/bench_driver_$k.err | tail -7; done
