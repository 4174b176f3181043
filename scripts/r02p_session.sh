mkdir -p gpurun_out/r02p
bash scripts/ab.sh r02p_c2 "--steps 20 --warmup 5" abx/libmmas_col2.so abx/libmmas_inl.so abx/libmmas_noinl.so
bash scripts/ab.sh r02p_c2_400 "--steps 400 --warmup 5" abx/libmmas_col2.so abx/libmmas_inl.so abx/libmmas_noinl.so
for L in inl noinl; do MMAS_LIB=$PWD/abx/libmmas_$L.so timeout 900 python bench.py --config C5L --steps 4 --warmup 5 --no-cpu-baseline > gpurun_out/r02p/bench_C5L_$L.json 2>gpurun_out/r02p/bench_C5L_$L.err; python -c "
import json;d=json.loads(open('gpurun_out/r02p/bench_C5L_$L.json').read().splitlines()[0]);print('C5L $L',d['value'],d['ms_per_step'],d['phases_ms_per_step'])"; done
MMAS_LIB=$PWD/abx/libmmas_noinl.so timeout 600 python -m pytest tests/test_lean_gpu.py -m gpu -q -x > gpurun_out/r02p/pytest_lean.log 2>&1; tail -2 gpurun_out/r02p/pytest_lean.log
