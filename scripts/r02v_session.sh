mkdir -p gpurun_out/r02v
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_full_gpu.py tests/test_colonies_gpu.py tests/test_checkpoint_gpu.py -m gpu -q -x -k "not C4 and not C3 and not C5" > gpurun_out/r02v/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02v/pytest.log; tail -2 gpurun_out/r02v/pytest.log
bash scripts/ab.sh r02v_c2 "--steps 20 --warmup 5" abx/libmmas_noinl.so abx/libmmas_pf2.so
bash scripts/ab.sh r02v_c2_400 "--steps 400 --warmup 5" abx/libmmas_noinl.so abx/libmmas_pf2.so
bash scripts/ab.sh r02v_c2x8 "--config C2x8 --steps 20 --warmup 5" abx/libmmas_noinl.so abx/libmmas_pf2.so
