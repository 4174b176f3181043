mkdir -p gpurun_out/r02r
timeout 1200 python -m pytest tests -m gpu -q -x -k "two_opt or C5 or c5 or ls or local" > gpurun_out/r02r/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02r/pytest.log; tail -3 gpurun_out/r02r/pytest.log
bash scripts/ab.sh r02r_c5 "--config C5 --steps 3 --warmup 3" abx/libmmas_ls0.so abx/libmmas_mm.so
timeout 600 python tools/ls_rounds.py C5 2 2>&1 | tail -1
