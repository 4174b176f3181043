mkdir -p gpurun_out/r02o
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_full_gpu.py tests/test_colonies_gpu.py -m gpu -q -x -k "not C4 and not C5 and not C3" > gpurun_out/r02o/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02o/pytest.log; tail -3 gpurun_out/r02o/pytest.log
bash scripts/ab.sh r02o_c2 "--steps 20 --warmup 5" abx/libmmas_cur.so@MMAS_FB_HELPERS=0 abx/libmmas_cur.so abx/libmmas_cur.so@MMAS_FB_HELPERS=2
bash scripts/ab.sh r02o_c2_400 "--steps 400 --warmup 5" abx/libmmas_cur.so@MMAS_FB_HELPERS=0 abx/libmmas_cur.so
bash scripts/ab.sh r02o_c1 "--config C1 --steps 50 --warmup 5" abx/libmmas_cur.so@MMAS_FB_HELPERS=0 abx/libmmas_cur.so
bash scripts/ab.sh r02o_c5 "--config C5 --steps 3 --warmup 3" abx/libmmas_ls0.so abx/libmmas_cur.so
for mode in fused full; do timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_runs.py $mode > gpurun_out/r02o/racecheck_$mode.log 2>&1; tail -1 gpurun_out/r02o/racecheck_$mode.log; done
