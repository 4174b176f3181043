mkdir -p gpurun_out/r02aa
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_full_gpu.py -m gpu -q -x -k "staged or c5 or C5 or n1500 or two_opt" > gpurun_out/r02aa/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02aa/pytest.log; tail -2 gpurun_out/r02aa/pytest.log
bash scripts/ab.sh r02aa_c5 "--config C5 --steps 3 --warmup 3" abx/libmmas_pf2.so abx/libmmas_coop.so abx/libmmas_coop.so@MMAS_COOP_FB=0
