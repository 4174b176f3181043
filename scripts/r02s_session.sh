mkdir -p gpurun_out/r02s
bash scripts/ab.sh r02s_c5 "--config C5 --steps 3 --warmup 3" abx/libmmas_rpf.so@MMAS_ROW_PF=0 abx/libmmas_rpf.so
bash scripts/ab.sh r02s_c5l "--config C5L --steps 3 --warmup 3" abx/libmmas_rpf.so@MMAS_ROW_PF=0 abx/libmmas_rpf.so
bash scripts/ab.sh r02s_c3 "--config C3 --steps 20 --warmup 5" abx/libmmas_rpf.so@MMAS_ROW_PF=0 abx/libmmas_rpf.so
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "staged or pruned or n1500 or two_opt_bit_exact" > gpurun_out/r02s/pytest.log 2>&1; tail -2 gpurun_out/r02s/pytest.log
