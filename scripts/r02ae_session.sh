mkdir -p gpurun_out/r02ae
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02ae/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02ae/pytest.log; tail -2 gpurun_out/r02ae/pytest.log
bash scripts/ab.sh r02ae_c2 "--steps 20 --warmup 5" abx/libmmas_cur2.so abx/libmmas_lc5.so
bash scripts/ab.sh r02ae_c3 "--config C3 --steps 20 --warmup 5" abx/libmmas_cur2.so abx/libmmas_lc5.so
bash scripts/ab.sh r02ae_c5 "--config C5 --steps 3 --warmup 3" abx/libmmas_cur2.so abx/libmmas_lc5.so
bash scripts/ab.sh r02ae_c5l "--config C5L --steps 3 --warmup 3" abx/libmmas_cur2.so abx/libmmas_lc5.so
