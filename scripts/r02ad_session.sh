mkdir -p gpurun_out/r02ad
bash scripts/ab.sh r02ad_c5 "--config C5 --steps 3 --warmup 3" abx/libmmas_lsw2.so abx/libmmas_lsw3.so abx/libmmas_lsw4b.so abx/libmmas_lsw5.so abx/libmmas_lsw6.so
